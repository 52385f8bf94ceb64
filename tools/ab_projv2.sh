# A/B: k_project_views2 CTAs per SM (GSR_PROJV_MINB 6 / 8 default / 10 / 12), speculative staging on
python tools/projv_probe.py scannetpp libgsr.so libgsr_pvb6.so libgsr_pvb10.so libgsr_pvb12.so
python tools/projv_probe.py large libgsr.so libgsr_pvb6.so libgsr_pvb10.so libgsr_pvb12.so
