# A/B: speculative staging of the 8 non-mean rows in gs_project_views (GSR_PROJV_SPEC)
python tools/projv_probe.py scannetpp libgsr.so libgsr_pvspec.so
python tools/projv_probe.py large libgsr.so libgsr_pvspec.so
LIBS="libgsr.so libgsr_pvspec.so libgsr.so libgsr_pvspec.so" CFGS="scannetpp" STEPS=20 bash tools/ab_lib.sh
LIBS="libgsr.so libgsr_pvspec.so" CFGS="large" STEPS=4 bash tools/ab_lib.sh
