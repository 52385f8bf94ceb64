# A/B: k_project2 CTAs per SM (GSR_PROJ_MINB 8 / 10 default / 12), single-view gs_project
for c in scannetpp large replica; do PROBE_SINGLE=1 python tools/projv_probe.py $c libgsr.so libgsr_pb8.so libgsr_pb12.so; done
LIBS="libgsr.so libgsr_pb8.so libgsr.so libgsr_pb8.so" CFGS="replica scannetpp" STEPS=20 bash tools/ab_lib.sh
