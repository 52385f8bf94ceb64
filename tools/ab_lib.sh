# A/B of library builds (GSR_LIB=...) on the device-timed step: LIBS="libgsr.so libgsr_x.so" CFGS="large scannetpp"
for c in ${CFGS:-large}; do for L in ${LIBS:-libgsr.so}; do
  GSR_LIB=$L python bench.py --config $c --steps ${STEPS:-6} --warmup 3 --no-e2e --no-naive --no-cpu-baseline 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); st={k: round(v*1000,1) for k,v in d['stage_ms'].items()}; print('$c $L', round(d['ms_per_step'],3), st)"
done; done
