# A/B of (env, library) pairs on the device-timed step: RUNS="ENV=a:libgsr.so ENV=b:libgsr_x.so" CFGS="large"
for c in ${CFGS:-large}; do for run in $RUNS; do
  e=${run%%:*}; L=${run#*:}
  env $e GSR_LIB=$L python bench.py --config $c --steps ${STEPS:-6} --warmup 3 --no-e2e --no-naive --no-cpu-baseline 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); st={k: round(v*1000,1) for k,v in d['stage_ms'].items()}; print('$c $e $L', round(d['ms_per_step'],3), st)"
done; done
