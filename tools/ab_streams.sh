# config-4 / scannetpp step time vs render / bin streams (32 hardware queues)
for c in ${CFGS:-large}; do
for s in ${STREAMS:-8 12 16}; do for b in ${BINS:-8}; do
  GSR_BIN_STREAMS=$b python bench.py --config $c --streams $s --steps ${STEPS:-6} --warmup 3 --no-e2e --no-naive --no-cpu-baseline 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c streams $s bins $b', round(d['ms_per_step'],2))"
done; done; done
