# A/B of the bin streams' lag (GSR_BIN_LAG) and head-first binning (GSR_BIN_HEAD) at scannetpp / config 4
for cfg in scannetpp; do
for e in "GSR_BIN_LAG=0" "GSR_BIN_HEAD=1" "GSR_BIN_LAG=4" "GSR_BIN_LAG=2" "GSR_BIN_LAG=0" "GSR_BIN_HEAD=1" "GSR_BIN_LAG=3" "GSR_BIN_LAG=6"; do
  env $e python bench.py --config $cfg --steps 20 --no-e2e --no-cpu-baseline --no-naive > gpurun_out/ab_$cfg.tmp 2>/dev/null
  python -c "import json,sys; d=json.loads(open('gpurun_out/ab_$cfg.tmp').readline()); print('$cfg', '$e', round(d['ms_per_step'],4))"
done; done
