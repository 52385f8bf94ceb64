set -x
python bench.py --no-naive --no-cpu-baseline > gpurun_out/bench3.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench3.log
python bench.py --profile --steps 2 --warmup 3 > gpurun_out/plain3.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --nvtx --nvtx-include "timed/" --csv --log-file gpurun_out/launches_warm.csv python bench.py --profile --steps 2 --warmup 3 > gpurun_out/ncu3.log 2>&1; echo "ncu rc=$?"
