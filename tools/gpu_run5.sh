python bench.py > gpurun_out/bench5.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench5.log
python bench.py --no-naive --no-cpu-baseline --no-e2e --streams 4 > gpurun_out/bench5_s4.log 2>&1; tail -1 gpurun_out/bench5_s4.log | cut -c1-300
