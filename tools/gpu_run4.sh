set -x
python -m pytest tests/test_gpu_parity.py -x -q -k "trainer" > gpurun_out/pytest4.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest4.log
for s in 1 2 3; do python bench.py --no-naive --no-cpu-baseline --no-e2e --streams $s > gpurun_out/bench4_s$s.log 2>&1; tail -1 gpurun_out/bench4_s$s.log | cut -c1-400; done
python bench.py --no-naive --no-cpu-baseline --streams 2 --config large --steps 3 > gpurun_out/bench4_large.log 2>&1; tail -1 gpurun_out/bench4_large.log | cut -c1-400
