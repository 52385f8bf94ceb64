set -x
nvidia-smi -L
python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/pytest_gpu.log
python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?"; tail -3 gpurun_out/bench.log
python bench.py --config large --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_large.log 2>&1; tail -2 gpurun_out/bench_large.log
python bench.py --profile --steps 2 --warmup 3 > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --profile --steps 2 --warmup 3 > gpurun_out/ncu.log 2>&1; echo "ncu rc=$?"
