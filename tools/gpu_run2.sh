set -x
python -m pytest tests/test_gpu_naive.py -x -q > gpurun_out/pytest_naive.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_naive.log
python bench.py > gpurun_out/bench2.log 2>&1; echo "bench rc=$?"; tail -2 gpurun_out/bench2.log
python bench.py --profile --steps 1 --warmup 3 > gpurun_out/plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "timed/" -k regex:"k_render_(fwd|bwd)" -c 4 -o gpurun_out/render_r01b python bench.py --profile --steps 1 --warmup 3 > gpurun_out/ncu2.log 2>&1; echo "ncu rc=$?"
