set -e
GSR_RENDER_ROWS=1 python bench.py --config large --profile --steps 1 --warmup 3 --streams 1 > gpurun_out/pl_plain.log 2>&1
ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "timed/" -k regex:"k_render_(fwd|bwd)" -c 2 \
    -o gpurun_out/large_render env GSR_RENDER_ROWS=1 python bench.py --config large --profile --steps 1 --warmup 3 --streams 1 > gpurun_out/pl_ncu.log 2>&1
echo done
