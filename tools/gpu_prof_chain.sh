set -e
python bench.py --profile --steps 1 --warmup 3 > gpurun_out/pc_plain.log 2>&1
ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "timed/" -k regex:"k_project_bwd|k_adam" -c 3 \
    -o gpurun_out/chain_r01 python bench.py --profile --steps 1 --warmup 3 > gpurun_out/pc_ncu.log 2>&1
echo done
