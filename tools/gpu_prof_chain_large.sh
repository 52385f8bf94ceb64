set -e
# ncu --set full of config 4's wide projection-backward chain (both kernels) and Adam
ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "timed/" -k regex:"k_project_bwd|k_adam" -c 3 \
    -o gpurun_out/chain_large python bench.py --config large --profile --steps 1 --warmup 3 > gpurun_out/pcl_ncu.log 2>&1
echo done
