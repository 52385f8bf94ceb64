set -e
python bench.py --profile --steps 1 --warmup 3 > gpurun_out/pp_plain.log 2>&1
ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "timed/" -k regex:"k_project|k_compact|k_onesweep|k_emit" -c 8 \
    -o gpurun_out/project_r01 python bench.py --profile --steps 1 --warmup 3 > gpurun_out/pp_ncu.log 2>&1
echo done
