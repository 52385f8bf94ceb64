# Profile refresh: plain run first (must exit 0), then the launch list of the timed
# region (warm caches) and one --set full capture of the top kernels.
set -e
python bench.py --profile --steps 2 --warmup 3 > gpurun_out/ph_plain.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --nvtx --nvtx-include "timed/" \
    --csv --log-file gpurun_out/launches_timed_r01k.csv python bench.py --profile --steps 2 --warmup 3 > gpurun_out/ph_ncu1.log 2>&1
ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "timed/" \
    -k regex:"k_render_(fwd|bwd)|k_project<|k_tscatter|k_adam|k_emit|k_compact|k_onesweep|k_project_bwd" -c 16 \
    -o gpurun_out/full_r01k python bench.py --profile --steps 1 --warmup 3 > gpurun_out/ph_ncu2.log 2>&1
echo prof done
