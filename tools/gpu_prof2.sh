set -e
python bench.py --profile --steps 2 --warmup 3 > gpurun_out/p2_plain.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --nvtx --nvtx-include "timed/" \
    --csv --log-file gpurun_out/launches_timed_r01d.csv python bench.py --profile --steps 2 --warmup 3 > gpurun_out/p2_ncu1.log 2>&1
ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "timed/" \
    -k regex:"k_render_(fwd|bwd)|k_project|k_adam|k_tscatter|k_emit|k_compact" -c 14 \
    -o gpurun_out/full_r01d python bench.py --profile --steps 1 --warmup 3 > gpurun_out/p2_ncu2.log 2>&1
python bench.py --tsdf --config replica --steps 4 --warmup 2 > gpurun_out/p2_tsdf_plain.log 2>&1
ncu --set full --clock-control none -k regex:"k_tsdf|k_qt|k_seed" -c 6 -o gpurun_out/tsdf_r01d python bench.py --tsdf --config replica --steps 4 --warmup 2 > gpurun_out/p2_ncu3.log 2>&1
echo prof done
