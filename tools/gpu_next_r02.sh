# Round-2 re-measure of the NEXT rows' bench lines on the final build (one B200):
# NEXT-3 TSDF fusion, NEXT-1 keyframe schedule, the online loop (NEXT-1 + 3 + 4).
python bench.py --tsdf --config replica --steps 20 --warmup 5 > gpurun_out/next_tsdf_replica.jsonl 2> gpurun_out/next_tsdf.err; echo "tsdf rc=$?"
python bench.py --tsdf --config scannetpp --steps 20 --warmup 5 > gpurun_out/next_tsdf_scannetpp.jsonl 2> gpurun_out/next_tsdf2.err; echo "tsdf2 rc=$?"
python bench.py --schedule --config replica > gpurun_out/next_schedule_replica.jsonl 2> gpurun_out/next_sched.err; echo "sched rc=$?"
python bench.py --schedule --config scannetpp > gpurun_out/next_schedule_scannetpp.jsonl 2> gpurun_out/next_sched2.err; echo "sched2 rc=$?"
python bench.py --online --config replica --steps 100 > gpurun_out/next_online_replica.jsonl 2> gpurun_out/next_online.err; echo "online rc=$?"
