python -m pytest tests/test_gpu_parity.py -x -q -k "keyframe" > gpurun_out/pytest8.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest8.log
python bench.py --config replica --schedule > gpurun_out/sched_replica.log 2>&1; echo rc=$?; tail -1 gpurun_out/sched_replica.log
python bench.py --config scannetpp --schedule > gpurun_out/sched_scannetpp.log 2>&1; echo rc=$?; tail -1 gpurun_out/sched_scannetpp.log
