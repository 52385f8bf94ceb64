rm -f paper_2408_12677_b200/*.so oracle/*.so
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/fc_build.log 2>&1; echo "build rc=$?"
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fc_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/fc_smoke.log
python -m pytest tests -x -q -m gpu > gpurun_out/fc_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/fc_pytest.log
python bench.py > gpurun_out/fc_bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/fc_bench.log | cut -c1-300
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/fc_ref.log 2>&1; echo "ref rc=$?"; tail -1 gpurun_out/fc_ref.log | cut -c1-300
