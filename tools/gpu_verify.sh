python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/v_smoke.log 2>&1; echo "smoke rc=$?"
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/v_gputest.log 2>&1; echo "gputest rc=$?"
python bench.py > gpurun_out/v_bench.jsonl 2> gpurun_out/v_bench.err; echo "bench rc=$?"
