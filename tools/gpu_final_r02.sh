# Round-2 checkpoint on one B200: build + smoke, the whole -m gpu suite, the default bench
# line and the reference arm, every config's bench line, the timed-region launch list and
# one --set full capture of the step's kernels.  Outputs under gpurun_out/final_*.
TAG=${TAG:-r02}
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/final_smoke.log 2>&1; echo "smoke rc=$?"
python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/final_gputest.log 2>&1; echo "gputest rc=$?"
python bench.py > gpurun_out/final_bench_scannetpp.jsonl 2> gpurun_out/final_bench.err; echo "bench rc=$?"
python bench.py --impl reference > gpurun_out/final_ref.jsonl 2> gpurun_out/final_ref.err; echo "ref rc=$?"
for c in tiny small replica large; do
  st=10; [ $c = large ] && st=4
  python bench.py --config $c --steps $st > gpurun_out/final_all_$c.jsonl 2> gpurun_out/final_all_$c.err; echo "$c rc=$?"
done
python bench.py --profile --steps 2 --warmup 3 > gpurun_out/final_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --nvtx --nvtx-include "timed/" \
    --csv --log-file gpurun_out/launches_timed_$TAG.csv python bench.py --profile --steps 2 --warmup 3 > gpurun_out/final_ncu1.log 2>&1
echo "launch list rc=$?"
ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "timed/" \
    -k regex:"k_render_(fwd|bwd)|k_project2|k_project_views2|k_tscatter|k_adam|k_emit|k_compact|k_onesweep|k_project_bwd|k_offsets|k_tscan|k_tcount" -c 24 \
    -o gpurun_out/full_$TAG python bench.py --profile --steps 1 --warmup 3 > gpurun_out/final_ncu2.log 2>&1
echo "full capture rc=$?"
