for c in tiny small replica scannetpp large; do
  st=10; [ $c = large ] && st=3
  python bench.py --config $c --steps $st > gpurun_out/all_$c.log 2>&1; echo "$c rc=$?"
done
