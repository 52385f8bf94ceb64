# N > 1 launch path on one GPU: the self-launch refusal, then the exchange + optimiser
# paths at world size 1 (GSR_FORCE_DIST) with CUDA-graph capture of the whole iteration.
python bench.py --gpus 2 --steps 2 --warmup 3 > gpurun_out/dist_gpus2.log 2>&1; echo "gpus2 rc=$?" >> gpurun_out/dist_gpus2.log
for o in peer sharded replicated sparse; do
  GSR_FORCE_DIST=1 python -m torch.distributed.run --nnodes=1 --nproc-per-node=1 --master-addr 127.0.0.1 --master-port 29555 \
    bench.py --gpus 1 --steps 5 --warmup 3 --optim $o --no-e2e --no-cpu-baseline --no-naive > gpurun_out/dist_$o.log 2>&1
  echo "$o rc=$?" >> gpurun_out/dist_$o.log
done
