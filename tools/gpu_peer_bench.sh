#!/bin/bash
# Code-path check of bench.py's N > 1 peer transport on a one-GPU box: two and
# four ranks share cuda:0 over gloo (DA_BENCH_SAME_GPU=1). Not a measurement.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for n in 2 4; do
  DA_BENCH_SAME_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus $n --steps 3 --warmup 3 > gpurun_out/peer_bench_$n.log 2>&1
  echo "peer bench n=$n rc=$?"; tail -1 gpurun_out/peer_bench_$n.log | cut -c1-300
done
timeout 300 python tools/probes/shard_cost.py > gpurun_out/shard_cost.log 2>&1; echo "shard_cost rc=$?"; cat gpurun_out/shard_cost.log | tail -4
