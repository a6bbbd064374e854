#!/bin/bash
# The N>1 bench path (C++ multi-GPU calls under torchrun) on ONE GPU: a 1-rank
# torchrun with GBX_BENCH_SHARDED=1 takes the same code path as --gpus N.
mkdir -p gpurun_out
export GBX_BENCH_SHARDED=1
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29531"
for w in pagerank tc bfs bc; do
  timeout -s KILL 600 $TR bench.py --gpus 1 --steps 5 --warmup 3 --workload $w > gpurun_out/mg_bench_$w.json 2> gpurun_out/mg_bench_$w.err
  echo "$w rc=$? $(head -c 600 gpurun_out/mg_bench_$w.json)"
  tail -2 gpurun_out/mg_bench_$w.err
done
unset GBX_BENCH_SHARDED
timeout -s KILL 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/ref.json 2>gpurun_out/ref.err; echo ref rc=$?; head -c 400 gpurun_out/ref.json
