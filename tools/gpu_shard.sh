#!/bin/bash
# sharded PageRank: one-GPU multi-rank composition tests + the N>1 bench path on a 1-rank NCCL group
mkdir -p gpurun_out/shard
timeout -s KILL 600 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "shard" > gpurun_out/shard/pytest.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/shard/pytest.log
GBX_BENCH_SHARDED=1 timeout -s KILL 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29555 bench.py --gpus 1 --steps 5 --warmup 3 > gpurun_out/shard/bench1.json 2> gpurun_out/shard/bench1.err; echo bench rc=$?
tail -c 1500 gpurun_out/shard/bench1.json; tail -5 gpurun_out/shard/bench1.err
