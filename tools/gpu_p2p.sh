#!/bin/bash
mkdir -p gpurun_out/shard
for sc in 14 22; do
timeout -s KILL 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29561 tools/p2p_check.py $sc > gpurun_out/shard/p2p_$sc.log 2>&1; echo p2p $sc rc=$?; grep -v Warn gpurun_out/shard/p2p_$sc.log | tail -4
done
for ex in p2p nccl; do
GBX_PR_EXCHANGE=$ex GBX_BENCH_SHARDED=1 timeout -s KILL 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29565 bench.py --gpus 1 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/shard/bench_$ex.json 2> gpurun_out/shard/bench_$ex.err; echo bench $ex rc=$?
python -c "import json; d=json.load(open('gpurun_out/shard/bench_$ex.json')); print('$ex', d['ms_per_step'], d['config']['iterations'], d['e2e']['value'], d['config']['exchange'][:30])" || tail -3 gpurun_out/shard/bench_$ex.err
done
