#!/bin/bash
mkdir -p gpurun_out/bfs
for d in 2 3 4 6 8 16; do
GBX_BFS64_PULLDIV=$d timeout -s KILL 300 python bench.py --workload bfs64 --steps 10 --warmup 3 > gpurun_out/bfs/d$d.json 2> gpurun_out/bfs/d$d.err
python -c "import json; d=json.load(open('gpurun_out/bfs/d$d.json')); print('div $d', round(d['ms_per_step'],4), 'ms', round(d['value'],1), 'GTEPS')" || tail -3 gpurun_out/bfs/d$d.err
done
