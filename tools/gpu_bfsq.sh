#!/bin/bash
mkdir -p gpurun_out/bfs
timeout -s KILL 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "bfs" > gpurun_out/bfs/pytest.log 2>&1; echo pytest rc=$?; tail -1 gpurun_out/bfs/pytest.log
timeout -s KILL 600 python -m pytest tests/test_full_configs_gpu.py -q -x -p no:cacheprovider -k "bfs" 2>&1 | tail -1
for i in 1 2; do
timeout -s KILL 300 python bench.py --workload bfs64 --steps 20 --warmup 3 > gpurun_out/bfs/b64.json 2> gpurun_out/bfs/b64.err
python -c "import json; d=json.load(open('gpurun_out/bfs/b64.json')); print('bfs64', round(d['ms_per_step'],4), 'ms', round(d['value'],1), 'GTEPS frac', round(d['roofline']['frac'],3))" || tail -3 gpurun_out/bfs/b64.err
timeout -s KILL 300 python bench.py --workload bfs --steps 10 --warmup 3 > gpurun_out/bfs/b1.json 2> gpurun_out/bfs/b1.err
python -c "import json; d=json.load(open('gpurun_out/bfs/b1.json')); print('bfs22', round(d['ms_per_step'],3), 'ms', round(d['value'],1), 'GTEPS frac', round(d['roofline']['frac'],3))" || tail -3 gpurun_out/bfs/b1.err
done
GBX_BFS_TLOG=1 timeout -s KILL 300 python bench.py --workload bfs64 --steps 1 --warmup 3 2>&1 >/dev/null | grep "^bfs64" | head -7
