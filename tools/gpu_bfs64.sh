#!/bin/bash
# BFS parity tests + bfs64/bfs benches with per-level timing
mkdir -p gpurun_out
timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "bfs" > gpurun_out/bfs_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/bfs_tests.log
tail -3 gpurun_out/bfs_tests.log
for pd in 2; do
GBX_BFS64_PULLDIV=$pd timeout -s KILL 200 python bench.py --workload bfs64 --steps 5 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('bfs64 pd=$pd', d['value'], d['unit'], round(d['ms_per_step'],3))"
done
GBX_BFS_TLOG=1 timeout -s KILL 200 python bench.py --workload bfs64 --steps 1 --warmup 3 2>gpurun_out/bfs64_tlog.txt >/dev/null
tail -12 gpurun_out/bfs64_tlog.txt
timeout -s KILL 200 python bench.py --workload bfs --steps 5 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('bfs', d['value'], d['unit'], round(d['ms_per_step'],3))"
