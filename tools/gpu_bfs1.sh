#!/bin/bash
mkdir -p gpurun_out
timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "bfs" > gpurun_out/bfs_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/bfs_tests.log
tail -2 gpurun_out/bfs_tests.log
PYTHONPATH=. timeout -s KILL 300 python tools/bfs_calltime.py
for al in 14; do
GBX_BFS_ALPHA=$al timeout -s KILL 200 python bench.py --workload bfs --steps 5 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('bfs alpha=$al', d['value'], d['unit'], round(d['ms_per_step'],3))"
done
PYTHONPATH=. GBX_BFS_TLOG=1 timeout -s KILL 300 python tools/bfs_one.py 0 2>&1 | tail -10
