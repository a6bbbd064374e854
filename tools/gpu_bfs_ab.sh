#!/bin/bash
mkdir -p gpurun_out/bfs
timeout -s KILL 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "bfs" > gpurun_out/bfs/pytest.log 2>&1; echo pytest rc=$?; tail -1 gpurun_out/bfs/pytest.log
V=paper_2104_01661_b200/_variants
for v in new old new old; do
if [ $v = new ]; then L="X=1"; else L="GBX_LIB=$V/libgbx_bfsold.so"; fi
env $L timeout -s KILL 300 python bench.py --workload bfs64 --steps 20 --warmup 3 > gpurun_out/bfs/$v.json 2> gpurun_out/bfs/$v.err
python -c "import json; d=json.load(open('gpurun_out/bfs/$v.json')); print('$v bfs64', round(d['ms_per_step'],4), 'ms')" || tail -3 gpurun_out/bfs/$v.err
env $L timeout -s KILL 300 python bench.py --workload bfs --steps 10 --warmup 3 > gpurun_out/bfs/$v.json 2> gpurun_out/bfs/$v.err
python -c "import json; d=json.load(open('gpurun_out/bfs/$v.json')); print('$v bfs22', round(d['ms_per_step'],4), 'ms')" || tail -3 gpurun_out/bfs/$v.err
done
