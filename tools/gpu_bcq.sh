#!/bin/bash
mkdir -p gpurun_out/bc
timeout -s KILL 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "bc or betweenness" > gpurun_out/bc/pytest.log 2>&1; echo pytest rc=$?; tail -1 gpurun_out/bc/pytest.log
V=paper_2104_01661_b200/_variants
for v in new old new old; do
if [ $v = new ]; then L="X=1"; else L="GBX_LIB=$V/libgbx_bcold.so"; fi
env $L timeout -s KILL 300 python bench.py --workload bc --steps 5 --warmup 3 > gpurun_out/bc/$v.json 2> gpurun_out/bc/$v.err
python -c "import json; d=json.load(open('gpurun_out/bc/$v.json')); print('$v', round(d['ms_per_step'],3), 'ms')" || tail -3 gpurun_out/bc/$v.err
done
