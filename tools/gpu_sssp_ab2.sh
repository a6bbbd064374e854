#!/bin/bash
mkdir -p gpurun_out/sssp
timeout -s KILL 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "sssp" > gpurun_out/sssp/pytest.log 2>&1; echo pytest rc=$?; tail -1 gpurun_out/sssp/pytest.log
V=paper_2104_01661_b200/_variants
for v in base direct base direct; do
if [ $v = base ]; then L="X=1"; else L="GBX_LIB=$V/libgbx_sssp$v.so"; fi
env $L timeout -s KILL 300 python bench.py --workload sssp --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/sssp/$v.json 2> gpurun_out/sssp/$v.err
python -c "import json; d=json.load(open('gpurun_out/sssp/$v.json')); print('$v', round(d['ms_per_step'],2), 'ms')" || tail -3 gpurun_out/sssp/$v.err
done
