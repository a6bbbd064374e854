#!/bin/bash
mkdir -p gpurun_out/tc
timeout -s KILL 600 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "tc or triangle" > gpurun_out/tc/pytest.log 2>&1; echo pytest rc=$?; tail -1 gpurun_out/tc/pytest.log
V=paper_2104_01661_b200/_variants
for v in base tcskip; do
if [ $v = base ]; then L=""; else L="GBX_LIB=$V/libgbx_$v.so"; fi
env $L timeout -s KILL 300 python bench.py --workload tc --steps 5 --warmup 3 > gpurun_out/tc/$v.json 2> gpurun_out/tc/$v.err
python -c "import json; d=json.load(open('gpurun_out/tc/$v.json')); print('$v', round(d['ms_per_step'],3), 'ms frac', round(d['roofline']['frac'],3))" || tail -3 gpurun_out/tc/$v.err
done
