#!/bin/bash
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?; tail -2 gpurun_out/pytest_gpu.log
timeout -s KILL 600 python bench.py > gpurun_out/bench_main.json 2> gpurun_out/bench_main.err; echo bench_rc=$?
python -c "import json; d=json.load(open('gpurun_out/bench_main.json')); print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['e2e'])"
