#!/bin/bash
mkdir -p gpurun_out
timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "tc" > gpurun_out/tc_tests.log 2>&1; tail -3 gpurun_out/tc_tests.log
timeout -s KILL 300 python bench.py --workload tc --steps 3 --warmup 3 2>&1 | tail -1 | cut -c1-200
timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/tc_launches.csv python tools/prof_algo.py tc 22 > gpurun_out/tc_ncu.log 2>&1
