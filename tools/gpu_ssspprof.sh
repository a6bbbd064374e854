#!/bin/bash
mkdir -p gpurun_out
timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k sssp > gpurun_out/sssp_tests.log 2>&1; tail -2 gpurun_out/sssp_tests.log
timeout -s KILL 900 ncu --set full --clock-control none --import-source on --kernel-name-base function -k regex:'^k_sssp_b' -c 1 -o gpurun_out/sssp_b -f python tools/prof_algo.py sssp 24 > gpurun_out/sssp_prof.log 2>&1; echo rc=$?; tail -3 gpurun_out/sssp_prof.log
