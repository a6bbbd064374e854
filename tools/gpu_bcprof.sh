#!/bin/bash
mkdir -p gpurun_out
timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "bc" > gpurun_out/bc_tests.log 2>&1; tail -2 gpurun_out/bc_tests.log
timeout -s KILL 600 ncu --set full --clock-control none --import-source on --kernel-name-base function -k regex:'^k_bc_pull$' -c 1 -o gpurun_out/bc_pull -f python tools/prof_algo.py bc 24 > gpurun_out/bc_prof1.log 2>&1; echo rc=$?
timeout -s KILL 600 ncu --set full --clock-control none --import-source on --kernel-name-base function -k regex:'^k_bc_back$' --launch-skip 4 -c 1 -o gpurun_out/bc_back -f python tools/prof_algo.py bc 24 > gpurun_out/bc_prof2.log 2>&1; echo rc=$?
timeout -s KILL 600 ncu --set full --clock-control none --import-source on --kernel-name-base function -k regex:'^k_bc_back_hub$' --launch-skip 5 -c 1 -o gpurun_out/bc_backhub -f python tools/prof_algo.py bc 24 > gpurun_out/bc_prof3.log 2>&1; echo rc=$?
