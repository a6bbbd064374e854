#!/bin/bash
mkdir -p gpurun_out
timeout -s KILL 600 ncu --set full --clock-control none --import-source on --kernel-name-base function -k regex:'^k_tc_warp$' -c 1 -o gpurun_out/tc_warp -f python tools/prof_algo.py tc 22 > gpurun_out/tc_prof.log 2>&1; echo rc=$?
