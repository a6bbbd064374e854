#!/bin/bash
mkdir -p gpurun_out
timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/bc_launches.csv python tools/prof_algo.py bc 24 > gpurun_out/bc_ncu.log 2>&1
echo rc=$?
tail -3 gpurun_out/bc_ncu.log
