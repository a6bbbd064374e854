#!/bin/bash
mkdir -p gpurun_out/bc
PYTHONPATH=. timeout -s KILL 300 python tools/bc_breakdown.py 24 2>&1 | tail -2
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/bc/launches.csv python tools/bc_breakdown.py 24 > gpurun_out/bc/ncu.log 2>&1; echo ncu rc=$?
