#!/bin/bash
mkdir -p gpurun_out
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/pr_launches.csv python bench.py --steps 2 --warmup 1 > gpurun_out/pr_ncu.log 2>&1; echo rc=$?
