#!/bin/bash
mkdir -p gpurun_out/relabel
timeout -s KILL 600 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "pagerank or pr_ or shard" > gpurun_out/relabel/pytest.log 2>&1; echo pytest rc=$?; tail -1 gpurun_out/relabel/pytest.log
GBX_PLAN_TIMING=1 PYTHONPATH=. timeout -s KILL 300 python tools/e2e_phases.py 2>&1 | tail -2
timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'k_pr_gather|k_pr_long|k_pr_list' -c 12 python tools/e2e_phases.py 2>&1 | grep -E 'k_pr_|duration' | head -24
