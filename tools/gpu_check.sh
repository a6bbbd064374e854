#!/bin/bash
# GPU check: every GPU test, smoke, then the headline bench (no CPU legs).
# usage (under gpurun): bash tools/gpu_check.sh [pytest -k expr]
mkdir -p gpurun_out
K=${1:+-k "$1"}
eval timeout -s KILL 1200 python -m pytest tests -m gpu -q -x -p no:cacheprovider $K > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?; tail -3 gpurun_out/pytest_gpu.log
timeout -s KILL 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?; tail -1 gpurun_out/smoke.log
timeout -s KILL 600 python bench.py --steps 20 --no-cpu-baseline > gpurun_out/bench_main.json 2> gpurun_out/bench_main.err; echo bench_rc=$?; cat gpurun_out/bench_main.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['roofline']['launch_ms'], d['roofline']['frac'], d['e2e']['value'], d['clocks'])"
