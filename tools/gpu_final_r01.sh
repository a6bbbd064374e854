#!/bin/bash
# Round-end check after the PageRank carveout change: every GPU test, smoke,
# the headline bench, then the PageRank profiling subset.
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?; tail -1 gpurun_out/pytest_gpu.log
timeout -s KILL 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?; tail -1 gpurun_out/smoke.log
timeout -s KILL 600 python bench.py > gpurun_out/bench_main.json 2> gpurun_out/bench_main.err; echo bench_rc=$?; cat gpurun_out/bench_main.json
bash tools/gpu_profiles_pr.sh r01
