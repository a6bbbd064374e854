#!/bin/bash
# PageRank tests with the 32 KB carveout default, then the L1 evict_last window sweep
mkdir -p gpurun_out
timeout -s KILL 600 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "pagerank or pr_ or smoke or full" > gpurun_out/pytest_pr.log 2>&1; echo pytest rc=$?; tail -1 gpurun_out/pytest_pr.log
for rep in 1 2; do
  NOTEST=1 bash tools/gpu_prsweep.sh w160:: w144::GBX_PR_L1_KB=144 w128::GBX_PR_L1_KB=128 w112::GBX_PR_L1_KB=112 w96::GBX_PR_L1_KB=96 w64::GBX_PR_L1_KB=64 2>&1 | grep -v "^pytest\|^tail"
done
