#!/bin/bash
# PageRank shared-memory hot prefix sweep (persistent 1024-thread variant)
mkdir -p gpurun_out/sweep
GBX_PR_HOT_KB=160 timeout -s KILL 600 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "pagerank or pr_" > gpurun_out/sweep/pytest_hot.log 2>&1; echo pytest_hot rc=$?; tail -1 gpurun_out/sweep/pytest_hot.log
bash tools/gpu_prsweep.sh base:: hot96::GBX_PR_HOT_KB=96 hot128::GBX_PR_HOT_KB=128 hot160::GBX_PR_HOT_KB=160 hot192::GBX_PR_HOT_KB=192 hot160l0::"GBX_PR_HOT_KB=160 GBX_PR_L1X_KB=0" hot128l96::"GBX_PR_HOT_KB=128 GBX_PR_L1X_KB=96" hot192l16::"GBX_PR_HOT_KB=192 GBX_PR_L1X_KB=16"
