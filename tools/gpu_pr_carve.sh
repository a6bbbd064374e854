#!/bin/bash
# A/B: shared-memory carveout of the persistent PageRank kernel (GBX_PR_CARVEOUT,
# percent; the driver default picked a 64 KB carveout -> 192 KB of L1)
mkdir -p gpurun_out
for rep in 1 2; do
  NOTEST=1 bash tools/gpu_prsweep.sh def:: c14::GBX_PR_CARVEOUT=14 c10::GBX_PR_CARVEOUT=10 c25::GBX_PR_CARVEOUT=25 c0::GBX_PR_CARVEOUT=0 2>&1 | grep -v "^pytest\|^tail"
done
