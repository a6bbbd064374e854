#!/bin/bash
# A/B: 32 KB carveout (GBX_PR_CARVEOUT=10 -> 224 KB of L1) x L1 evict_last window (GBX_PR_L1_KB)
mkdir -p gpurun_out
for rep in 1 2; do
  NOTEST=1 bash tools/gpu_prsweep.sh def:: c10::GBX_PR_CARVEOUT=10 c10w144::"GBX_PR_CARVEOUT=10 GBX_PR_L1_KB=144" c10w176::"GBX_PR_CARVEOUT=10 GBX_PR_L1_KB=176" c10w192::"GBX_PR_CARVEOUT=10 GBX_PR_L1_KB=192" c10w208::"GBX_PR_CARVEOUT=10 GBX_PR_L1_KB=208" c12::GBX_PR_CARVEOUT=12 2>&1 | grep -v "^pytest\|^tail"
done
