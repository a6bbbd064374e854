#!/bin/bash
# A/B: warp-per-row PageRank units with the next row range prefetched (GBX_PR_B0PF)
mkdir -p gpurun_out
for rep in 1 2 3; do
  NOTEST=1 bash tools/gpu_prsweep.sh base:base: b0pf:b0pf: b0pf5:b0pf5: b0pf_ipl8:b0pf_ipl8: 2>&1 | grep -v "^pytest"
done
