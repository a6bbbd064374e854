#!/bin/bash
# A/B: PageRank rows kernel at 8 resident CTAs per SM (32 registers) x gathers in flight
mkdir -p gpurun_out
for rep in 1 2; do
  NOTEST=1 bash tools/gpu_prsweep.sh base:base: m8:m8: m8i8:m8i8: m8i4:m8i4: m8i4b1:m8i4b1: 2>&1 | grep -v "^pytest\|^tail"
done
