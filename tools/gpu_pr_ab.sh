#!/bin/bash
# A/B of PageRank library variants (tools/build_variant.sh), interleaved:
#   bash tools/gpu_pr_ab.sh long512 [other ...]
for rep in 1 2; do
  python tools/pr_trace.py 22 2>&1 | grep -v "^iterations" | tail -3
  for v in "$@"; do
    GBX_LIB=paper_2104_01661_b200/_variants/libgbx_$v.so python tools/pr_trace.py 22 2>&1 | grep -v "^iterations" | tail -3
  done
done
