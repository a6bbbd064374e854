#!/bin/bash
# PageRank-only subset of tools/gpu_profiles.sh. Regenerates (profiles/rNN/): the ncu launch
# list of the headline bench command, one `ncu --set full` capture per hot
# kernel, and the per-level device timing logs of the cooperative kernels.
# Run under gpurun; then `python tools/profiles_summarize.py rNN` here.
R=${1:-r01}
OUT=gpurun_out/prof_$R
mkdir -p $OUT
NCU="timeout -s KILL 900 ncu --clock-control none"
FULL="$NCU --set full --import-source on --kernel-name-base function"
# 1) launch list of the bench command itself (cold, serialised per-launch times)
# (the PageRank iterations run inside one persistent cooperative kernel,
# k_pr_persist; GBX_PR_NO_GRAPH=1 launches the same row / finish code as one
# k_pr_rows + k_pr_finish pair per iteration, which splits the shares)
$NCU --metrics gpu__time_duration.sum -c 2000 --csv \
  --log-file $OUT/bench_pagerank_launches.csv \
  python bench.py --steps 2 --warmup 1 > $OUT/bench_launches.log 2>&1; echo launches rc=$?
GBX_PR_NO_GRAPH=1 $NCU --metrics gpu__time_duration.sum -c 2000 --csv \
  --log-file $OUT/bench_pagerank_launches_split.csv \
  python bench.py --steps 2 --warmup 1 > $OUT/bench_launches_split.log 2>&1; echo launches-split rc=$?
# 2) full captures of the hot kernels (one launch each)
GBX_PR_NO_GRAPH=1 $FULL -k regex:'^k_pr_rows' -s 4 -c 1 -o $OUT/pagerank_k_pr_rows -f \
  python tools/prof_pr.py 22 4 > $OUT/pr.log 2>&1; echo pr rc=$?
echo done
