#!/bin/bash
# Regenerates the committed profiling evidence (profiles/rNN/): the ncu launch
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
$FULL -k regex:'^k_tc_warp$' -c 1 -o $OUT/tc_k_tc_warp -f python tools/prof_algo.py tc 22 > $OUT/tc.log 2>&1; echo tc rc=$?
$FULL -k regex:'^k_bc_pull$' -c 1 -o $OUT/bc_k_bc_pull -f python tools/prof_algo.py bc 24 > $OUT/bc1.log 2>&1; echo bc1 rc=$?
$FULL -k regex:'^k_bc_back$' -s 4 -c 1 -o $OUT/bc_k_bc_back -f python tools/prof_algo.py bc 24 > $OUT/bc2.log 2>&1; echo bc2 rc=$?
$FULL -k regex:'^k_sssp_b' -c 1 -o $OUT/sssp_k_sssp_b -f python tools/prof_algo.py sssp 24 > $OUT/sssp.log 2>&1; echo sssp rc=$?
# 3) cooperative-kernel level timing (%globaltimer), not a profiler run
PYTHONPATH=. GBX_BFS_TLOG=1 timeout -s KILL 300 python tools/bfs_one.py 0 > $OUT/bfs1_levels.txt 2>&1
GBX_BFS_TLOG=1 timeout -s KILL 300 python bench.py --workload bfs64 --steps 1 --warmup 3 2>&1 >/dev/null | grep "^bfs64" > $OUT/bfs64_levels.txt
PYTHONPATH=. GBX_SSSP_TLOG=1 timeout -s KILL 300 python tools/sssp_diag.py > $OUT/sssp_levels.txt 2>&1
echo done
