#!/bin/bash
# Regenerates the committed profiling evidence (profiles/rNN/): the ncu launch
# list of the headline bench command, one `ncu --set full` capture per hot
# kernel, and the per-level device timing logs of the cooperative kernels.
# Run under gpurun (one GPU); then `python tools/profiles_summarize.py rNN` here.
#   bash tools/gpu_profiles.sh r02 [pr|all]
R=${1:-r02}
WHAT=${2:-all}
OUT=gpurun_out/prof_$R
mkdir -p $OUT
NCU="timeout -s KILL 900 ncu --clock-control none"
FULL="$NCU --set full --import-source on --kernel-name-base function"
BENCH="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-secondary"
# 1) launch list of the headline bench command itself (cold, serialised
#    per-launch times; the iterations run inside ONE persistent cooperative
#    kernel, k_pr_persist), and the same with the option pagerank.host_loop=1:
#    the same row / finish code launched as one k_pr_rows + k_pr_finish pair per
#    iteration, which splits the shares.  Each command first runs plain.
$BENCH > $OUT/bench_plain.log 2>&1 && \
$NCU --metrics gpu__time_duration.sum -c 2000 --csv --log-file $OUT/bench_pagerank_launches.csv \
  $BENCH > $OUT/bench_launches.log 2>&1; echo launches rc=$?
$BENCH --option pagerank.host_loop=1 > $OUT/bench_plain_split.log 2>&1 && \
$NCU --metrics gpu__time_duration.sum -c 2000 --csv --log-file $OUT/bench_pagerank_launches_split.csv \
  $BENCH --option pagerank.host_loop=1 > $OUT/bench_launches_split.log 2>&1; echo launches-split rc=$?
# 2) full captures of the hot kernels (one launch each)
python tools/prof_pr.py 22 4 pagerank.host_loop=1 > $OUT/pr_plain.log 2>&1 && \
$FULL -k regex:'^k_pr_rows' -s 4 -c 1 -o $OUT/pagerank_k_pr_rows -f \
  python tools/prof_pr.py 22 4 pagerank.host_loop=1 > $OUT/pr.log 2>&1; echo pr rc=$?
[ "$WHAT" = "pr" ] && { echo done; exit 0; }
for w in "tc 22 ^k_tc_warp$ 0" "bc 24 ^k_bc_pull$ 0" "bc 24 ^k_bc_back$ 0" "bc 24 ^k_bc_back_push$ 2" "sssp 24 ^k_sssp_b 0" "bfs 22 ^k_bfs1$ 0" "bfs64 16 ^k_bfs64$ 0"; do
  set -- $w
  python tools/prof_algo.py $1 $2 > $OUT/${1}_plain.log 2>&1 && \
  $FULL -k regex:"$3" -s $4 -c 1 -o $OUT/${1}_$(echo $3 | tr -d '^$') -f python tools/prof_algo.py $1 $2 \
    > $OUT/${1}_ncu.log 2>&1; echo $1 rc=$?
done
# 3) cooperative-kernel level timing (%globaltimer), not a profiler run
PYTHONPATH=. timeout -s KILL 300 python tools/bfs_one.py 0 bfs.trace=1 > $OUT/bfs1_levels.txt 2>&1
timeout -s KILL 300 python bench.py --workload bfs64 --steps 1 --warmup 3 --option bfs.trace=1 2>&1 >/dev/null | grep "^bfs64" > $OUT/bfs64_levels.txt
PYTHONPATH=. timeout -s KILL 300 python tools/sssp_diag.py 24 sssp.trace=1 > $OUT/sssp_levels.txt 2>&1
echo done
