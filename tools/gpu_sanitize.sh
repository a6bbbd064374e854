#!/bin/bash
# one compute-sanitizer tool per gpurun call (B200_PROFILING.md), after a plain
# run of the same fixtures has exited 0:  bash tools/gpu_sanitize.sh memcheck
TOOL=${1:-memcheck}
mkdir -p gpurun_out
timeout -s KILL 300 python tools/sanitize.py > gpurun_out/sanitize_plain.log 2>&1 || { echo plain_failed; tail -5 gpurun_out/sanitize_plain.log; exit 1; }
EXTRA=""
[ "$TOOL" = "racecheck" ] && EXTRA="--racecheck-report all"
timeout -s KILL 2400 /usr/local/cuda/bin/compute-sanitizer --tool $TOOL $EXTRA --error-exitcode 9 \
  --log-file gpurun_out/sanitize_$TOOL.txt python tools/sanitize.py > gpurun_out/sanitize_${TOOL}_stdout.log 2>&1
echo sanitize_rc=$?
tail -3 gpurun_out/sanitize_${TOOL}_stdout.log
tail -5 gpurun_out/sanitize_$TOOL.txt
