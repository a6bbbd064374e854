#!/bin/bash
mkdir -p gpurun_out/relabel
timeout -s KILL 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/relabel/pytest.log 2>&1; echo pytest rc=$?; tail -1 gpurun_out/relabel/pytest.log
for m in sort2 agather; do
echo "== $m"; GBX_PR_RELABEL=$m GBX_PLAN_TIMING=1 PYTHONPATH=. timeout -s KILL 300 python tools/e2e_phases.py 2>&1 | tail -2
done
bash tools/gpu_prsweep.sh sort::GBX_PR_RELABEL=sort2 new:: sort2::GBX_PR_RELABEL=sort2 new2::
