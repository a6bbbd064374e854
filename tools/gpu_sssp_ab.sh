#!/bin/bash
# SSSP A/B: parity tests, then the config-4 bench with and without the light/heavy split.
mkdir -p gpurun_out/sssp
timeout -s KILL 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "sssp" > gpurun_out/sssp/pytest.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/sssp/pytest.log
for v in split nosplit; do
  if [ $v = nosplit ]; then export GBX_SSSP_NOSPLIT=1; else unset GBX_SSSP_NOSPLIT; fi
  timeout -s KILL 300 python bench.py --workload sssp --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/sssp/$v.json 2> gpurun_out/sssp/$v.err
  V=$v python -c 'import json,os; v=os.environ["V"]; d=json.load(open(f"gpurun_out/sssp/{v}.json")); print(v, round(d["ms_per_step"],2), "ms")' || tail -3 gpurun_out/sssp/$v.err
done
unset GBX_SSSP_NOSPLIT
PYTHONPATH=. GBX_SSSP_TLOG=1 timeout -s KILL 300 python tools/sssp_diag.py > gpurun_out/sssp/levels.txt 2>&1; echo diag rc=$?
