#!/bin/bash
# SSSP A/B: per-vertex {begin, light end, end} records vs row_ptr + nlight, light group sweep
mkdir -p gpurun_out/sssp
timeout -s KILL 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "sssp" > gpurun_out/sssp/pytest.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/sssp/pytest.log
run() {
  local v=$1; shift
  env "$@" timeout -s KILL 300 python bench.py --workload sssp --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/sssp/$v.json 2> gpurun_out/sssp/$v.err
  V=$v python -c 'import json,os; v=os.environ["V"]; d=json.load(open(f"gpurun_out/sssp/{v}.json")); print(v, round(d["ms_per_step"],2), "ms")' || tail -3 gpurun_out/sssp/$v.err
}
run novm GBX_SSSP_NOVM=1
run vm_lg2 X=1
run vm_lg1 GBX_SSSP_LG=1
run vm_lg4 GBX_SSSP_LG=4
PYTHONPATH=. GBX_SSSP_TLOG=1 timeout -s KILL 300 python tools/sssp_diag.py > gpurun_out/sssp/levels.txt 2>&1; echo diag rc=$?
