#!/bin/bash
# SSSP L2 residency A/B: persisting window on/off, evict-first edge loads
mkdir -p gpurun_out/sssp
run() {
  local v=$1; shift
  env "$@" timeout -s KILL 300 python bench.py --workload sssp --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/sssp/$v.json 2> gpurun_out/sssp/$v.err
  V=$v python -c 'import json,os; v=os.environ["V"]; d=json.load(open(f"gpurun_out/sssp/{v}.json")); print(v, round(d["ms_per_step"],2), "ms")' || tail -3 gpurun_out/sssp/$v.err
}
V=paper_2104_01661_b200/_variants
run base X=1
run nopersist GBX_SSSP_NOPERSIST=1
run ef GBX_LIB=$V/libgbx_ef.so
run ef_nopersist GBX_LIB=$V/libgbx_ef.so GBX_SSSP_NOPERSIST=1
PYTHONPATH=. GBX_SSSP_TLOG=1 timeout -s KILL 300 python tools/sssp_diag.py 2>&1 | grep 'max persist' | head -2
