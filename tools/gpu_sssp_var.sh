#!/bin/bash
# SSSP variant sweep: name:lib:env specs (lib from _variants/, empty = libgbx.so)
mkdir -p gpurun_out/sssp
timeout -s KILL 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "sssp" > gpurun_out/sssp/pytest.log 2>&1; echo pytest rc=$?; tail -1 gpurun_out/sssp/pytest.log
V=paper_2104_01661_b200/_variants
for spec in "$@"; do
  IFS=: read name lib envs <<< "$spec"
  if [ -n "$lib" ]; then L="GBX_LIB=$V/libgbx_$lib.so"; else L="X=1"; fi
  env $L $envs timeout -s KILL 300 python bench.py --workload sssp --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/sssp/$name.json 2> gpurun_out/sssp/$name.err
  N=$name python -c 'import json,os; v=os.environ["N"]; d=json.load(open(f"gpurun_out/sssp/{v}.json")); print(v, round(d["ms_per_step"],2), "ms", "frac", round(d.get("roofline",{}).get("frac",0),3))' || tail -3 gpurun_out/sssp/$name.err
done
