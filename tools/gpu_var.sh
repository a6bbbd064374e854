#!/bin/bash
# Variant sweep for one bench workload: tools/gpu_var.sh WORKLOAD name:lib:env ...
# (lib from paper_2104_01661_b200/_variants/, empty = libgbx.so)
W=$1; shift
mkdir -p gpurun_out/var
V=paper_2104_01661_b200/_variants
for spec in "$@"; do
  IFS=: read name lib envs <<< "$spec"
  if [ -n "$lib" ]; then L="GBX_LIB=$V/libgbx_$lib.so"; else L="X=1"; fi
  env $L $envs timeout -s KILL 300 python bench.py --workload $W --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/var/$W-$name.json 2> gpurun_out/var/$W-$name.err
  N=$W-$name python -c 'import json,os; v=os.environ["N"]; d=json.load(open(f"gpurun_out/var/{v}.json")); print(v, round(d["value"],3), d["unit"], round(d["ms_per_step"],4), "ms frac", round(d.get("roofline",{}).get("frac",0),4))' || tail -3 gpurun_out/var/$W-$name.err
done
