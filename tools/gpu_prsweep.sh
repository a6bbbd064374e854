#!/bin/bash
# PageRank A/B sweep: variant libraries x cache knobs, bench line per run.
mkdir -p gpurun_out/sweep
[ -n "$NOTEST" ] || timeout -s KILL 600 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "pagerank or pr_" > gpurun_out/sweep/pytest.log 2>&1; echo pytest rc=$?; tail -1 gpurun_out/sweep/pytest.log
run() {  # name, env...
  local name=$1; shift
  env "$@" timeout -s KILL 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/sweep/$name.json 2> gpurun_out/sweep/$name.err
  python - "$name" <<'PY'
import json,sys
n=sys.argv[1]
try:
    d=json.load(open(f"gpurun_out/sweep/{n}.json"))
    print(f"{n:28s} ms/step {d['ms_per_step']:.4f} it {d['config']['iterations']} us/iter {1e3*d['ms_per_step']/d['config']['iterations']:.1f} frac {d['roofline']['frac']:.3f} e2e {d['e2e']['value']:.3e}")
except Exception as e:
    print(n, "FAILED", e)
PY
}
V=paper_2104_01661_b200/_variants
for spec in "$@"; do
  IFS=: read name lib envs <<< "$spec"
  if [ -n "$lib" ]; then run $name GBX_LIB=$V/libgbx_$lib.so $envs; else run $name $envs; fi
done
