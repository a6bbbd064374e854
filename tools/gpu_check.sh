#!/bin/bash
# GPU check: every GPU test, smoke, then the default bench line exactly as the
# driver runs it (headline + secondary configs + CPU baselines).
# usage (under gpurun): bash tools/gpu_check.sh [pytest -k expr | bench]
mkdir -p gpurun_out
K=${1:+-k "$1"}
if [ "$1" != "bench" ]; then
  eval timeout -s KILL 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider $K > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?; tail -3 gpurun_out/pytest_gpu.log
  timeout -s KILL 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?; tail -1 gpurun_out/smoke.log
fi
T0=$SECONDS
timeout -s KILL 900 python bench.py > gpurun_out/bench_main.json 2> gpurun_out/bench_main.err; echo bench_rc=$? wall=$((SECONDS - T0))s; tail -1 gpurun_out/bench_main.err
python - <<'PY'
import json
d = json.loads(open("gpurun_out/bench_main.json").read())
print("value", d["value"], "ms", d["ms_per_step"], "rows_frac", d["roofline"]["frac"],
      "iter_frac", d["roofline"]["frac_per_iteration"], "e2e", d["e2e"]["value"], d["clocks"])
print("cpu", d.get("cpu_baseline", {}).get("value"), d.get("cpu_baseline_port", {}).get("value"))
for k, v in d.get("secondary", {}).items():
    print(k, v["value"], v["unit"], round(v["ms_per_step"], 3), round(v["roofline"]["frac"], 3),
          round(v["roofline"]["frac_actual"], 3), v["clocks"]["sm_mhz"], v["clocks"]["reasons"])
PY
