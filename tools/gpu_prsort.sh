#!/bin/bash
timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py -q -x -k "pagerank or pr_" 2>&1 | tail -1
for v in 1 2; do
  PYTHONPATH=. GBX_PLAN_TIMING=1 timeout -s KILL 300 python tools/e2e_phases.py 2>&1 | tail -9
  timeout -s KILL 600 python bench.py --steps 60 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print(d['value'], d['ms_per_step'], d['e2e']['value'])"
done
