make -s -C paper_2104_01661_b200/csrc -q && echo built_ok
timeout -s KILL 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?; tail -3 gpurun_out/pytest_gpu.log
timeout -s KILL 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?; tail -1 gpurun_out/smoke.log
for w in bfs bfs64 tc sssp bc; do
  timeout -s KILL 300 python bench.py --workload $w --steps 3 --warmup 3 > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err
  python -c "import json; d=json.load(open('gpurun_out/bench_$w.json')); print('$w', d['metric'], round(d['value'],3), d['unit'], 'ms', round(d['ms_per_step'],3))" || tail -3 gpurun_out/bench_$w.err
done
timeout -s KILL 600 python bench.py > gpurun_out/bench_main.json 2> gpurun_out/bench_main.err; echo bench_rc=$?; cat gpurun_out/bench_main.json
