make -s -C paper_2104_01661_b200/csrc -q && echo built_ok
timeout 900 python -m pytest tests -m gpu -q --timeout 300 -p no:cacheprovider -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?; tail -3 gpurun_out/pytest_gpu.log
for w in bfs bfs64 tc sssp bc; do
  timeout 600 python bench.py --workload $w --steps 3 --warmup 3 > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err
  python -c "import json; d=json.load(open('gpurun_out/bench_$w.json')); print('$w', d['metric'], round(d['value'],3), d['unit'], 'ms', round(d['ms_per_step'],3))" || tail -3 gpurun_out/bench_$w.err
done
