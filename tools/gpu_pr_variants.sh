make -s -C paper_2104_01661_b200/csrc -q && echo built_ok
timeout 600 python -m pytest tests -m gpu -q --timeout 300 -p no:cacheprovider -k "pagerank" > gpurun_out/pytest_gpu.log 2>&1; echo rc=$?; tail -2 gpurun_out/pytest_gpu.log
for lib in libgbx libgbx_mb8; do
  GBX_LIB=$PWD/paper_2104_01661_b200/$lib.so timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_x.json 2> gpurun_out/bench_x.err
  python -c "import json; d=json.load(open('gpurun_out/bench_x.json')); print('$lib','value',round(d['value']/1e9,1),'ms',round(d['ms_per_step'],3),'frac',round(d['roofline']['frac'],3),'it',d['config']['iterations'])" || tail -3 gpurun_out/bench_x.err
done
