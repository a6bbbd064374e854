make -s -C paper_2104_01661_b200/csrc -q && echo built_ok; timeout 900 python -m pytest tests -m gpu -q --timeout 300 -p no:cacheprovider -k "pagerank" > gpurun_out/pytest_gpu.log 2>&1; echo rc=$?; tail -2 gpurun_out/pytest_gpu.log
for hk in 0 48 96; do
  GBX_PR_HOT_KB=$hk timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_x.json 2> gpurun_out/bench_x.err
  python -c "import json; d=json.load(open('gpurun_out/bench_x.json')); print('hot',$hk,'value',round(d['value']/1e9,1),'ms',round(d['ms_per_step'],3),'frac',round(d['roofline']['frac'],3),'it',d['config']['iterations'])" || tail -3 gpurun_out/bench_x.err
done
export GBX_PR_NO_GRAPH=1 GBX_PR_HOT_KB=96; python tools/prof_pr.py 22 4 > gpurun_out/prof_plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_pr_rows -s 4 -c 1 -o gpurun_out/pr_full13 python tools/prof_pr.py 22 4 > gpurun_out/ncu2.log 2>&1; tail -1 gpurun_out/ncu2.log
