make -s -C paper_2104_01661_b200/csrc -q && echo built_ok
timeout -s KILL 300 python -m pytest tests -m gpu -q -p no:cacheprovider -k "sssp" > gpurun_out/pytest_gpu.log 2>&1; echo rc=$?; tail -2 gpurun_out/pytest_gpu.log
timeout -s KILL 300 python bench.py --workload sssp --steps 3 --warmup 3 > gpurun_out/bench_sssp.json 2> gpurun_out/bench_sssp.err
python -c "import json; d=json.load(open('gpurun_out/bench_sssp.json')); print('sssp', round(d['value']/1e9,3), 'ms', round(d['ms_per_step'],3))" || tail -3 gpurun_out/bench_sssp.err
timeout -s KILL 120 python tools/prof_algo.py sssp 24 > gpurun_out/sssp_plain.log 2>&1 && timeout -s KILL 300 ncu --set full --clock-control none --import-source on -k regex:k_sssp -s 1 -c 1 -o gpurun_out/sssp_full5 python tools/prof_algo.py sssp 24 > gpurun_out/ncu_sssp.log 2>&1; tail -1 gpurun_out/ncu_sssp.log; cat gpurun_out/sssp_plain.log
