make -s -C paper_2104_01661_b200/csrc -q && echo built_ok
timeout 900 python -m pytest tests -m gpu -q --timeout 300 -p no:cacheprovider -k "tc" > gpurun_out/pytest_gpu.log 2>&1; echo rc=$?; tail -2 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --workload tc --steps 3 --warmup 3 > gpurun_out/bench_tc.json 2> gpurun_out/bench_tc.err
python -c "import json; d=json.load(open('gpurun_out/bench_tc.json')); print('tc', round(d['value']/1e9,3), 'ms', round(d['ms_per_step'],3))" || tail -3 gpurun_out/bench_tc.err
python tools/prof_algo.py tc 22 > gpurun_out/tc_plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_tc_warp -s 1 -c 1 -o gpurun_out/tc_full4 python tools/prof_algo.py tc 22 > gpurun_out/ncu_tc.log 2>&1; tail -1 gpurun_out/ncu_tc.log
