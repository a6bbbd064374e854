mkdir -p gpurun_out
bash tools/gpu_all.sh
timeout -s KILL 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref_rc=$?; cat gpurun_out/bench_ref.json
