for sc in 24 23 22; do
timeout -s KILL 300 python bench.py --workload sssp --scale $sc --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print($sc, d['value']/1e9, 'Grelax/s', d['ms_per_step'])"
done
