for lib in libgbx libgbx_oldbfs; do for w in bfs64 bfs; do
GBX_LIB=$PWD/paper_2104_01661_b200/$lib.so timeout -s KILL 200 python bench.py --workload $w --steps 5 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('$lib $w', round(d['value'],2), 'ms', round(d['ms_per_step'],3))"
done; done
