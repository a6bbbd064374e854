#!/bin/bash
for lib in libgbx_u8_m5 libgbx_u4_m5 libgbx_u8_m4 libgbx_u16_m4; do
GBX_LIB=$PWD/paper_2104_01661_b200/$lib.so timeout -s KILL 200 python bench.py --workload bc --steps 6 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('$lib', round(d['ms_per_step'],3))"
done
