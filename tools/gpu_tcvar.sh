#!/bin/bash
for lib in libgbx libgbx_l16_u4 libgbx_l32_u8 libgbx_l16_u8 libgbx_l24_u4; do
GBX_LIB=$PWD/paper_2104_01661_b200/$lib.so timeout -s KILL 200 python bench.py --workload tc --steps 5 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('$lib', round(d['ms_per_step'],3))"
done
