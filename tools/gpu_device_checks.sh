#!/bin/bash
# compute-sanitizer is closed on this GPU pool; instead every GPU test and the
# sanitize fixtures run against a GBX_DEVICE_CHECKS build of the library
# (bounds of every column-derived gather index; a failed check traps):
#   bash tools/build_variant.sh checks "-DGBX_DEVICE_CHECKS" $(sed -n "s/^SRCS := //p" paper_2104_01661_b200/csrc/Makefile | sed "s/\.cu//g")
#   gpurun -- bash tools/gpu_device_checks.sh
mkdir -p gpurun_out
export GBX_LIB=paper_2104_01661_b200/_variants/libgbx_checks.so
timeout -s KILL 300 python tools/sanitize.py > gpurun_out/device_checks_fixtures.log 2>&1; echo fixtures_rc=$?; tail -2 gpurun_out/device_checks_fixtures.log
timeout -s KILL 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/device_checks_pytest.log 2>&1; echo pytest_rc=$?; tail -3 gpurun_out/device_checks_pytest.log
echo device_check_failures=$(cat gpurun_out/device_checks_*.log | grep -c "device check failed")
