#!/bin/bash
set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.txt 2>&1
tail -3 gpurun_out/gpu_tests.txt
: > gpurun_out/ab_async.txt
for rep in 1 2; do
for L in paper_1401_4780_b200/libasyrk_b200.so scripts/r02a/libasyrk_b200.so; do
  ASYRK_LIB=$L timeout 300 python scripts/ab_async.py slice >> gpurun_out/ab_async.txt 2>&1
done
done
for L in paper_1401_4780_b200/libasyrk_b200.so scripts/r02a/libasyrk_b200.so; do
ASYRK_LIB=$L timeout 600 ncu --kernel-name regex:cols_final --launch-skip 10 --launch-count 3 --clock-control none \
  --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sectors_srcunit_tex_op_read.sum \
  python scripts/ab_async.py slice > gpurun_out/ncu_cols_$(basename $(dirname $L)).txt 2>&1
done
