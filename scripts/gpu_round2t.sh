#!/bin/bash
set -u
mkdir -p gpurun_out
: > gpurun_out/ab_async.txt
for rep in 1 2; do
for L in paper_1401_4780_b200/libasyrk_b200.so scripts/alt_noaudit/libasyrk_b200.so scripts/alt_slice/libasyrk_b200.so; do
  ASYRK_LIB=$L timeout 300 python scripts/ab_async.py slice >> gpurun_out/ab_async.txt 2>&1
done
done
