#!/bin/bash
set -u
mkdir -p gpurun_out
: > gpurun_out/ab_det.txt
for rep in 1 2; do
for L in scripts/r02c/libasyrk_b200.so paper_1401_4780_b200/libasyrk_b200.so; do
  timeout 120 python scripts/ab_det.py $L reassoc >> gpurun_out/ab_det.txt 2>&1
  timeout 120 python scripts/ab_det.py $L >> gpurun_out/ab_det.txt 2>&1
done
done
