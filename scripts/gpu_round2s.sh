#!/bin/bash
set -u
mkdir -p gpurun_out
: > gpurun_out/ab_det.txt
for L in paper_1401_4780_b200/libasyrk_b200.so; do
  timeout 300 python scripts/ab_det.py $L >> gpurun_out/ab_det.txt 2>&1
  timeout 300 python scripts/ab_det.py $L reassoc >> gpurun_out/ab_det.txt 2>&1
done
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.txt 2>&1
tail -3 gpurun_out/gpu_tests.txt
