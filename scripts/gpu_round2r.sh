#!/bin/bash
set -u
mkdir -p gpurun_out
: > gpurun_out/ab_det.txt
for L in scripts/r01lib/libasyrk_b200.so paper_1401_4780_b200/libasyrk_b200.so; do
  timeout 300 python scripts/ab_det.py $L >> gpurun_out/ab_det.txt 2>&1
done
timeout 300 python scripts/ab_det.py paper_1401_4780_b200/libasyrk_b200.so reassoc >> gpurun_out/ab_det.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity2.py tests/test_gpu_rowlen.py -q -x > gpurun_out/gputest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/gputest.log
