#!/bin/bash
set -u
mkdir -p gpurun_out
: > gpurun_out/ab_det.txt
L=paper_1401_4780_b200/libasyrk_b200.so
for P in 0 2 4 8 16 32; do
  echo "poll $P" >> gpurun_out/ab_det.txt
  ASYRK_DET_POLL_NS=$P timeout 300 python scripts/ab_det.py $L reassoc >> gpurun_out/ab_det.txt 2>&1
done
for P in 8 16 32 48; do
  echo "poll $P" >> gpurun_out/ab_det.txt
  ASYRK_DET_POLL_NS=$P timeout 300 python scripts/ab_det.py $L >> gpurun_out/ab_det.txt 2>&1
done
