#!/bin/bash
set -u
mkdir -p gpurun_out
: > gpurun_out/ab_det.txt
for L in paper_1401_4780_b200/libasyrk_b200.so scripts/alt_w24/libasyrk_b200.so scripts/alt_w16/libasyrk_b200.so scripts/alt_relax/libasyrk_b200.so; do
  timeout 300 python scripts/ab_det.py $L >> gpurun_out/ab_det.txt 2>&1
  timeout 300 python scripts/ab_det.py $L reassoc >> gpurun_out/ab_det.txt 2>&1
done
for P in 16 64; do ASYRK_DET_POLL_NS=$P timeout 300 python scripts/ab_det.py scripts/alt_relax/libasyrk_b200.so reassoc >> gpurun_out/ab_det.txt 2>&1; done
