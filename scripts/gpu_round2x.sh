#!/bin/bash
set -u
mkdir -p gpurun_out
: > gpurun_out/long_ab.txt
for rep in 1 2; do
for L in scripts/r02c/libasyrk_b200.so paper_1401_4780_b200/libasyrk_b200.so; do
  echo "== $L" >> gpurun_out/long_ab.txt
  ASYRK_LIB=$L KLS=64 timeout 600 python scripts/probe_cfg5.py >> gpurun_out/long_ab.txt 2>&1
done
done
