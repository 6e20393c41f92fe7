#!/bin/bash
set -u
mkdir -p gpurun_out
: > gpurun_out/e2e_ab.txt
for rep in 1 2 3; do
for L in scripts/r02b/libasyrk_b200.so paper_1401_4780_b200/libasyrk_b200.so; do
  echo "== $L" >> gpurun_out/e2e_ab.txt
  ASYRK_LIB=$L CALLS=12 timeout 300 python scripts/probe_e2e_phases.py 2>&1 | tail -9 | head -8 | awk '{print $3}' | tr '\n' ' ' >> gpurun_out/e2e_ab.txt
  echo >> gpurun_out/e2e_ab.txt
done
done
