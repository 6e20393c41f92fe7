#!/bin/bash
set -u
mkdir -p gpurun_out
: > gpurun_out/e2e_thr.txt
for rep in 1 2; do
for T in 8 12 16; do
  echo "== threads $T" >> gpurun_out/e2e_thr.txt
  ASYRK_STAGER_THREADS=$T CALLS=12 timeout 300 python scripts/probe_e2e_phases.py 2>&1 | tail -9 | head -8 | awk '{print $3}' | tr '\n' ' ' >> gpurun_out/e2e_thr.txt
  echo >> gpurun_out/e2e_thr.txt
done
done
