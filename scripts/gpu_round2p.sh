#!/bin/bash
set -u
mkdir -p gpurun_out
: > gpurun_out/e2e_stage.txt
for T in 4 8 12 16; do for C in 2048 4096 8192 16384; do
  echo "threads=$T chunk_kb=$C" >> gpurun_out/e2e_stage.txt
  ASYRK_STAGER_THREADS=$T ASYRK_STAGE_CHUNK_KB=$C CALLS=8 timeout 120 python scripts/probe_e2e_phases.py 2>&1 | grep "^call" | tail -4 >> gpurun_out/e2e_stage.txt
done; done
nproc >> gpurun_out/e2e_stage.txt
