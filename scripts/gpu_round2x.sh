#!/bin/bash
set -u
mkdir -p gpurun_out
: > gpurun_out/csc.txt
for C in 0 1; do
  echo "== csc $C" >> gpurun_out/csc.txt
  ASYRK_MRHS_CSC_MONITOR=$C KLS=32,16,8 timeout 600 python scripts/probe_cfg5.py >> gpurun_out/csc.txt 2>&1
done
