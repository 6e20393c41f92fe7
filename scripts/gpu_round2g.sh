#!/bin/bash
set -u
mkdir -p gpurun_out
: > gpurun_out/probe_cfg5.txt
WARPS=4736 KLS=64,32,16,8 timeout 300 python scripts/probe_cfg5.py >> gpurun_out/probe_cfg5.txt 2>&1
for B in 4 8; do
  ASYRK_MRHS_BATCH=$B WARPS=2368,3552 KLS=64,32,16,8 timeout 300 python scripts/probe_cfg5.py >> gpurun_out/probe_cfg5.txt 2>&1
done
timeout 600 python bench.py --workload cfg1 --steps 5 --warmup 3 > gpurun_out/cfg1.json 2> gpurun_out/cfg1.err; echo "cfg1 rc=$?"
