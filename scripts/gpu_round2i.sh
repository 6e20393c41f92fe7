#!/bin/bash
set -u
mkdir -p gpurun_out
: > gpurun_out/probe_cfg5.txt
ASYRK_MRHS_ROWPAR=1 WARPS=1184,2368,4736 KLS=64,32,16,8 timeout 600 python scripts/probe_cfg5.py >> gpurun_out/probe_cfg5.txt 2>&1
echo "probe rc=$?"
# the bitwise deterministic path with the round-1 library (A/B: did config 1 slow down?)
timeout 300 python bench.py --workload cfg1 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/cfg1_new.json 2>&1
timeout 300 python scripts/ab_det.py scripts/r01lib/libasyrk_b200.so > gpurun_out/ab_det.txt 2>&1
timeout 300 python scripts/ab_det.py paper_1401_4780_b200/libasyrk_b200.so >> gpurun_out/ab_det.txt 2>&1
timeout 300 python scripts/ab_det.py paper_1401_4780_b200/libasyrk_b200.so reassoc >> gpurun_out/ab_det.txt 2>&1
ASYRK_DET_POLL_NS=0 timeout 300 python scripts/ab_det.py paper_1401_4780_b200/libasyrk_b200.so reassoc >> gpurun_out/ab_det.txt 2>&1
ASYRK_DET_POLL_NS=64 timeout 300 python scripts/ab_det.py paper_1401_4780_b200/libasyrk_b200.so reassoc >> gpurun_out/ab_det.txt 2>&1
echo done
