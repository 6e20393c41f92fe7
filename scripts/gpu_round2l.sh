#!/bin/bash
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_mrhs.py tests/test_gpu_parity2.py -q -x --timeout 600 > gpurun_out/gputest.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/gputest.log
: > gpurun_out/probe_cfg5.txt
KLS=64,32,16,8 timeout 600 python scripts/probe_cfg5.py >> gpurun_out/probe_cfg5.txt 2>&1
ASYRK_MRHS_CSC_MONITOR=1 KLS=64,8 timeout 600 python scripts/probe_cfg5.py >> gpurun_out/probe_cfg5.txt 2>&1
echo "probe rc=$?"
ASYRK_PROFILE_CREATE=1 timeout 300 python scripts/probe_e2e_phases.py > gpurun_out/e2e_phases.txt 2>&1
echo "e2e rc=$?"
