#!/bin/bash
set -u
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity2.py tests/test_gpu_rowlen.py -q -x --timeout 600 > gpurun_out/gputest.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/gputest.log
timeout 600 python scripts/probe_cfg5.py > gpurun_out/probe_cfg5.txt 2>&1; echo "probe rc=$?"
ASYRK_MRHS_LOOPED=1 timeout 600 python scripts/probe_cfg5.py >> gpurun_out/probe_cfg5.txt 2>&1
python scripts/cfg5_once.py > gpurun_out/cfg5_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/cfg5_launches.csv python scripts/cfg5_once.py > gpurun_out/cfg5_ncu.log 2>&1; echo "ncu rc=$?"
