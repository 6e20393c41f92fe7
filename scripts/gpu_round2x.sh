#!/bin/bash
set -u
mkdir -p gpurun_out
KLS=64,32,8 timeout 600 python scripts/probe_cfg5.py > gpurun_out/probe_cfg5.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_mrhs.py tests/test_multirank.py -x -q > gpurun_out/t.txt 2>&1; tail -2 gpurun_out/t.txt
