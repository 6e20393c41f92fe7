#!/bin/bash
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_mrhs.py -x -q > gpurun_out/t.txt 2>&1; tail -2 gpurun_out/t.txt
