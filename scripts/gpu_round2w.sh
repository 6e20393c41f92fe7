#!/bin/bash
set -u
mkdir -p gpurun_out
python scripts/probe_solve_marks.py > gpurun_out/marks.txt 2>&1
python scripts/probe_solve_overhead.py > gpurun_out/overhead.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.txt 2>&1
tail -3 gpurun_out/gpu_tests.txt
