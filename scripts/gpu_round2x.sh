#!/bin/bash
set -u
mkdir -p gpurun_out
python scripts/probe_solve_marks.py > gpurun_out/marks.txt 2>&1
python scripts/probe_solve_overhead.py > gpurun_out/overhead.txt 2>&1
: > gpurun_out/e2e_ab.txt
for L in scripts/r02c/libasyrk_b200.so paper_1401_4780_b200/libasyrk_b200.so; do
  echo "== $L" >> gpurun_out/e2e_ab.txt
  ASYRK_LIB=$L CALLS=12 timeout 300 python scripts/probe_e2e_phases.py 2>&1 | tail -9 | head -8 | awk '{print $3}' | tr '\n' ' ' >> gpurun_out/e2e_ab.txt
  echo >> gpurun_out/e2e_ab.txt
done
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.txt 2>&1; tail -2 gpurun_out/gpu_tests.txt
