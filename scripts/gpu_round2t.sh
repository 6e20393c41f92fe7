#!/bin/bash
set -u
mkdir -p gpurun_out
: > gpurun_out/ab_async.txt
for rep in 1 2; do
  timeout 300 python scripts/ab_async.py slice >> gpurun_out/ab_async.txt 2>&1
done
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_q.json 2> gpurun_out/bench_q.err; echo "bench rc=$?"
KLS=64,8 timeout 600 python scripts/probe_cfg5.py > gpurun_out/probe_cfg5.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.txt 2>&1; tail -2 gpurun_out/gpu_tests.txt
