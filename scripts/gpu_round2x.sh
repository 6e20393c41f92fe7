#!/bin/bash
set -u
mkdir -p gpurun_out
g++ -O2 -std=c++20 -Iinclude scripts/cpp/csr_host_timing.cpp -Lpaper_1401_4780_b200 -lasyrk_b200 -Wl,-rpath,$PWD/paper_1401_4780_b200 -o /tmp/cht && /tmp/cht > gpurun_out/cht.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.txt 2>&1; tail -2 gpurun_out/gpu_tests.txt
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-cfg5 > gpurun_out/bench_q.json 2> gpurun_out/bench_q.err; echo "bench rc=$?"
