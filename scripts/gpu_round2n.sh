#!/bin/bash
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q --timeout 600 -x > gpurun_out/gputest.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/gputest.log
timeout 600 python bench.py --steps 20 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
tail -2 gpurun_out/bench.err
: > gpurun_out/ab_det.txt
timeout 300 python scripts/ab_det.py paper_1401_4780_b200/libasyrk_b200.so >> gpurun_out/ab_det.txt 2>&1
timeout 300 python scripts/ab_det.py paper_1401_4780_b200/libasyrk_b200.so reassoc >> gpurun_out/ab_det.txt 2>&1
