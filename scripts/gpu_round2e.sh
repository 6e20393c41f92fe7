#!/bin/bash
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q --timeout 600 > gpurun_out/gputest.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/gputest.log
: > gpurun_out/probe_cfg5.txt
WARPS=4736 KLS=64,32,16,8 timeout 300 python scripts/probe_cfg5.py >> gpurun_out/probe_cfg5.txt 2>&1
timeout 600 python bench.py --steps 20 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
tail -2 gpurun_out/bench.err
bash scripts/other_round2.sh
