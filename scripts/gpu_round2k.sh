#!/bin/bash
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_mrhs.py tests/test_gpu_parity2.py -q -x --timeout 600 > gpurun_out/gputest.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/gputest.log
: > gpurun_out/probe_cfg5.txt
KLS=64,32,16,8,4,2 timeout 600 python scripts/probe_cfg5.py >> gpurun_out/probe_cfg5.txt 2>&1
echo "probe rc=$?"
timeout 900 python bench.py --workload cfg5shards --steps 5 --warmup 3 > gpurun_out/cfg5shards.json 2> gpurun_out/cfg5shards.err; echo "shards rc=$?"
