#!/bin/bash
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_mrhs.py tests/test_gpu_parity2.py tests/test_gpu_parity.py tests/test_gpu_rowlen.py -q -x --timeout 600 > gpurun_out/gputest.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/gputest.log
: > gpurun_out/probe_cfg5.txt
KLS=64,32,16,8 timeout 600 python scripts/probe_cfg5.py >> gpurun_out/probe_cfg5.txt 2>&1
echo "probe rc=$?"
: > gpurun_out/ab_det.txt
for L in scripts/r01lib/libasyrk_b200.so scripts/altdet/libasyrk_b200.so paper_1401_4780_b200/libasyrk_b200.so; do
  timeout 300 python scripts/ab_det.py $L >> gpurun_out/ab_det.txt 2>&1
done
timeout 300 python scripts/ab_det.py paper_1401_4780_b200/libasyrk_b200.so reassoc >> gpurun_out/ab_det.txt 2>&1
timeout 900 python bench.py --workload cfg5shards --steps 5 --warmup 3 > gpurun_out/cfg5shards.json 2> gpurun_out/cfg5shards.err; echo "shards rc=$?"
