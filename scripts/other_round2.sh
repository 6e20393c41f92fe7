#!/bin/bash
# the other BASELINE configs and the secondary workloads (one GPU), round 2
set -u
mkdir -p gpurun_out
for w in cfg1 cfg3 cfg3x cfg4 cfg5 cfg5shards sweep mc lsq; do
  timeout 900 python bench.py --workload $w --steps 5 --warmup 3 > gpurun_out/$w.json 2> gpurun_out/$w.err; echo "$w rc=$?"
  tail -c 300 gpurun_out/$w.json; echo
done
timeout 600 python bench.py --workload lsq --impl reference --steps 3 --warmup 1 > gpurun_out/lsq_ref.json 2>&1; echo "lsq ref rc=$?"
timeout 600 python bench.py --workload mc --impl reference --steps 3 --warmup 1 > gpurun_out/mc_ref.json 2>&1; echo "mc ref rc=$?"
