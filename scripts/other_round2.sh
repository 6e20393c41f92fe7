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
# the deterministic kernel (config 1, bitwise then tolerance mode), one launch each under ncu
python scripts/ab_det.py paper_1401_4780_b200/libasyrk_b200.so > gpurun_out/det_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:det_dataflow -s 2 -c 1 -o gpurun_out/det \
  python scripts/ab_det.py paper_1401_4780_b200/libasyrk_b200.so > gpurun_out/ncu_det.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:det_dataflow -s 2 -c 1 -o gpurun_out/det_reassoc \
  python scripts/ab_det.py paper_1401_4780_b200/libasyrk_b200.so reassoc > gpurun_out/ncu_det_reassoc.log 2>&1
echo "det ncu rc=$?"
