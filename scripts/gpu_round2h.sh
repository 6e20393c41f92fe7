#!/bin/bash
set -u
mkdir -p gpurun_out
KL=8 python scripts/cfg5_once.py > gpurun_out/cfg5n_plain.log 2>&1 && \
KL=8 ncu --set full --clock-control none --import-source on -k regex:"mrhs_worker" -s 10 -c 1 -o gpurun_out/mrhs8 python scripts/cfg5_once.py > gpurun_out/ncu_mrhs8.log 2>&1
echo "kl8 rc=$?"
KL=8 ASYRK_MRHS_ROWS=1 ncu --set full --clock-control none --import-source on -k regex:"mrhs_worker" -s 10 -c 1 -o gpurun_out/mrhs8L python scripts/cfg5_once.py > gpurun_out/ncu_mrhs8L.log 2>&1
echo "kl8 long rc=$?"
