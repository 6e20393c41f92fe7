#!/bin/bash
# Round-2 profiling recipe (run on a GPU box via gpurun from the repo root):
# GPU tests, bench (cfg2 + cfg5 sub-line), reference arm, x-side + config-5
# probes, ncu launch list, ncu --set full of the worker / monitor kernels, the
# x-side microbenchmark and the config-5 worker. Outputs land in gpurun_out/.
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q --timeout 600 > gpurun_out/gputest.log 2>&1; echo "pytest rc=$?"
tail -4 gpurun_out/gputest.log
timeout 600 python bench.py --steps 20 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/ref.json 2> gpurun_out/ref.err; echo "ref rc=$?"
timeout 300 python scripts/probe_xside.py > gpurun_out/xside.txt 2>&1
timeout 300 python scripts/probe_cfg5.py > gpurun_out/probe_cfg5.txt 2>&1
KLS=32,16,8 timeout 300 python scripts/probe_cfg5.py >> gpurun_out/probe_cfg5.txt 2>&1
CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-cfg5"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1
echo "launch list rc=$?"
# one epoch per worker launch for the capture (ASYRK_NO_FUSE=1), so its DRAM bytes are per epoch
ASYRK_NO_FUSE=1 ncu --set full --clock-control none --import-source on -k regex:"worker_kernel|rows_kernel|cols_final_kernel" -s 200 -c 3 -o gpurun_out/full $CMD > gpurun_out/ncu_full.log 2>&1
echo "full rc=$?"
python scripts/probe_xside.py ncu > gpurun_out/xside_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:xside_kernel -c 4 -o gpurun_out/xside python scripts/probe_xside.py ncu > gpurun_out/ncu_xside.log 2>&1
echo "xside rc=$?"
python scripts/cfg5_once.py > gpurun_out/cfg5_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/cfg5_launches.csv python scripts/cfg5_once.py > gpurun_out/cfg5_ncu.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"mrhs_worker|mrhs_rows|mrhs_cols" -s 40 -c 3 -o gpurun_out/mrhs python scripts/cfg5_once.py > gpurun_out/ncu_mrhs.log 2>&1
echo "mrhs rc=$?"
# narrow shard (8 columns, the G = 8 width): the row-parallel worker and monitor, and the x-side
# microbenchmark in the worker's shape
KL=8 python scripts/cfg5_once.py > gpurun_out/cfg5_kl8.log 2>&1 && \
KL=8 ncu --set full --clock-control none --import-source on -k regex:"mrhs_worker|mrhs_rows|mrhs_gnorm" -s 30 -c 3 -o gpurun_out/mrhs8 python scripts/cfg5_once.py > gpurun_out/ncu_mrhs8.log 2>&1
echo "mrhs8 rc=$?"
KL=8 python scripts/xside_mrhs_once.py > gpurun_out/xs8.log 2>&1 && \
KL=8 ncu --set full --clock-control none -k regex:"xside_mrhs" -s 2 -c 1 -o gpurun_out/xside_mrhs8 python scripts/xside_mrhs_once.py > gpurun_out/ncu_xs8.log 2>&1
echo "xside8 rc=$?"
