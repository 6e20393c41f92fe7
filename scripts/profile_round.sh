#!/bin/bash
# Round profiling recipe (run on a GPU box via gpurun from the repo root):
# plain bench, reference arm, x-side microbenchmark, ncu launch list, ncu --set full
# of the worker and monitor kernels. Outputs land in gpurun_out/.
set -u
mkdir -p gpurun_out
python bench.py --steps 30 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/ref.json 2> gpurun_out/ref.err
python scripts/probe_xside.py > gpurun_out/xside.txt 2>&1
CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1
echo "launch list rc=$?"
ncu --set full --clock-control none --import-source on -k regex:"worker_kernel|rows_kernel|cols_final_kernel" -s 200 -c 3 -o gpurun_out/full $CMD > gpurun_out/ncu_full.log 2>&1
echo "full rc=$?"
