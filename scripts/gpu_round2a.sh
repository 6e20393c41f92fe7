#!/bin/bash
# round-2 call A: GPU tests, bench (cfg2 + cfg5 sub-line), x-side probe + its ncu capture
set -u
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/gputest.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/gputest.log
python bench.py --steps 20 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
tail -2 gpurun_out/bench.err
python scripts/probe_xside.py > gpurun_out/xside.txt 2>&1; echo "xside rc=$?"
python scripts/probe_xside.py ncu > gpurun_out/xside_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:xside_kernel -c 4 -o gpurun_out/xside \
    python scripts/probe_xside.py ncu > gpurun_out/ncu_xside.log 2>&1; echo "ncu xside rc=$?"
