# late round-2 final measurement (after the fused launches and the schedule placement):
# the round-2 profiling recipe, the other configs, randomized async stress
set -u
bash scripts/profile_round2.sh
bash scripts/other_round2.sh
timeout 600 python scripts/stress_async.py 1000 21 > gpurun_out/stress_async.txt 2>&1; tail -1 gpurun_out/stress_async.txt
