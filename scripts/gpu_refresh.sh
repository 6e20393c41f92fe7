# refresh after the fusion rule: GPU tests, headline bench, configs 3 / 3x / 4 / 5 / shard projection
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q --timeout 600 > gpurun_out/gputest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/gputest.log
timeout 600 python bench.py --steps 20 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
for w in cfg3 cfg3x cfg4 cfg5 cfg5shards; do
  timeout 900 python bench.py --workload $w --steps 5 --warmup 3 > gpurun_out/$w.json 2> gpurun_out/$w.err; echo "$w rc=$?"
done
