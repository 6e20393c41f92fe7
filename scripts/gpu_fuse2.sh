# A/B: fused multi-RHS worker launches (config 5 at one GPU, and the per-rank shard projection)
mkdir -p gpurun_out
timeout 300 python bench.py --workload cfg5 --steps 5 --warmup 2 > gpurun_out/c5_on.json 2>gpurun_out/c5_on.err; echo "c5 on rc=$?"
ASYRK_NO_FUSE=1 timeout 300 python bench.py --workload cfg5 --steps 5 --warmup 2 > gpurun_out/c5_off.json 2>gpurun_out/c5_off.err; echo "c5 off rc=$?"
timeout 600 python bench.py --workload cfg5shards --steps 5 --warmup 2 > gpurun_out/c5s_on.json 2>gpurun_out/c5s_on.err; echo "shards on rc=$?"
ASYRK_NO_FUSE=1 timeout 600 python bench.py --workload cfg5shards --steps 5 --warmup 2 > gpurun_out/c5s_off.json 2>gpurun_out/c5s_off.err; echo "shards off rc=$?"
for f in c5_on c5_off; do python -c "
import json,sys; d=json.loads(open('gpurun_out/$f.json').read().strip().splitlines()[-1]); print('$f', 'ms %.3f'%d['ms_per_step'], 'value %.3e'%d['value'], {k:d.get(k) for k in ('epochs','records_per_solve','worker_launches_per_solve')})"; done
tail -c 1500 gpurun_out/c5s_on.json; echo; tail -c 1500 gpurun_out/c5s_off.json; echo
timeout 900 python -m pytest tests/test_gpu_mrhs.py tests/test_gpu_parity.py tests/test_gpu_parity2.py -q -x --timeout 600 > gpurun_out/gputest2.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/gputest2.log
