# A/B of the fused launches at configs 3, 3 (fp64 x) and 4
mkdir -p gpurun_out
for w in cfg3x cfg3 cfg4; do for f in 0 1; do
  ASYRK_NO_FUSE=$f timeout 300 python bench.py --workload $w --steps 5 --warmup 2 --no-cpu-baseline > gpurun_out/f3_${w}_$f.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/f3_${w}_$f.json').read().strip().splitlines()[-1]); print('$w no_fuse=$f', 'ms %.3f'%d['ms_per_step'], 'epochs', d.get('epochs'))"
done; done
