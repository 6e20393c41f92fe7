# A/B (history): x gathers through L1 (an experiment build with -DASYRK_X_L1=1, not kept; results in
# profiles/r02_x_l1_ab.txt and DESIGN §10) vs L1-bypassing
mkdir -p gpurun_out
for i in 1 2; do
  timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-cfg5 > gpurun_out/l1_off_$i.json 2>/dev/null; echo "off rc=$?"
  ASYRK_LIB=$PWD/paper_1401_4780_b200/libasyrk_b200_l1.so timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-cfg5 > gpurun_out/l1_on_$i.json 2>gpurun_out/l1_on.err; echo "on rc=$?"
done
python - <<'PY'
import json
for tag in ("off_1","on_1","off_2","on_2"):
    d=json.loads(open(f"gpurun_out/l1_{tag}.json").read().strip().splitlines()[-1])
    r=d["roofline"]
    print(tag, "ms/step %.3f"%d["ms_per_step"], "value %.3e"%d["value"], "epochs", d["epochs"], "worker proj/s %.3e"%r["achieved_proj_per_s"], "R_x %.3e"%r["peak_proj_per_s"], "epoch ms %.4f"%r["avg_worker_epoch_ms"])
PY
for w in cfg4 cfg3; do
  timeout 300 python bench.py --workload $w --steps 5 --warmup 2 --no-cpu-baseline > gpurun_out/l1_${w}_off.json 2>/dev/null
  ASYRK_LIB=$PWD/paper_1401_4780_b200/libasyrk_b200_l1.so timeout 300 python bench.py --workload $w --steps 5 --warmup 2 --no-cpu-baseline > gpurun_out/l1_${w}_on.json 2>/dev/null
  for t in off on; do python -c "
import json; d=json.loads(open('gpurun_out/l1_${w}_$t.json').read().strip().splitlines()[-1]); print('$w $t', 'ms %.3f'%d['ms_per_step'], 'epochs', d.get('epochs'))"; done
done
