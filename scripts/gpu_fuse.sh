# A/B: fused worker launches between scheduled evaluations (default) vs one launch per epoch
mkdir -p gpurun_out
for i in 1 2; do
  timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-cfg5 > gpurun_out/fuse_on_$i.json 2>gpurun_out/fuse_on.err; echo "on rc=$?"
  ASYRK_NO_FUSE=1 timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-cfg5 > gpurun_out/fuse_off_$i.json 2>gpurun_out/fuse_off.err; echo "off rc=$?"
done
python - <<'PY'
import json
for tag in ("on_1","off_1","on_2","off_2"):
    d=json.loads(open(f"gpurun_out/fuse_{tag}.json").read().strip().splitlines()[-1])
    print(tag, "ms/step %.3f"%d["ms_per_step"], "value %.3e"%d["value"], "launches/solve", d["worker_launches_per_solve"], "epochs", d["epochs"], "records", d["records_per_solve"], "frac %.3f"%d["roofline"]["frac"], "step_frac %.3f"%d["roofline"]["step_frac"], "e2e ms %.2f"%d["e2e"]["ms_per_step"], "instr ms %.3f"%d["instrumented"]["ms_per_solve"])
PY
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 > gpurun_out/gputest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/gputest.log
