"""Copy one profiling round (scripts/profile_round.sh outputs in gpurun_out/)
into profiles/ under a round tag: bench / reference lines, x-side probe,
ncu launch-list summary, ncu --set full metric summary, and the worker's
per-launch DRAM traffic that bench.py reports as roofline.traffic."""
import csv
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
src = os.path.join(ROOT, "gpurun_out")
dst = os.path.join(ROOT, "profiles")
tag = sys.argv[1] if len(sys.argv) > 1 else "r01"

for name, out in [("bench.json", f"{tag}_bench.json"), ("ref.json", f"{tag}_ref.json"),
                  ("xside.txt", f"{tag}_xside.txt"), ("launches.csv", f"{tag}_launches.csv")]:
    p = os.path.join(src, name)
    if os.path.exists(p):
        shutil.copy(p, os.path.join(dst, out))

launches = os.path.join(src, "launches.csv")
if os.path.exists(launches):
    txt = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "launches.py"), launches],
                         capture_output=True, text=True).stdout
    open(os.path.join(dst, f"{tag}_launches.txt"), "w").write(
        "# ncu --metrics gpu__time_duration.sum --clock-control none (cold, serialized launches)\n"
        "# python bench.py --steps 1 --warmup 1 --no-cpu-baseline\n" + txt)

rep = os.path.join(src, "full.ncu-rep")
if os.path.exists(rep):
    txt = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "ncu_summary.py"), rep],
                         capture_output=True, text=True).stdout
    open(os.path.join(dst, f"{tag}_ncu_full.txt"), "w").write(
        "# ncu --set full --clock-control none --import-source on -k regex:worker_kernel|rows_kernel|cols_kernel|cols_final_kernel\n" + txt)
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    h = rows[0]
    reqs = {}
    for v in rows[2:]:  # L2 requests per launch of each captured kernel (first launch of each)
        name = v[h.index("Kernel Name")]
        key = "worker" if "worker_kernel" in name else "rows" if "rows_kernel" in name else \
            "cols" if "cols" in name else None
        if key and key not in reqs:
            reqs[key] = float(v[h.index("lts__t_requests.sum")].replace(",", ""))
    for v in rows[2:]:
        if "worker_kernel" in v[h.index("Kernel Name")]:
            num = lambda k: float(v[h.index(k)].replace(",", ""))  # noqa: E731
            unit = rows[1][h.index("dram__bytes_read.sum")]
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
            d = {"kernel": v[h.index("Kernel Name")], "round": tag,
                 "dram_bytes_per_launch": int((num("dram__bytes_read.sum") + num("dram__bytes_write.sum")) * scale),
                 "gpu_time_us": num("gpu__time_duration.sum"),
                 "lts_t_requests": num("lts__t_requests.sum"),
                 "lts_tag_requests_pct_avg": num("lts__t_tag_requests.avg.pct_of_peak_sustained_elapsed"),
                 "lts_tag_requests_pct_max": num("lts__t_tag_requests.max.pct_of_peak_sustained_elapsed"),
                 "projections_per_launch": 200000,
                 "lts_requests_per_launch": reqs}
            json.dump(d, open(os.path.join(dst, "worker_ncu_summary.json"), "w"), indent=1)
            break
print("saved", tag)
