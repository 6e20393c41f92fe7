"""Copy one profiling round (scripts/profile_round2.sh outputs) into profiles/
under a round tag: bench / reference lines, x-side and config-5 probes, ncu
launch-list summaries, ncu --set full metric summaries (worker + monitor,
x-side microbenchmark, config-5 kernels), and the worker's per-launch DRAM
traffic / L2 requests that bench.py reports (profiles/worker_ncu_summary.json).

  python scripts/save_profiles.py <tag> [source dir (default gpurun_out)]
"""
import csv
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag = sys.argv[1] if len(sys.argv) > 1 else "r02"
src = sys.argv[2] if len(sys.argv) > 2 else os.path.join(ROOT, "gpurun_out")
dst = os.path.join(ROOT, "profiles")

for name, out in [("bench.json", f"{tag}_bench.json"), ("ref.json", f"{tag}_ref.json"),
                  ("xside.txt", f"{tag}_xside.txt"), ("probe_cfg5.txt", f"{tag}_cfg5_probe.txt")]:
    p = os.path.join(src, name)
    if os.path.exists(p):
        shutil.copy(p, os.path.join(dst, out))


def summary(rep, header):
    txt = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "ncu_summary.py"), rep],
                         capture_output=True, text=True).stdout
    return header + txt


for name, cmd in [("launches.csv", "python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-cfg5"),
                  ("cfg5_launches.csv", "python scripts/cfg5_once.py")]:
    p = os.path.join(src, name)
    if os.path.exists(p):
        txt = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "launches.py"), p],
                             capture_output=True, text=True).stdout
        base = name.replace(".csv", "")
        open(os.path.join(dst, f"{tag}_{base}.txt"), "w").write(
            "# ncu --metrics gpu__time_duration.sum --clock-control none (cold, serialized launches)\n"
            f"# {cmd}\n" + txt)

for rep, out, hdr in [
        ("full.ncu-rep", "ncu_full", "# ncu --set full --clock-control none -k regex:worker_kernel|rows_kernel|cols_final_kernel"
                                     " (config 2 bench, 1 step)\n"),
        ("xside.ncu-rep", "ncu_xside", "# ncu --set full -k regex:xside_kernel: python scripts/probe_xside.py ncu "
                                       "(2 rows in flight, then 1; f64, n=100000, theta=30, 3552 warps, 256 proj/warp)\n"),
        ("mrhs.ncu-rep", "ncu_mrhs", "# ncu --set full -k regex:mrhs_worker|mrhs_rows|mrhs_cols: python scripts/cfg5_once.py "
                                     "(config 5, 64 columns on one GPU)\n"),
        ("mrhs8.ncu-rep", "ncu_mrhs8", "# ncu --set full -k regex:mrhs_worker|mrhs_rows|mrhs_gnorm: KL=8 python scripts/cfg5_once.py "
                                       "(config 5, an 8-column shard: the row-parallel worker and monitor)\n"),
        ("xside_mrhs8.ncu-rep", "ncu_xside_mrhs8", "# ncu --set full -k regex:xside_mrhs: KL=8 python "
                                                   "scripts/xside_mrhs_once.py (the 8-column x-side pattern, "
                                                   "row-parallel shape)\n"),
        ("det.ncu-rep", "ncu_det", "# ncu --set full -k regex:det_dataflow -s 2 -c 1: python scripts/ab_det.py "
                                   "(config 1, bitwise mode: one launch = one epoch, 20 000 row events)\n"),
        ("det_reassoc.ncu-rep", "ncu_det_reassoc", "# ncu --set full -k regex:det_dataflow -s 2 -c 1: python "
                                                   "scripts/ab_det.py reassoc (config 1, tolerance mode: one launch = one epoch)\n")]:
    p = os.path.join(src, rep)
    if os.path.exists(p):
        open(os.path.join(dst, f"{tag}_{out}.txt"), "w").write(summary(p, hdr))

rep = os.path.join(src, "full.ncu-rep")
if os.path.exists(rep):
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
            def num(k):
                x = float(v[h.index(k)].replace(",", ""))
                unit = rows[1][h.index(k)]
                return x * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
            d = {"kernel": v[h.index("Kernel Name")], "round": tag,
                 "source": f"profiles/{tag}_ncu_full.txt (ncu --set full, cold caches, 1 launch)",
                 "dram_bytes_per_launch": int(num("dram__bytes_read.sum") + num("dram__bytes_write.sum")),
                 "gpu_time_us": num("gpu__time_duration.sum"),
                 "lts_t_requests": num("lts__t_requests.sum"),
                 "lts_tag_requests_pct_avg": num("lts__t_tag_requests.avg.pct_of_peak_sustained_elapsed"),
                 "lts_tag_requests_pct_max": num("lts__t_tag_requests.max.pct_of_peak_sustained_elapsed"),
                 "lts_atomic_input_pct_avg": num("lts__d_atomic_input_cycles_active.avg.pct_of_peak_sustained_elapsed"),
                 "projections_per_launch": 200000,
                 "lts_requests_per_launch": reqs}
            json.dump(d, open(os.path.join(dst, "worker_ncu_summary.json"), "w"), indent=1)
            break
print("saved", tag)
