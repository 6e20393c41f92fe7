#!/usr/bin/env python3
"""AsyRK hot-path benchmark (BASELINE.json metric on config 2).

Workload (N=1, BASELINE.json configs[1]): m=200000, n=100000, 30 nonzeros per
row at distinct uniform columns, N(0,1) values, rows normalized, fp64;
x* ~ N(0,1), b = A x*, x0 = 0; asynchronous lock-free warp-workers with
slice-shuffle row sampling (each worker reshuffles its slice of the rows every
epoch — the reference's default ParSampling, parallel.hpp:14-31, and the only
one its Python solve_parallel uses), gamma = 1, a residual snapshot every
epoch (snapshot_interval = 1, the reference default), stop at
||Ax-b|| / ||b|| < 1e-6. One "step" = one full solve to tolerance.

  value  projections/s of the whole job: row projections applied by all ranks
         / max-over-ranks device time (CUDA events on the solve stream), A and
         b resident in HBM, L2 flushed (256 MiB write) before every step.
  e2e    the same metric through the C ABI one-shot entry point
         asyrk_solve_parallel with HOST buffers: CSR upload + device packing,
         solve, trace + final_x download inside the timed region.
  --impl reference  the reference's own multithreaded CPU solve_parallel
         (oracle/_ref, the unmodified reference sources) on this host.

Multi-GPU (torchrun, N > 1): each rank solves an independent system of the
same shape (seed + rank) — replicas, no data-path collective ("scaling":
"weak"); timing is the max over ranks.
"""
import argparse
import gc
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Kaczmarz row projections/sec; time to ||Ax-b||/||b||<1e-6 vs CPU AsyRK"
CFG2 = dict(m=200000, n=100000, theta=30, seed=1002)
TOL = 1e-6
BYTES_PER_PROJ_F64 = 864  # S_A 384 + x gather 240 + atomic payload 240
S_A_F64 = 384             # A stream per projection: 16 B header + 30 x (8 B value + 4 B column), record-padded
X_BYTES_F64 = 480         # x side per projection: 30 gathered + 30 reduced doubles (L2-resident x)
L2_FLUSH_BYTES = 256 << 20


def workload_config():
    """The workload both arms run (identical dict on both lines; run-specific
    parameters such as warp / thread counts go to the sibling key "run")."""
    return {
        "workload": "config2: m=200000 n=100000 theta=30 N(0,1) unit rows fp64, x0=0, async to ||r||/||b||<1e-6",
        "sampling": "slice_shuffle (per-worker row slices reshuffled every epoch; the reference default)",
        "gamma": 1.0,
        "snapshot_interval": 1,
        "instance_seed": CFG2["seed"],
        "x0": "zeros",
        "l2": "GPU arm: 256 MiB L2 flush before every step (A, 75 MB of records, re-read from HBM each step)",
    }


def cpu_model():
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ["clocks.sm", "clocks.max.sm", "power.draw", "clocks_event_reasons.hw_slowdown",
              "clocks_event_reasons.hw_thermal_slowdown", "clocks_event_reasons.sw_thermal_slowdown",
              "clocks_event_reasons.sw_power_cap"]

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", "--query-gpu=" + ",".join(self.FIELDS),
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for ln in self.proc.stdout:
            self.lines.append(ln.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            p = [x.strip() for x in ln.split(",")]
            if len(p) < 7:
                continue
            try:
                sm.append(float(p[0]))
                mx.append(float(p[1]))
            except ValueError:
                continue
            for nm, v in zip(names, p[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


def measured_peak_hbm():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        return float(json.load(open(p))["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def ncu_summary():
    """Per-launch ncu counters of the worker (K2) from the committed capture
    (profiles/worker_ncu_summary.json, made by scripts/ncu_summary.py), or None."""
    p = os.path.join(ROOT, "profiles", "worker_ncu_summary.json")
    try:
        return json.load(open(p))
    except Exception:
        return None


def gen_system(seed):
    from paper_1401_4780_b200 import capi

    return capi.generate_fixed_theta(CFG2["m"], CFG2["n"], CFG2["theta"], seed=seed)


def gen_system_ref(seed, **kw):
    """The same instance for the reference arm, built by the C restatement of the
    generator (oracle/workload.c, pinned bit for bit to the product generator by
    tests/test_oracle.py) so the product library never maps into that process."""
    import oracle

    return oracle.C.generate_fixed_theta(CFG2["m"], CFG2["n"], CFG2["theta"], seed=seed, **kw)


# --------------------------------------------------------------------------- reference arm
def ref_solve_once(R, Ah, b, threads, target, epochs=10000, sampling="slice_shuffle"):
    x0 = np.zeros(Ah.n)
    t = R.solve_parallel(Ah, b, x0, threads=threads, gamma=1.0, epochs=epochs, target=target,
                         variant="full_row", sampling=sampling, seed=7, snapshot_interval=1, cap=epochs + 2)
    return int(t["updates_applied"][-1]), float(t["wall_seconds"][-1]), t


def load_ref():
    import oracle

    if oracle.REF is None:
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "ref"], check=False)
        import importlib

        importlib.reload(oracle)
    return oracle.REF


def ref_matrix(R, A):
    rows = np.repeat(np.arange(A.m, dtype=np.int64), np.diff(A.row_ptr))
    Ah, _ = R.build(A.m, A.n, rows, A.col_idx, A.values, normalize=True, b=None)
    return Ah


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    R = load_ref()
    if R is None:
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref not built and reference sources absent"}))
        return 0
    A, b, xs = gen_system_ref(CFG2["seed"])
    Ah = ref_matrix(R, A)
    target = TOL * TOL * float(b @ b)
    cores = host_cores()
    for _ in range(args.warmup):
        ref_solve_once(R, Ah, b, cores, target)
    proj, wall, ttt = 0, 0.0, []
    for _ in range(args.steps):
        p, w, t = ref_solve_once(R, Ah, b, cores, target)
        proj += p
        wall += w
        ttt.append(w)
    value = proj / wall
    cpu = {"value": value, "unit": "proj/s", "cores": cores, "kind": "reference", "cpu_model": cpu_model(),
           "sample": f"{args.steps} full config-2 solves to 1e-6 (reference solve_parallel, {cores} threads, "
                     "slice_shuffle, gamma=1, snapshot_interval=1)"}
    # the rest of SURVEY §8(d)'s CPU protocol, reported beside the line: T = 1
    # (a bounded 5-epoch sample) and with_replacement sampling at T = nproc
    p1, w1, _ = ref_solve_once(R, Ah, b, 1, 0.0, epochs=5)
    ps, ws, ts = ref_solve_once(R, Ah, b, cores, target, sampling="with_replacement")
    protocol = {"T1_slice_shuffle_proj_s": p1 / w1, "T1_sample": "5 epochs",
                f"T{cores}_with_replacement_proj_s": ps / ws,
                f"T{cores}_with_replacement_time_to_tolerance_ms": 1e3 * ws,
                f"T{cores}_with_replacement_epochs": int(ts["epoch_index"][-1])}
    line = {
        "metric": METRIC, "value": value, "unit": "proj/s", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * wall / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "impl": "reference",
        "config": workload_config(),
        "run": {"threads": cores, "cpu_model": cpu_model(), "cpu_protocol": protocol,
                "instance": "oracle/workload.c (C restatement of the product generator, bitwise-pinned)"},
        "time_to_tolerance_ms": 1e3 * statistics.median(ttt), "epochs": int(t["epoch_index"][-1]),
        "cpu_baseline": cpu, "e2e": {"value": value, "unit": "proj/s", "h2d_bytes_per_step": 0,
                                     "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))
    return 0


# --------------------------------------------------------------------------- GPU arm
def run_gpu(args):
    import torch

    from paper_1401_4780_b200 import capi

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    capi.check(capi.lib().asyrk_set_device(local))
    dist = None
    if world > 1:
        import torch.distributed as dist

        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    A, b, xs = gen_system(CFG2["seed"] + rank)
    bb = float(b @ b)
    target = TOL * TOL * bb
    stream = torch.cuda.Stream()
    S = capi.System(A, b, stream=stream.cuda_stream)
    # all resident warp slots
    W = args.warps or S.max_resident_warps()
    lam, lam_iters = S.power_iteration(1e-6)  # stats.cpp:15-50 on the device; tau bound beside the warp count
    flush = torch.empty(L2_FLUSH_BYTES, dtype=torch.uint8, device="cuda")
    solve_kw = dict(threads=W, gamma=1.0, epochs=2000, target=target, sampling=capi.SLICE_SHUFFLE,
                    snapshot_interval=1, want_x=False)

    for w in range(args.warmup):
        with torch.cuda.stream(stream):
            flush.zero_()
        S.solve(seed=100 + w, **solve_kw)

    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    stats = []
    epochs = []
    records = []
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        for k in range(args.steps):
            with torch.cuda.stream(stream):
                flush.zero_()
            ev[k][0].record(stream)
            r = S.solve(seed=1000 + k, **solve_kw)
            ev[k][1].record(stream)
            stats.append(S.stats())
            epochs.append(int(r["epoch_index"][-1]))
            records.append(len(r["epoch_index"]))
            rel = float(np.sqrt(r["r_sq"][-1] / bb))
            if not rel < TOL:
                raise RuntimeError(f"step {k} stopped at relative residual {rel} (epochs {epochs[-1]})")
        torch.cuda.synchronize()
    if dist:
        dist.barrier()
    step_ms = [a.elapsed_time(c) for a, c in ev]
    dev_ms = sum(step_ms)
    proj = sum(s["projections"] for s in stats)
    launches = sum(s["kernel_launches"] for s in stats)
    w_ms = sum(s["worker_ms"] for s in stats)
    w_launch = sum(s["worker_launches"] for s in stats)
    if dist:
        t = torch.tensor([dev_ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        tot = torch.tensor([float(proj)], device="cuda", dtype=torch.float64)
        dist.all_reduce(tot)
        dev_ms_max, proj_all = float(t.item()), float(tot.item())
    else:
        dev_ms_max, proj_all = dev_ms, float(proj)
    value = proj_all / (dev_ms_max * 1e-3)

    # ---- instrumented drop-in call (the reference's Python solve_parallel always
    # passes &rep, module.cpp:190-191): the same solve with the increment audit on
    instr_ms, instr_wms = [], []
    for k in range(-1, min(args.steps, 10)):
        with torch.cuda.stream(stream):
            flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        ri = S.solve(seed=3000 + k, instrument=True, **solve_kw)
        e1.record(stream)
        torch.cuda.synchronize()
        if k >= 0:
            instr_ms.append(e0.elapsed_time(e1))
            instr_wms.append(S.stats()["worker_ms"])
        if not ri["instrument"]["consistent"]:
            raise RuntimeError("instrumented solve failed the increment audit")

    # ---- the reference-facing Python call itself (pybind, module.cpp:297-303
    # signature: triplets in, rows normalized inside, always instrumented,
    # slice_shuffle): wall clock per call, host conversions included
    dropin = None
    if rank == 0:
        import paper_1401_4780_b200 as asyrk_mod

        rows_t = np.repeat(np.arange(A.m, dtype=np.int64), np.diff(A.row_ptr))
        calls = []
        for k in range(2):
            t0 = time.perf_counter()
            rd = asyrk_mod.solve_parallel(A.m, A.n, rows_t, A.col_idx, A.values, b, threads=W, gamma=1.0,
                                          epochs=2000, target=target, seed=4000 + k)
            calls.append(1e3 * (time.perf_counter() - t0))
        dropin = {"ms_per_call": statistics.median(calls), "calls_ms": [round(c, 2) for c in calls],
                  "epochs": int(rd["epoch_index"][-1]), "instrument_consistent": bool(rd["instrument"]["consistent"]),
                  "call": "paper_1401_4780_b200.solve_parallel(m, n, rows, cols, vals, b, threads=W, ...) — the "
                          "reference's Python signature (triplets -> CSR -> normalize_rows -> device solve with the "
                          "increment audit -> dict)"}

    # ---- e2e: one-shot C-ABI call with host buffers (one untimed warm-up call)
    e2e_steps = args.steps
    e2e_wall = 0.0
    e2e_proj = 0
    e2e_calls = []
    gc.collect()
    gc.disable()  # no interpreter collection pauses inside the timed host calls
    for k in range(-3, e2e_steps):  # 3 untimed warm-up calls
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = capi.solve_parallel_host(A, b, threads=W, gamma=1.0, epochs=2000, target=target,
                                     sampling=capi.SLICE_SHUFFLE, seed=2000 + k)
        dt = time.perf_counter() - t0
        if k >= 0:
            e2e_wall += dt
            e2e_proj += int(r["updates_applied"][-1])
            e2e_calls.append(round(1e3 * dt, 2))
    gc.enable()
    if dist:
        t = torch.tensor([e2e_wall], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_wall = float(t.item())
        tot = torch.tensor([float(e2e_proj)], device="cuda", dtype=torch.float64)
        dist.all_reduce(tot)
        e2e_proj = float(tot.item())
    # row_ptr (int64), col_idx (narrowed to int32 while staging), values (fp64), row_norm, b
    h2d = 8 * (A.m + 1) + 12 * A.nnz + 8 * A.m + 8 * A.m
    d2h = 8 * A.n + 48 * (max(epochs) + 2)  # final_x + trace records

    # ---- config 5 (the sharded configuration) at this N: k = 64 RHS split over the ranks
    c5 = None
    if not args.no_cfg5:
        try:  # a failure here must not cost the headline line
            c5 = cfg5_sharded(max(2, min(args.steps, 5)), 1, dist, rank, world, local, stream)
        except Exception as e:  # noqa: BLE001
            c5 = {"error": f"{type(e).__name__}: {e}"}
            print(f"[rank {rank}] cfg5_sharded failed: {c5['error']}", file=sys.stderr, flush=True)

    out = None
    if rank == 0:
        # worker time per epoch of work (launches span several epochs: the chunks
        # between two scheduled evaluations run as one launch)
        avg_launch_ms = w_ms / max(sum(epochs), 1)
        worker_rate = proj / (w_ms * 1e-3)  # credited projections / worker time: discarded epochs count as time
        out = {
            "metric": METRIC, "value": value, "unit": "proj/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": dev_ms_max / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": workload_config(),
            "run": {"warps": W, "resident_warps": stats[0]["resident_warps"], "lambda_max": lam,
                    "tau_max": CFG2["m"] / (2 * np.e * lam) - 1, "rows_in_flight": 2 * W,
                    "parallelism": f"replicas x{world} (config 2 is one system: x is not sharded)"},
            "time_to_tolerance_ms": statistics.median(step_ms), "epochs": statistics.median(epochs),
            "records_per_solve": statistics.median(records),
            "worker_launches_per_solve": w_launch / args.steps,
            "library_solve_ms_per_step": sum(s["solve_ms"] for s in stats) / args.steps,
            "e2e": {"value": e2e_proj / e2e_wall, "unit": "proj/s", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h, "ms_per_step": 1e3 * e2e_wall / e2e_steps, "calls_ms": e2e_calls},
            "instrumented": {"ms_per_solve": statistics.median(instr_ms),
                             "worker_ms_per_solve": statistics.median(instr_wms),
                             "uninstrumented_worker_ms_per_solve": w_ms / args.steps,
                             "ratio_vs_uninstrumented": statistics.median(instr_ms) / statistics.median(step_ms),
                             "call": "System.solve(..., instrument=True): the increment audit of "
                                     "solve_parallel's InstrumentReport (parallel.cpp:94-106)"},
            "gpu_launches": launches,
            "dropin_python_call": dropin,
            "roofline": roofline(S, W, worker_rate, avg_launch_ms, value),
            "clocks": clk.summary(),
        }
        if c5 is not None:
            out["cfg5_sharded"] = c5
        if world == 1 and not args.no_cpu_baseline:
            out["cpu_baseline"] = cpu_baseline(A, b)
    if dist:
        dist.barrier()
        dist.destroy_process_group()
    S.close()
    if out is not None:
        print(json.dumps(out))
    return 0


def roofline(S, W, worker_rate, avg_launch_ms, step_rate):
    """The binding ceiling of K2: R_proj = min(BW_HBM / S_A, R_x),
    R_x = the x-side traffic of a projection alone (30 random L2 gathers ->
    warp reduce -> 30 random red.add.f64), measured live at the worker's warp
    count and x footprint, with 1 and 2 rows in flight per warp. Expressed in
    GB/s of x-side L2 traffic (480 B per projection) so the unit matches the
    contract; the proj/s figures sit beside it."""
    from paper_1401_4780_b200 import capi

    # on the solver's own x buffer (same address / pages, L2-resident) at the worker's warp count
    rx1 = max(S.microbench_xside(W, 1024, 0) for _ in range(3))
    rx2 = max(S.microbench_xside(W, 1024, 16) for _ in range(3))
    rx = max(rx1, rx2)
    rx_alloc = max(capi.microbench_xside(CFG2["n"], CFG2["theta"], capi.F64, W, 1024, 16) for _ in range(3))
    peak_hbm, hbm_kind = measured_peak_hbm()
    r_hbm = peak_hbm * 1e9 / S_A_F64
    r_proj = min(r_hbm, rx)
    ncu = ncu_summary()
    dram = ncu.get("dram_bytes_per_launch") if ncu else None
    out = {"bound": "l2_atomic", "unit": "GB/s",
           "achieved": worker_rate * X_BYTES_F64 / 1e9, "peak": r_proj * X_BYTES_F64 / 1e9,
           "frac": worker_rate / r_proj, "traffic": dram,
           "kernel": "K2 worker_kernel (csrc/worker.cu)",
           "achieved_proj_per_s": worker_rate, "peak_proj_per_s": r_proj,
           "R_x_proj_per_s": {"rows_in_flight_1": rx1, "rows_in_flight_2": rx2,
                              "fresh_buffer_rows_in_flight_2": rx_alloc},
           "R_hbm_proj_per_s": r_hbm,
           "step_frac": step_rate / r_proj,
           "peak_source": "x-side microbenchmark measured live in this run on the solver's own x buffer "
                          "(asyrk_system_microbench_xside), the faster of 1 and 2 rows in flight per warp; ncu "
                          "counters of it in profiles/",
           "achieved_source": "credited projections / worker time in the timed steps: CUDA-event pairs around "
                              "each multi-epoch worker launch (K2: the epochs between two scheduled evaluations "
                              "run as one launch) and a sample of the one-epoch ones; their ms per epoch times "
                              "all epochs of work",
           "avg_worker_epoch_ms": avg_launch_ms,
           "x_bytes_per_proj": X_BYTES_F64, "alg_bytes_per_proj": BYTES_PER_PROJ_F64}
    # the A stream against HBM: algorithmic 384 B/projection vs ncu DRAM bytes
    alg_launch = S_A_F64 * CFG2["m"]
    out["hbm"] = {"achieved": alg_launch / (avg_launch_ms * 1e-3) / 1e9, "peak": peak_hbm, "unit": "GB/s",
                  "frac": alg_launch / (avg_launch_ms * 1e-3) / 1e9 / peak_hbm, "peak_source": hbm_kind,
                  "alg_bytes_per_epoch": alg_launch, "dram_bytes_per_epoch": dram,
                  "dram_source": "ncu --set full of one-epoch worker launches (ASYRK_NO_FUSE=1: same kernel, one "
                                 "epoch per launch)",
                  "traffic_over_alg": (dram / alg_launch) if dram else None,
                  "source": ncu.get("source") if ncu else None}
    return out


def cpu_baseline(A, b):
    R = load_ref()
    if R is None:
        return None
    Ah = ref_matrix(R, A)
    cores = host_cores()
    target = TOL * TOL * float(b @ b)
    p, w, t = ref_solve_once(R, Ah, b, cores, target)
    return {"value": p / w, "unit": "proj/s", "cores": cores, "kind": "reference", "cpu_model": cpu_model(),
            "sample": f"1 full config-2 solve to 1e-6 ({int(t['epoch_index'][-1])} epochs, {w:.2f} s) with the "
                      f"reference solve_parallel, {cores} threads, slice_shuffle",
            "time_to_tolerance_ms": 1e3 * w}


CFG5 = dict(m=500000, n=250000, theta=20, k=64, seed=1005)
TOL5 = 1e-5


def cfg5_sharded(steps, warmup, dist, rank, world, local, stream, W=0):
    """BASELINE config 5 at this job's N: k=64 right-hand sides split into N
    contiguous column shards, one per rank (A replicated), each rank's
    lock-free warp-workers on its shard, and one NCCL all-reduce of the shard
    residual norms per evaluated boundary as the global stop test. The loop is
    the library's native driver (asyrk_mrhs_solve_nccl): the NCCL communicator
    is built by the library from a unique id broadcast over torch.distributed
    (a 1-rank communicator at N = 1). Returns the summary on rank 0."""
    import torch

    from paper_1401_4780_b200 import capi
    from paper_1401_4780_b200.mrhs import shard_columns

    A, B, Xs = capi.generate_fixed_theta(CFG5["m"], CFG5["n"], CFG5["theta"], seed=CFG5["seed"], k=CFG5["k"])
    B = B.astype(np.float32)
    bb = float((B.astype(np.float64) ** 2).sum())
    c0, c1 = shard_columns(CFG5["k"], world, rank)
    flush = torch.empty(L2_FLUSH_BYTES, dtype=torch.uint8, device="cuda")
    if dist:
        uid = capi.nccl_unique_id() if rank == 0 else bytes(capi.NCCL_UNIQUE_ID_BYTES)
        t = torch.tensor(list(uid), dtype=torch.uint8, device="cuda")
        dist.broadcast(t, src=0)
        uid = bytes(t.cpu().tolist())
    else:
        uid = capi.nccl_unique_id()
    comm = capi.NcclComm(world, uid, rank)
    sh = capi.MultiRHS(A, B, c0, c1, stream=stream.cuda_stream)
    W = W or sh.max_resident_warps()  # every co-resident worker warp (4736 at 64 columns on 148 SMs)
    kw = dict(threads=W, gamma=1.0, epochs=2000, target=TOL5 * TOL5 * bb, snapshot_interval=1,
              sampling=capi.SLICE_SHUFFLE)
    for w in range(warmup):
        with torch.cuda.stream(stream):
            flush.zero_()
        sh.solve_nccl(comm, seed=100 + w, want_x=False, **kw)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    rows, epochs, records, wms, wl, lib_ms = 0, [], [], 0.0, 0, 0.0
    with ClockSampler(local) as clk:
        for k in range(steps):
            with torch.cuda.stream(stream):
                flush.zero_()
            ev[k][0].record(stream)
            t = sh.solve_nccl(comm, seed=1000 + k, want_x=False, **kw)
            ev[k][1].record(stream)
            st = sh.stats()
            wms += st["worker_ms"]
            lib_ms += st["solve_ms"]
            wl += st["worker_launches"]
            rows += int(t["updates_applied"][-1])
            epochs.append(int(t["epoch_index"][-1]))
            records.append(len(t["epoch_index"]))
            rel = float(np.sqrt(t["r_sq"][-1] / bb))
            if not rel < TOL5:
                raise RuntimeError(f"config 5 step {k} stopped at relative residual {rel}")
        torch.cuda.synchronize()
    # the stop test's collective alone: an all-reduce of 3 doubles over the job's
    # NCCL fabric (torch's communicator), device time per call
    ar_us = 0.0
    if dist:
        nt = torch.zeros(3, dtype=torch.float64, device="cuda")
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        for _ in range(10):
            dist.all_reduce(nt)
        e0.record()
        for _ in range(200):
            dist.all_reduce(nt)
        e1.record()
        torch.cuda.synchronize()
        ar_us = 1e3 * e0.elapsed_time(e1) / 200
        dist.barrier()
    step_ms = [a.elapsed_time(c) for a, c in ev]
    dev_ms = sum(step_ms)
    col_proj = rows * (c1 - c0)  # one row event projects every owned RHS column
    if dist:
        t = torch.tensor([dev_ms, ar_us], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dev_ms, ar_us = float(t[0].item()), float(t[1].item())
        t = torch.tensor([float(col_proj)], device="cuda", dtype=torch.float64)
        dist.all_reduce(t)
        col_proj = float(t.item())
    # the multi-RHS x-side ceiling at this shard's width and warp count (no A / B stream), on the
    # shard's own X (a fresh buffer measures lower, as config 2's R_x does)
    kl = c1 - c0
    warps = W // (128 // kl) if kl in (8, 16, 32) else W  # the row-parallel worker runs 128/kl workers per warp
    rx5 = max(sh.microbench_xside(warps, 64) for _ in range(2))
    rx5_fresh = capi.microbench_xside_mrhs(CFG5["n"], CFG5["theta"], kl, warps, 64)
    sh.close()
    comm.close()
    if rank != 0:
        return None
    worker_rate = rows / (wms * 1e-3) if wms > 0 else 0.0  # row projections per worker second (this rank)
    return {"metric": "config 5 column projections/sec (row projections x owned RHS columns, all ranks)",
            "value": col_proj / (dev_ms * 1e-3), "unit": "proj/s", "n_gpus": world, "steps": steps,
            "ms_per_step": dev_ms / steps, "time_to_tolerance_ms": statistics.median(step_ms),
            "epochs": statistics.median(epochs), "records_per_solve": statistics.median(records),
            "worker_ms_per_solve": wms / steps, "worker_launches_per_solve": wl / steps,
            "library_solve_ms_per_step": lib_ms / steps,
            "roofline": {"bound": "l2_x_side", "unit": "row proj/s", "achieved": worker_rate, "peak": rx5,
                         "frac": worker_rate / rx5 if rx5 else None,
                         "peak_fresh_buffer": rx5_fresh,
                         "source": "achieved = rank 0's row projections / its worker-launch time; peak = "
                                   "asyrk_mrhs_microbench_xside (the K2b worker's X gathers and v4 reds, no A/B "
                                   "stream) on the shard's own X at the same width and warps, measured live",
                         "note": "the microbenchmark is the worker's X pattern stripped of the A / B streams, not a "
                                 "hardware roof: frac ~1.0 (up to 1.05 at 64 columns, where the worker interleaves "
                                 "its gathers and reds more evenly than the stripped loop) says the worker runs at "
                                 "the rate of its own X traffic; the saturated unit is the L1TEX pipeline "
                                 "(ncu: 73% at 64 columns, 90% at 8; profiles/r02_ncu_mrhs*.txt)",
                         "x_bytes_per_row_proj": 2 * CFG5["theta"] * (c1 - c0) * 4},
            "allreduce_us_per_call": ar_us, "scaling": "strong", "columns_per_gpu": c1 - c0,
            "driver": "asyrk_mrhs_solve_nccl (native loop, NCCL all-reduce of the shard norms per evaluated boundary)",
            "sampling": "slice_shuffle",
            "workload": "config5: m=500000 n=250000 theta=20 k=64 fp32, RHS columns sharded over the ranks, "
                        "all-reduced stop at ||R||_F/||B||_F<1e-5",
            "warps": W, "clocks": clk.summary()}


def run_gpu_cfg5(args):
    """BASELINE config 5 as its own line (bench.py --workload cfg5)."""
    import torch

    from paper_1401_4780_b200 import capi

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    capi.check(capi.lib().asyrk_set_device(local))
    dist = None
    if world > 1:
        import torch.distributed as dist

        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    stream = torch.cuda.Stream()
    c5 = cfg5_sharded(args.steps, args.warmup, dist, rank, world, local, stream, W=args.warps)
    if rank == 0:
        line = {"metric": METRIC + " (config 5: column projections/sec)", "value": c5["value"], "unit": "proj/s",
                "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": c5["ms_per_step"],
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
                "data": "synthetic", "config": {"workload": c5["workload"]},
                "run": {"warps": c5["warps"], "columns_per_gpu": c5["columns_per_gpu"],
                        "parallelism": f"rhs-shard x{world}"},
                "time_to_tolerance_ms": c5["time_to_tolerance_ms"], "epochs": c5["epochs"],
                "records_per_solve": c5["records_per_solve"], "allreduce_us_per_call": c5["allreduce_us_per_call"],
                "driver": c5["driver"], "clocks": c5["clocks"]}
        if world == 1 and not args.no_cpu_baseline:
            import oracle  # noqa: F401  (the reference's CPU path on a bounded sample)

            R = load_ref()
            if R is not None:  # the reference solves one RHS at a time: 1 epoch of column 0 on all host threads
                A, B, _ = oracle.C.generate_fixed_theta(CFG5["m"], CFG5["n"], CFG5["theta"], seed=CFG5["seed"],
                                                        k=CFG5["k"])
                Ah = ref_matrix(R, A)
                cores = host_cores()
                bn = B[:, 0].astype(np.float32).astype(np.float64)
                t = R.solve_parallel(Ah, bn, np.zeros(A.n), threads=cores, gamma=1.0, epochs=1, target=0.0,
                                     variant="full_row", sampling="with_replacement", seed=7, snapshot_interval=1,
                                     cap=4)
                line["cpu_baseline"] = {
                    "value": int(t["updates_applied"][-1]) / float(t["wall_seconds"][-1]), "unit": "proj/s",
                    "cores": cores, "kind": "reference", "cpu_model": cpu_model(),
                    "sample": "1 epoch of solve_parallel (fp64) on RHS column 0; the reference solves the 64 "
                              "columns one after another"}
        print(json.dumps(line))
    if dist:
        dist.destroy_process_group()
    return 0


# ---- the other BASELINE configs (BASELINE.json configs[0], [2], [3]) and the warp sweep
OTHER = {
    "cfg1": dict(m=20000, n=10000, theta=20, seed=1001, dist="normal", scale=0.0, tol=1e-8, epochs=20,
                 desc="config1: m=20000 n=10000 theta=20 N(0,1) unit rows fp64, deterministic 1 worker, uniform "
                      "seeded sequence, until ||r||/||b||<1e-8 or 20 epochs"),
    "cfg3": dict(m=2000000, n=1000000, theta=50, seed=1003, dist="uniform", scale=0.0, tol=1e-5, epochs=400,
                 desc="config3: m=2000000 n=1000000 theta=50 U(-1,1) unit rows, fp32 values + fp32 x/atomics, "
                      "async to ||r||/||b||<1e-5"),
    "cfg3x": dict(m=2000000, n=1000000, theta=50, seed=1003, dist="uniform", scale=0.0, tol=1e-5, epochs=400,
                  desc="config3 (fp64-x variant): fp32 values, fp64 x/atomics, async to ||r||/||b||<1e-5"),
    "cfg4": dict(m=400000, n=100000, theta=25, seed=1004, dist="normal", scale=1.0, tol=1e-6, epochs=1000,
                 desc="config4: m=400000 n=100000 theta=25 N(0,1) rows scaled log-uniform [0.1,10] fp64, "
                      "alias sampling P(i)=||a_i||^2/||A||_F^2, async to ||r||/||b||<1e-6"),
}


def run_other(args):
    """Throughput and time-to-tolerance of BASELINE configs 1, 3 (+fp64-x), 4 on one GPU
    (device time, CUDA events), with the reference's CPU path on a bounded sample
    beside it (rank 0 only; replicas are not run for these)."""
    import torch

    from paper_1401_4780_b200 import capi

    if int(os.environ.get("RANK", "0")) != 0:
        return 0
    c = OTHER[args.workload]
    A, b, xs = capi.generate_fixed_theta(c["m"], c["n"], c["theta"], seed=c["seed"], dist=c["dist"],
                                         scale_decades=c["scale"])
    bb = float(b @ b)
    target = c["tol"] ** 2 * bb
    prec = {"cfg3": capi.F32, "cfg3x": capi.F32X64}.get(args.workload, capi.F64)
    S = capi.System(A, b, precision=prec)
    det = args.workload == "cfg1"
    W = 1 if det else (args.warps or S.max_resident_warps())
    if det:
        run = lambda k: S.rk_solve(max_epochs=c["epochs"], target=target, seed=42 + k,  # noqa: E731
                                   sampling=capi.RK_UNIFORM, x_star=xs)
    else:
        samp = capi.NORM_PROPORTIONAL if args.workload == "cfg4" else capi.SLICE_SHUFFLE
        run = lambda k: S.solve(threads=W, gamma=1.0, epochs=c["epochs"], target=target, sampling=samp,  # noqa: E731
                                seed=100 + k, snapshot_interval=1, x_star=xs, want_x=False, precision=prec)
    for k in range(args.warmup):
        run(k)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    torch.cuda.synchronize()
    proj, ttt, rels, errs, epochs = 0, [], [], [], []
    with ClockSampler(0) as clk:
        for k in range(args.steps):
            ev[k][0].record()
            t = run(1000 + k)
            ev[k][1].record()
            torch.cuda.synchronize()
            ttt.append(ev[k][0].elapsed_time(ev[k][1]))
            proj += int(t["updates_applied"][-1])
            epochs.append(int(t["epoch_index"][-1]))
            rels.append(float(np.sqrt(t["r_sq"][-1] / bb)))
            errs.append(float(np.sqrt(t["dist_sq"][-1] / float(xs @ xs))))
    dev_ms = sum(ttt)
    line = {"metric": METRIC + f" ({args.workload})", "value": proj / (dev_ms * 1e-3), "unit": "proj/s", "n_gpus": 1,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": dev_ms / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": {"cfg3": "f32", "cfg3x": "f32 values, f64 x"}.get(args.workload, "f64"), "data": "synthetic",
            "config": {"workload": c["desc"], "warps": W, "l2": "A resident (no flush between steps)"},
            "time_to_tolerance_ms": statistics.median(ttt), "epochs": statistics.median(epochs),
            "final_rel_residual": max(rels), "final_rel_error": max(errs), "tolerance": c["tol"],
            "gpu_launches": S.stats()["kernel_launches"] * args.steps, "clocks": clk.summary()}
    if det:
        line["parity"] = "final_x bit-identical to the reference rk_solve" if ref_cfg1_parity(A, b, c, xs, S) \
            else "MISMATCH against the reference rk_solve"
        # the tolerance mode (run config det_reassociate): same sequence, warp-tree dot
        fast_ms, fast_t = [], None
        for k in range(args.warmup + args.steps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fast_t = S.rk_solve(max_epochs=c["epochs"], target=target, seed=1000 + k, sampling=capi.RK_UNIFORM,
                                reassociate=True)
            e1.record()
            torch.cuda.synchronize()
            if k >= args.warmup:
                fast_ms.append(e0.elapsed_time(e1))
        exact_same = S.rk_solve(max_epochs=c["epochs"], target=target, seed=1000 + args.warmup + args.steps - 1,
                                sampling=capi.RK_UNIFORM)
        drift = float(np.linalg.norm(fast_t["final_x"] - exact_same["final_x"]) /
                      np.linalg.norm(exact_same["final_x"]))
        line["reassociated"] = {"time_to_tolerance_ms": statistics.median(fast_ms),
                                "value": int(fast_t["updates_applied"][-1]) / (statistics.median(fast_ms) * 1e-3),
                                "rel_diff_vs_bitwise_final_x": drift,
                                "mode": "det_reassociate=1: warp-tree dot, reciprocal coefficient, fused update"}
    if not args.no_cpu_baseline:
        line["cpu_baseline"] = other_cpu_baseline(args.workload, c, A, b)
    S.close()
    print(json.dumps(line))
    return 0


def ref_cfg1_parity(A, b, c, xs, S):
    from paper_1401_4780_b200 import capi

    R = load_ref()
    if R is None:
        return False
    Ah = ref_matrix(R, A)
    t = R.rk_solve(Ah, b, np.zeros(A.n), c["epochs"], c["tol"] ** 2 * float(b @ b), 42, "uniform", xs)
    mine = S.rk_solve(max_epochs=c["epochs"], target=c["tol"] ** 2 * float(b @ b), seed=42, sampling=capi.RK_UNIFORM,
                      x_star=xs)
    return bool(np.array_equal(t["final_x"], mine["final_x"]) and np.array_equal(t["r_sq"], mine["r_sq"]))


def other_cpu_baseline(name, c, A, b):
    """The reference's own CPU path on a bounded sample of the same workload."""
    R = load_ref()
    if R is None:
        return None
    Ah = ref_matrix(R, A)
    cores = host_cores()
    x0 = np.zeros(A.n)
    if name == "cfg1":  # serial rk_solve, the full run (20 epochs), median of 3 runs
        runs = [R.rk_solve(Ah, b, x0, c["epochs"], c["tol"] ** 2 * float(b @ b), 42, "uniform") for _ in range(3)]
        t = sorted(runs, key=lambda r: float(r["wall_seconds"][-1]))[1]
        p, w, cores, sample = int(t["updates_applied"][-1]), float(t["wall_seconds"][-1]), 1, \
            "the full config-1 run, median of 3"
    elif name == "cfg4":  # raw rows: the reference's async solver needs unit rows; serial norm-proportional rk_solve
        Ar, _ = R.build(A.m, A.n, np.repeat(np.arange(A.m), np.diff(A.row_ptr)), A.col_idx, A.values, False, None)
        t = R.rk_solve(Ar, b, x0, 1, 0.0, 42, "norm")
        p, w, cores, sample = int(t["updates_applied"][-1]), float(t["wall_seconds"][-1]), 1, \
            "1 epoch of serial rk_solve(norm_proportional) on the raw rows"
    else:  # cfg3: the reference runs fp64 only; 1 epoch of solve_parallel on all host threads
        t = R.solve_parallel(Ah, b, x0, threads=cores, gamma=1.0, epochs=1, target=0.0, variant="full_row",
                             sampling="slice_shuffle", seed=7, snapshot_interval=1, cap=4)
        p, w, sample = int(t["updates_applied"][-1]), float(t["wall_seconds"][-1]), \
            f"1 epoch of solve_parallel (fp64), {cores} threads"
    return {"value": p / w, "unit": "proj/s", "cores": cores, "kind": "reference", "sample": sample}


def run_sweep(args):
    """Config 2 with the active-warp count swept (BASELINE configs[1]): time to
    tolerance, epochs and throughput per warp count W beside the delay bound
    tau_max = m / (2 e lambda_max) - 1 (stepsize.cpp:59-82); ~2 W rows are in
    flight at once (2 per warp)."""
    import torch

    from paper_1401_4780_b200 import capi

    if int(os.environ.get("RANK", "0")) != 0:
        return 0
    A, b, xs = gen_system(CFG2["seed"])
    bb = float(b @ b)
    S = capi.System(A, b)
    lam, _ = S.power_iteration(1e-6)
    tau_max = CFG2["m"] / (2 * np.e * lam) - 1
    res = S.max_resident_warps()
    points = []
    for W in [32, 148, 592, 1184, 2368, 2664, 3552]:
        if W > res:
            continue
        kw = dict(threads=W, gamma=1.0, epochs=2000, target=TOL * TOL * bb, sampling=capi.SLICE_SHUFFLE,
                  snapshot_interval=1, x_star=xs, want_x=False)
        S.solve(seed=1, **kw)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        t = S.solve(seed=2, **kw)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        points.append({"warps": W, "rows_in_flight": 2 * W, "time_to_tolerance_ms": ms,
                       "epochs": int(t["epoch_index"][-1]), "proj_per_s": int(t["updates_applied"][-1]) / (ms * 1e-3),
                       "rel_error": float(np.sqrt(t["dist_sq"][-1] / float(xs @ xs)))})
    S.close()
    print(json.dumps({"metric": METRIC + " (warp sweep)", "unit": "proj/s", "n_gpus": 1, "data": "synthetic",
                      "dtype": "f64", "config": {"workload": workload_config()["workload"],
                                                 "lambda_max": lam, "tau_max": tau_max,
                                                 "resident_warps": res}, "points": points}))
    return 0


MC = dict(m=1200, n=60, theta=5, seed=77, runs=1000, iterations=2000, tau=5, gamma=0.15, base_seed=99)
MC_METRIC = "bounded-delay simulator iterations/sec (monte_carlo_ratios, acceptance C2 shape)"


def run_mc(args):
    """monte_carlo_ratios on acceptance criterion 2's shape
    (acceptance.cpp:137-155: 1000 runs x 2000 iterations, uniform delays tau=5,
    single component). b200 arm: device time of the resident-system call (CUDA
    events) as `value`, the one-shot host call as `e2e`. Reference arm: the
    reference's monte_carlo_ratios (oracle/_ref, single-threaded as upstream)
    on a bounded sample of 100 runs per step."""
    from paper_1401_4780_b200 import capi

    if int(os.environ.get("RANK", "0")) != 0:
        return 0
    A, b, _ = capi.generate_fixed_theta(MC["m"], MC["n"], MC["theta"], seed=MC["seed"])
    x0 = np.zeros(MC["n"])
    kw = dict(gamma=MC["gamma"], tau=MC["tau"], delay="uniform_random", iterations=MC["iterations"],
              base_seed=MC["base_seed"])
    cfg = {"workload": f"monte_carlo_ratios m={MC['m']} n={MC['n']} theta={MC['theta']} tau={MC['tau']} "
                       f"uniform_random single_component, {MC['iterations']} iterations"}
    line = {"metric": MC_METRIC, "unit": "iterations/s", "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic"}
    if args.impl == "reference":
        R = load_ref()
        if R is None:
            print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref not built"}))
            return 0
        Ar, _ = R.build(A.m, A.n, np.repeat(np.arange(A.m), np.diff(A.row_ptr)), A.col_idx, A.values, True, None)
        runs = 100
        for _ in range(args.warmup):
            R.monte_carlo(Ar, b, x0, runs=runs, **kw)
        t0 = time.perf_counter()
        for _ in range(args.steps):
            R.monte_carlo(Ar, b, x0, runs=runs, **kw)
        wall = time.perf_counter() - t0
        v = runs * MC["iterations"] * args.steps / wall
        line.update(value=v, ms_per_step=1e3 * wall / args.steps, impl="reference",
                    config=dict(cfg, runs=runs, threads=1),
                    cpu_baseline={"value": v, "unit": "iterations/s", "cores": 1, "kind": "reference",
                                  "sample": f"{runs} runs x {MC['iterations']} iterations per step"},
                    e2e={"value": v, "unit": "iterations/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0})
        print(json.dumps(line))
        return 0
    import torch

    runs = MC["runs"]
    S = capi.System(A, b)
    for _ in range(args.warmup):
        S.monte_carlo_ratios(x0, runs=runs, **kw)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    torch.cuda.synchronize()
    with ClockSampler(0) as clk:
        for k in range(args.steps):
            ev[k][0].record()
            S.monte_carlo_ratios(x0, runs=runs, **kw)
            ev[k][1].record()
        torch.cuda.synchronize()
    dev_ms = sum(a.elapsed_time(c) for a, c in ev)
    S.close()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        capi.monte_carlo_ratios(A, b, x0, runs=runs, **kw)
    wall = time.perf_counter() - t0
    it = runs * MC["iterations"] * args.steps
    line.update(value=it / (dev_ms * 1e-3), ms_per_step=dev_ms / args.steps, config=dict(cfg, runs=runs),
                e2e={"value": it / wall, "unit": "iterations/s",
                     "h2d_bytes_per_step": int(8 * (A.m + 1) + 12 * A.nnz + 16 * A.m + 8 * A.n),
                     "d2h_bytes_per_step": int(8 * (2 * MC["iterations"] + 1)), "ms_per_step": 1e3 * wall / args.steps},
                gpu_launches=3 * args.steps, clocks=clk.summary())
    print(json.dumps(line))
    return 0


LSQ = dict(m=4000, n=1000, theta=10, seed=7, noise=0.5, target_rel=1e-20, threads=256, gamma=1.0, epochs=20000)
LSQ_METRIC = "least-squares solves/sec (lsq_solve through the augmented system to the augmented-residual target)"


def run_lsq(args):
    """lsq_solve (lsq.cpp:103-170) on a noisy fixed-theta
    system. sigma_r (which the reference takes from its Eigen SVD, absent
    here) comes from the device dense SVD once and is passed to both arms.
    b200 arm: the host-buffer call (augment + upload + the augmented solve by
    LSQ['threads'] async warp workers + grad) — a host-to-host call, so value
    and e2e coincide; the deterministic (bit-identical) variant and the SVD
    time are reported in config. Reference arm: the reference lsq_solve
    (oracle/_ref, single core, rk_solve inside)."""
    from paper_1401_4780_b200 import capi

    if int(os.environ.get("RANK", "0")) != 0:
        return 0
    A, b, _ = capi.generate_fixed_theta(LSQ["m"], LSQ["n"], LSQ["theta"], seed=LSQ["seed"])
    b = b + LSQ["noise"] * np.random.default_rng(LSQ["seed"]).standard_normal(LSQ["m"])
    cfg = {"workload": f"lsq_solve m={LSQ['m']} n={LSQ['n']} theta={LSQ['theta']} N(0,1) unit rows, b = A x* + "
                       f"{LSQ['noise']} N(0,1); augmented {LSQ['m'] + LSQ['n']}^2 system to r_sq <= "
                       f"{LSQ['target_rel']} ||b_tilde||^2-scale target"}
    line = {"metric": LSQ_METRIC, "unit": "solves/s", "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic"}
    capi.dense_svd(A)  # (the first device call of the process also pays the CUDA context)
    t0 = time.perf_counter()
    sv = capi.dense_svd(A)
    svd_ms = 1e3 * (time.perf_counter() - t0)
    sr = float(sv["sigma"][sv["rank"] - 1])
    target = LSQ["target_rel"] * float(b @ b)
    kw = dict(sigma_r=sr, max_epochs=LSQ["epochs"], target=target, seed=1)
    if args.impl == "reference":
        R = load_ref()
        if R is None:
            print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref not built"}))
            return 0
        Ar, _ = R.build(A.m, A.n, np.repeat(np.arange(A.m), np.diff(A.row_ptr)), A.col_idx, A.values, True, None)
        for _ in range(args.warmup):
            r = R.lsq_solve(Ar, b, sr, max_epochs=LSQ["epochs"], target=target, seed=1)
        t0 = time.perf_counter()
        for _ in range(args.steps):
            r = R.lsq_solve(Ar, b, sr, max_epochs=LSQ["epochs"], target=target, seed=1)
        wall = time.perf_counter() - t0
        v = args.steps / wall
        line.update(value=v, ms_per_step=1e3 * wall / args.steps, impl="reference",
                    config=dict(cfg, solver="rk_solve (1 core)", grad_norm=r["grad_norm"],
                                epochs=int(r["trace"]["epoch_index"][-1])),
                    cpu_baseline={"value": v, "unit": "solves/s", "cores": 1, "kind": "reference",
                                  "sample": "one full lsq_solve per step"},
                    e2e={"value": v, "unit": "solves/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0})
        print(json.dumps(line))
        return 0

    def timed(threads, gamma, steps, warmup):
        for _ in range(warmup):
            capi.lsq_solve(A, b, threads=threads, gamma=gamma, **kw)
        t0 = time.perf_counter()
        for _ in range(steps):
            r = capi.lsq_solve(A, b, threads=threads, gamma=gamma, **kw)
        return 1e3 * (time.perf_counter() - t0) / steps, r

    with ClockSampler(0) as clk:
        ms, r = timed(LSQ["threads"], LSQ["gamma"], args.steps, args.warmup)
    det_ms, rd = timed(1, 1.0, max(1, args.steps // 5), 1)
    # kernel launches of one augmented solve (the resident-system twin of the call)
    phi, zeta = capi.lsq_optimal_params(sr)
    aug = capi.lsq_augment(A, b, zeta, phi)
    with capi.System(aug["a_tilde"], aug["b_tilde"]) as S:
        S.solve(threads=LSQ["threads"], gamma=LSQ["gamma"], epochs=LSQ["epochs"], target=target, seed=1,
                sampling=capi.WITH_REPLACEMENT)
        launches = int(S.stats()["kernel_launches"])
    cpu = None
    if not args.no_cpu_baseline:
        R = load_ref()
        if R is not None:
            Ar, _ = R.build(A.m, A.n, np.repeat(np.arange(A.m), np.diff(A.row_ptr)), A.col_idx, A.values, True, None)
            t0 = time.perf_counter()
            rr = R.lsq_solve(Ar, b, sr, max_epochs=LSQ["epochs"], target=target, seed=1)
            w = time.perf_counter() - t0
            cpu = {"value": 1.0 / w, "unit": "solves/s", "cores": 1, "kind": "reference",
                   "sample": f"one reference lsq_solve ({1e3 * w:.1f} ms, grad_norm {rr['grad_norm']:.3g})"}
    v = 1e3 / ms
    nbytes_in = int(8 * (A.m + 1) + 16 * A.nnz + 8 * A.m)
    line.update(value=v, ms_per_step=ms,
                config=dict(cfg, threads=LSQ["threads"], gamma=LSQ["gamma"], grad_norm=r["grad_norm"],
                            epochs=int(r["trace"]["epoch_index"][-1]), sigma_r=sr, dense_svd_ms=round(svd_ms, 2),
                            deterministic_ms=round(det_ms, 3), deterministic_grad_norm=rd["grad_norm"],
                            timing="wall clock of the host-buffer call (host-to-host API)"),
                e2e={"value": v, "unit": "solves/s", "h2d_bytes_per_step": nbytes_in,
                     "d2h_bytes_per_step": int(8 * (A.m + A.n)), "ms_per_step": ms},
                gpu_launches=launches, clocks=clk.summary())
    if cpu:
        line["cpu_baseline"] = cpu
    print(json.dumps(line))
    return 0


def run_cfg5_shards(args):
    """Config 5 per-rank work at G = 1, 2, 4, 8 on ONE GPU: the shard a rank of a
    G-GPU job owns (k/G RHS columns) solved alone (native loop, asyrk_mrhs_solve)
    with its own stop test. A projection of strong scaling, NOT a multi-GPU
    measurement: the G-GPU job adds one all-reduce of 3 doubles per evaluated
    boundary (NCCL) and its stop is global."""
    import torch

    from paper_1401_4780_b200 import capi
    from paper_1401_4780_b200.mrhs import shard_columns

    if int(os.environ.get("RANK", "0")) != 0:
        return 0
    A, B, Xs = capi.generate_fixed_theta(CFG5["m"], CFG5["n"], CFG5["theta"], seed=CFG5["seed"], k=CFG5["k"])
    B = B.astype(np.float32)
    points = []
    for G in [1, 2, 4, 8]:
        c0, c1 = shard_columns(CFG5["k"], G, 0)
        bb = float((B[:, c0:c1].astype(np.float64) ** 2).sum())
        S = capi.MultiRHS(A, B, c0, c1)
        W = args.warps or S.max_resident_warps()
        kw = dict(threads=W, gamma=1.0, epochs=2000, target=TOL5 * TOL5 * bb, snapshot_interval=1,
                  sampling=capi.SLICE_SHUFFLE, want_x=False)
        S.solve(seed=1, **kw)
        times, epochs, rows, wms = [], [], 0, 0.0
        for k in range(args.steps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record()
            t = S.solve(seed=100 + k, **kw)
            e1.record()
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1))
            epochs.append(int(t["epoch_index"][-1]))
            rows += int(t["updates_applied"][-1])
            wms += S.stats()["worker_ms"]
        S.close()
        ms = statistics.median(times)
        points.append({"gpus": G, "columns_per_gpu": c1 - c0, "warps": W, "shard_time_to_tolerance_ms": ms,
                       "epochs": statistics.median(epochs), "worker_ms_per_solve": wms / args.steps,
                       "shard_column_proj_per_s": rows * (c1 - c0) / (sum(times) * 1e-3)})
    t1 = points[0]["shard_time_to_tolerance_ms"]
    for p in points:
        p["projected_speedup_vs_1"] = t1 / p["shard_time_to_tolerance_ms"]
    print(json.dumps({"metric": METRIC + " (config 5 per-rank shard, projection)", "unit": "ms", "n_gpus": 1,
                      "data": "synthetic", "dtype": "f32", "steps": args.steps,
                      "config": {"workload": "config5: m=500000 n=250000 theta=20 k=64 fp32; each point = the "
                                             "k/G-column shard of one rank of a G-GPU job, solved alone on one "
                                             "GPU with a shard-local stop at 1e-5 (the real job all-reduces 3 "
                                             "doubles per evaluated boundary and stops globally)",
                                 "warps": "all co-resident worker warps per shard width", "sampling": "slice_shuffle"},
                      "points": points}))
    return 0


def _json_stdout():
    """The driver reads ONE JSON line from stdout, but native libraries print to
    file descriptor 1 on their own (NCCL's version banner when the box sets
    NCCL_DEBUG, its INFO log at N > 1): point fd 1 at stderr for everything else
    and give Python's print a private duplicate of the real stdout."""
    sys.stdout.flush()
    real = os.dup(1)
    os.dup2(2, 1)
    sys.stdout = os.fdopen(real, "w", buffering=1)


def main():
    _json_stdout()
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--warps", type=int, default=0, help="worker warps (0 = all resident warp slots)")
    ap.add_argument("--workload", default="cfg2", choices=["cfg2", "cfg5", "mc", "cfg1", "cfg3", "cfg3x", "cfg4",
                                                           "sweep", "cfg5shards", "lsq"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-cfg5", action="store_true", help="skip the config-5 (RHS-sharded) sub-line of the cfg2 run")
    args = ap.parse_args()
    if args.workload == "mc":
        return run_mc(args)
    if args.workload in OTHER:
        return run_other(args)
    if args.workload == "sweep":
        return run_sweep(args)
    if args.workload == "cfg5shards":
        return run_cfg5_shards(args)
    if args.workload == "lsq":
        return run_lsq(args)
    if args.impl == "reference":
        return run_reference(args)
    if args.workload == "cfg5":
        return run_gpu_cfg5(args)
    return run_gpu(args)


if __name__ == "__main__":
    sys.exit(main())
