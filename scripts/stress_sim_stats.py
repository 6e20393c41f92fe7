"""Randomized bit-identity stress of the device bounded-delay simulator
(simulate: records, events, history, probes, final_x) and compute_stats
(every structural field) against the C restatement.
Usage: python scripts/stress_sim_stats.py [cases] [seed]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import oracle  # noqa: E402
from paper_1401_4780_b200 import capi  # noqa: E402

SIM_KEYS = ["epoch_index", "r_sq", "grad_sq", "updates_applied", "final_x", "history", "probe_iteration",
            "probe_r_sq"]
STAT_KEYS = ["mu", "nu", "delta", "alpha", "frob_sq", "l_max", "l_res"]


def unit_system(rng, m, n):
    lens = rng.integers(1, min(n, 12) + 1, size=m)
    rp = np.concatenate([[0], np.cumsum(lens)])
    ci = np.concatenate([np.sort(rng.choice(n, size=k, replace=False)) for k in lens])
    v = rng.standard_normal(rp[-1])
    v /= np.repeat(np.sqrt(capi.serial_row_sumsq(rp, v)), lens)
    return capi.HostCsr(m, n, rp, ci, v), rng.standard_normal(m)


def main():
    cases = int(sys.argv[1]) if len(sys.argv) > 1 else 200
    rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 1)
    t0 = time.time()
    bad = 0
    for c in range(cases):
        m = int(rng.integers(3, 400))
        n = int(rng.integers(2, 200))
        A, b = unit_system(rng, m, n)
        Ao = oracle.C.from_arrays(A.m, A.n, A.row_ptr, A.col_idx, A.values)
        # simulate
        tau = int(rng.integers(0, 8))
        delay = str(rng.choice(["fixed", "uniform_random", "max_staleness"]))
        variant = str(rng.choice(["single_component", "full_row"]))
        gamma = float(rng.uniform(0.01, 0.6))
        iters = int(rng.integers(1, 3000))
        seed = int(rng.integers(0, 2**31))
        pe = int(rng.choice([0, 1, 7, 50]))
        pr = bool(pe and rng.random() < 0.7)
        me = int(rng.choice([0, 10, 5000]))
        x0 = rng.standard_normal(A.n) * float(rng.choice([0.0, 1.0]))
        try:
            got = capi.simulate(A, b, x0, gamma, tau, delay, iters, seed, variant, probe_every=pe, probe_r_sq=pr,
                                max_events=me)
        except capi.AsyrkError as e:
            got = str(e)
        try:
            want = oracle.C.simulate(Ao, b, x0, gamma, tau, delay, iters, seed, variant, pe, pr, me)
        except oracle.OracleError as e:
            want = str(e)
        if isinstance(got, str) or isinstance(want, str):
            ok = isinstance(got, str) and isinstance(want, str)
        else:
            ok = all(np.array_equal(np.asarray(got[k]), np.asarray(want[k])) for k in SIM_KEYS)
            ok &= all(np.array_equal(got["events"][k], want["events"][k]) for k in want["events"])
        if not ok:
            bad += 1
            print(f"SIM MISMATCH case {c}: m={m} n={n} tau={tau} {delay} {variant} iters={iters} pe={pe} pr={pr}",
                  flush=True)
        # compute_stats (structural fields; lambda_max is iterative on both sides)
        try:
            gs = capi.compute_stats(A)
            ws = oracle.C.stats_full(Ao)
            ok = all(gs[k] == ws[k] for k in STAT_KEYS) and np.array_equal(gs["theta"], ws["theta"])
            ok &= abs(gs["lambda_max"] - ws["lambda_max"]) <= 1e-6 * ws["lambda_max"]
        except (capi.AsyrkError, oracle.OracleError) as e:
            ok = "ZeroColumn" in str(e)
            try:
                capi.compute_stats(A)
                ok = False
            except capi.AsyrkError:
                pass
        if not ok:
            bad += 1
            print(f"STATS MISMATCH case {c}: m={m} n={n}", flush=True)
    print(f"{cases} cases, {bad} mismatches, {time.time() - t0:.1f} s", flush=True)
    return 1 if bad else 0


if __name__ == "__main__":
    sys.exit(main())
