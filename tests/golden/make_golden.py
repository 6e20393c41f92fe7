"""Generate tests/golden/golden.npz from the REFERENCE ITSELF (oracle/_ref,
the unmodified /root/reference sources compiled by oracle/Makefile).

Run here (where /root/reference exists):  python tests/golden/make_golden.py
The fixtures travel with the repo, so the GPU box never needs the reference.

Contents (all produced by reference code paths):
  rng/*            make_stream raw outputs, uniform_below, normals, cumulative
                   shuffles, alias draws (ref/include/asyrk/rng.hpp, kaczmarz.cpp:14-69)
  inst/<name>/*    gen_sparse_gaussian instances used by the reference tests
                   (CSR arrays after normalize_rows, b, x*)
  rk/<name>/<s>/*  rk_solve traces (uniform / shuffle / norm) incl. final_x
  par/<name>/<v>_<s>/*  solve_parallel(threads=1) traces + instrument reports
  res/<name>/*     residuals at a fixed x
  pow/<name>       power_iteration_lambda_max(tol=1e-10)
  stats/<name>/*   compute_stats(exact_spectral=false): STATS_FIELDS + theta (or error code)
  sim_inst/, sim/, mc/, fit/  simulate / monte_carlo_ratios / rate_fit cases (delay_sim.cpp)
  kat/*            known-answer vectors of the reference unit tests
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import REF  # noqa: E402

# (m, n, delta, seed) — instances of the reference's own tests
INSTANCES = {
    "par_shuffle_30x15": (30, 15, 0.25, 61),      # test_parallel.cpp:10-43
    "snap_24x12": (24, 12, 0.3, 67),               # test_parallel.cpp:45-60
    "instr_48x16": (48, 16, 0.3, 71),              # test_parallel.cpp:62-85
    "repl_40x20": (40, 20, 0.25, 73),              # test_parallel.cpp:87-98
    "diverge_20x10": (20, 10, 0.4, 79),            # test_parallel.cpp:100-109
    "at_solution_20x10": (20, 10, 0.4, 83),        # test_parallel.cpp:111-119
    "accept5_200x80": (200, 80, 0.1, 5150),        # acceptance.cpp:230-270 (C5)
    "stats_200x120": (200, 120, 0.05, 29),         # test_stats.cpp:47-62
    "seed_30x15": (30, 15, 0.25, 43),              # test_kaczmarz.cpp:94-106
    "dist_40x20": (40, 20, 0.2, 47),               # test_kaczmarz.cpp:108-122
    "delay0_20x12": (20, 12, 0.3, 7),              # test_delay_sim.cpp:28-52
    "accept9_2000x1500": (2000, 1500, 0.01, 90210),  # acceptance.cpp:400-418 (C9)
}


STATS_FIELDS = ["mu", "nu", "delta", "alpha", "lambda_max", "frob_sq", "l_max", "l_res"]


def stats_vector(st):
    return np.array([float(st[k]) for k in STATS_FIELDS])


# bounded-delay simulator cases of test_delay_sim.cpp (name: instance, x0 fill, kwargs)
SIM_INSTANCES = {
    "d20x12": (20, 12, 0.3, 7),     # test_delay_sim.cpp:28-52, 136-146
    "d8x5": (8, 5, 0.5, 17),        # :69-124
    "d6x4": (6, 4, 0.5, 19),        # :126-134
    "d10x8": (10, 8, 0.4, 23),      # :148-170
    "d10x6": (10, 6, 0.4, 29),      # :172-181
    "d30x20": (30, 20, 0.25, 3),    # :213-234
}
SIM_CASES = [
    ("serial_equiv", "d20x12", 0.0, dict(gamma=1.0, tau=0, delay="fixed", iterations=100, seed=42,
                                          variant="full_row")),
    ("fixed2_single", "d8x5", 0.0, dict(gamma=0.3, tau=2, delay="fixed", iterations=100, seed=5,
                                         variant="single_component", max_events=256)),
    ("maxst3_single", "d8x5", 0.0, dict(gamma=0.3, tau=3, delay="max_staleness", iterations=100, seed=5,
                                         variant="single_component", max_events=256)),
    ("unif3_single", "d8x5", 0.0, dict(gamma=0.3, tau=3, delay="uniform_random", iterations=200, seed=5,
                                        variant="single_component", max_events=256)),
    ("fixed1_full", "d8x5", 0.0, dict(gamma=0.5, tau=1, delay="fixed", iterations=60, seed=5, variant="full_row",
                                       max_events=256)),
    ("history", "d6x4", 0.0, dict(gamma=0.4, tau=2, delay="fixed", iterations=7, seed=11, variant="full_row")),
    ("partial_epoch", "d20x12", 0.0, dict(gamma=1.0, tau=0, delay="fixed", iterations=25, seed=4,
                                          variant="full_row")),
    ("probes", "d10x8", 0.0, dict(gamma=0.5, tau=1, delay="uniform_random", iterations=50, seed=2,
                                   variant="full_row", probe_every=10, probe_r_sq=True)),
    ("probes_single", "d30x20", 0.0, dict(gamma=0.06, tau=4, delay="uniform_random", iterations=700, seed=9,
                                           variant="single_component", probe_every=7, probe_r_sq=True,
                                           max_events=1000)),
]
MC_CASES = [
    ("frozen", "d10x6", 0.5, dict(gamma=0.0, tau=2, delay="uniform_random", iterations=5, runs=100, base_seed=77)),
    ("stale8", "d30x20", 0.0, dict(gamma=0.06, tau=8, delay="max_staleness", iterations=1200, runs=200,
                                    base_seed=11)),
    ("unif5_full", "d20x12", 0.0, dict(gamma=0.7, tau=5, delay="uniform_random", iterations=300, runs=100,
                                        base_seed=3, variant="full_row")),
]


def sim_golden(out):
    """simulate / monte_carlo_ratios / rate_fit outputs of the reference (delay_sim.cpp)."""
    insts = {}
    for nm, (m, n, delta, seed) in SIM_INSTANCES.items():
        A, b, xs = REF.gen_sparse_gaussian(m, n, delta, seed)
        e = A.export()
        insts[nm] = (A, b)
        p = f"sim_inst/{nm}/"
        out[p + "shape"] = np.array([m, n])
        for k in ["row_ptr", "col_idx", "values", "row_norm"]:
            out[p + k] = e[k]
        out[p + "b"] = b
    for case, nm, fill, kw in SIM_CASES:
        A, b = insts[nm]
        r = REF.simulate(A, b, np.full(A.n, fill), **kw)
        q = f"sim/{case}/"
        for k in ["epoch_index", "r_sq", "grad_sq", "updates_applied", "final_x", "history", "probe_iteration",
                  "probe_r_sq"]:
            out[q + k] = r[k]
        for k, v in r["events"].items():
            out[q + "ev_" + k] = v
    for case, nm, fill, kw in MC_CASES:
        A, b = insts[nm]
        r = REF.monte_carlo(A, b, np.full(A.n, fill), **kw)
        out[f"mc/{case}/mean_r_sq"] = r["mean_r_sq"]
        out[f"mc/{case}/ratios"] = r["ratios"]
    y = np.exp(-0.1 * np.arange(40)) * (1 + 0.01 * np.sin(np.arange(40)))
    out["fit/y"] = y
    f = REF.rate_fit(y, 3.0)
    out["fit/vals"] = np.array([f["slope"], f["r2"]])


# least-squares cases of test_lsq.cpp:128-213 and acceptance.cpp:316-340 (C7):
# name: (m, n, delta, seed, noise, lsq kwargs). The reference's inconsistent
# generator needs the Eigen SVD (absent), so b = consistent b + noise *
# N(0,1) from numpy's generator seeded with the instance seed; sigma_r (which
# the reference would take from its dense SVD) is LAPACK's via numpy and is
# passed to both implementations.
LSQ_CASES = {
    "l60x30": (60, 30, 0.25, 101, 0.4, dict(max_epochs=60000, target=1e-18, seed=3)),
    "l60x30_shuffle": (60, 30, 0.25, 101, 0.4, dict(max_epochs=300, target=0.0, seed=4, sampling="shuffle")),
    "l40x16_consistent": (40, 16, 0.3, 107, 0.0, dict(max_epochs=40000, target=1e-20)),
    "l30x12_explicit": (30, 12, 0.3, 109, 0.3, dict(zeta=0.37, phi=1.5, max_epochs=10)),
    "l200x100_c7": (200, 100, 0.1, 61, 0.5, dict(max_epochs=200000, target=1e-16, seed=17)),
}


def dense_of(e, m, n):
    D = np.zeros((m, n))
    for i in range(m):
        for k in range(e["row_ptr"][i], e["row_ptr"][i + 1]):
            D[i, e["col_idx"][k]] = e["values"][k]
    return D


def lsq_golden(out):
    for nm, (m, n, delta, seed, noise, kw) in LSQ_CASES.items():
        A, b, xs = REF.gen_sparse_gaussian(m, n, delta, seed)
        if noise:
            b = b + noise * np.random.default_rng(seed).standard_normal(m)
        e = A.export()
        s = np.linalg.svd(dense_of(e, m, n), compute_uv=False)
        sigma_r = float(s[s > 1e-10 * s[0]][-1])
        p = f"lsq/{nm}/"
        out[p + "shape"] = np.array([m, n])
        for k in ["row_ptr", "col_idx", "values", "row_norm"]:
            out[p + k] = e[k]
        out[p + "b"] = b
        out[p + "sigma_r"] = np.array([sigma_r])
        r = REF.lsq_solve(A, b, sigma_r, **kw)
        for k in ["x_ls", "y"]:
            out[p + k] = r[k]
        out[p + "scal"] = np.array([r["grad_norm"], r["zeta"], r["phi"], r["sigma_r"]])
        out[p + "r_sq"] = r["trace"]["r_sq"]
        out[p + "epoch_index"] = r["trace"]["epoch_index"]


# instances of the reference's acceptance criteria (acceptance.cpp:66-103):
# name: (m, n, delta, seed or None, tau, lambda_min floor). seed None = the
# find_feasible scan over seeds 1..400 (ZeroColumn draws skipped; lambda_min
# from the dense spectrum — LAPACK via numpy, the reference's Eigen being
# absent — must reach the floor and the corollary be feasible at tau).
ACCEPT = {
    "c1": (500, 200, 0.10, 20240501, 0, 0.0),   # criterion 1
    "c23": (1200, 60, 0.08, None, 5, 0.02),     # criteria 2 and 3 (shared instance)
    "c6": (100, 50, 0.08, None, 2, 0.04),       # criterion 6
}


def accept_golden(out):
    for nm, (m, n, delta, seed, tau, floor) in ACCEPT.items():
        for sd in ([seed] if seed is not None else range(1, 401)):
            A, b, xs = REF.gen_sparse_gaussian(m, n, delta, sd)
            try:
                st = REF.stats_full(A)
            except Exception:  # ZeroColumn: skipped as find_feasible does
                continue
            e = A.export()
            s = np.linalg.svd(dense_of(e, m, n), compute_uv=False)
            lmin = float(s[s > 1e-10 * s[0]][-1]) ** 2
            if seed is None:
                if lmin < floor or not REF.corollary(m, st["mu"], st["alpha"], float(s[0]) ** 2, tau)["feasible"]:
                    continue
            p = f"acc/{nm}/"
            out[p + "shape"] = np.array([m, n, sd])
            for k in ["row_ptr", "col_idx", "values", "row_norm"]:
                out[p + k] = e[k]
            out[p + "b"] = b
            out[p + "x_star"] = xs
            break
        else:
            raise RuntimeError(f"no feasible instance for {nm}")


def main():
    out = {}
    # ---- RNG known answers
    for seed, stream in [(0, 0), (42, 0), (31337, 3), (0x5CA1AB1E, 0)]:
        out[f"rng/raw/{seed}_{stream}"] = REF.stream_raw(seed, stream, 1000)
    out["rng/below/7_3_20000"] = REF.uniform_below_seq(7, 3, 20000, 2000)
    out["rng/below/9_0_3"] = REF.uniform_below_seq(9, 0, 3, 2000)
    out["rng/normal/1_2"] = REF.normal_seq(1, 2, 500)
    out["rng/shuffle/21_0_30x5"] = REF.shuffle_seq(21, 0, 30, 5)
    w = np.array([1.0, 2.0, 3.0])
    out["rng/alias/w"] = w
    out["rng/alias/123"] = REF.alias_sample_seq(w, 123, 5000)
    w2 = np.linspace(0.1, 4.0, 37) ** 2
    out["rng/alias2/w"] = w2
    out["rng/alias2/5"] = REF.alias_sample_seq(w2, 5, 5000)

    # ---- instances + traces
    for name, (m, n, delta, seed) in INSTANCES.items():
        A, b, xs = REF.gen_sparse_gaussian(m, n, delta, seed)
        e = A.export()
        p = f"inst/{name}/"
        out[p + "shape"] = np.array([m, n])
        out[p + "row_ptr"] = e["row_ptr"]
        out[p + "col_idx"] = e["col_idx"]
        out[p + "values"] = e["values"]
        out[p + "row_norm"] = e["row_norm"]
        out[p + "b"] = b
        out[p + "x_star"] = xs
        x0 = np.zeros(n)
        epochs = 40 if m <= 200 else 10
        for s in ["uniform", "shuffle", "norm"]:
            t = REF.rk_solve(A, b, x0, epochs, 0.0, 31337, s, xs)
            q = f"rk/{name}/{s}/"
            for k in ["epoch_index", "r_sq", "grad_sq", "dist_sq", "updates_applied", "final_x"]:
                out[q + k] = t[k]
        for v in ["full_row", "single"]:
            for s in ["slice_shuffle", "with_replacement"]:
                gamma = 1.0 if v == "full_row" else 0.05
                t = REF.solve_parallel(A, b, x0, 1, gamma, 13, 0.0, v, s, 21, 3, xs, True)
                q = f"par/{name}/{v}_{s}/"
                for k in ["epoch_index", "r_sq", "grad_sq", "dist_sq", "updates_applied", "final_x"]:
                    out[q + k] = t[k]
                ins = t["instrument"]
                out[q + "instrument"] = np.array([ins["row_updates"], ins["increments"], ins["max_abs_error"],
                                                  ins["tolerance"], float(ins["consistent"])])
        rng = np.random.default_rng(seed)
        xr = rng.standard_normal(n)
        out[f"res/{name}/x"] = xr
        out[f"res/{name}/vals"] = np.array(REF.residuals(A, xr, b))
        out[f"res/{name}/Ax"] = REF.multiply(A, xr)
        out[f"res/{name}/ATr"] = REF.multiply_transpose(A, rng.standard_normal(m))
        out[f"res/{name}/r_in"] = np.random.default_rng(seed).standard_normal(n + m)[n:]
        out[f"res/{name}/ATr"] = REF.multiply_transpose(A, out[f"res/{name}/r_in"])
        out[f"pow/{name}"] = np.array([REF.power_iteration(A, 1e-10, 200000)])
        try:  # compute_stats(exact_spectral=false), stats.cpp:52-130
            st = REF.stats_full(A, 1e-9, 200000)
            out[f"stats/{name}/vals"] = stats_vector(st)
            out[f"stats/{name}/theta"] = st["theta"]
        except Exception as ex:  # e.g. ZeroColumn on the tiny instances
            out[f"stats/{name}/error"] = np.array([ex.code])

    # ---- known answers of the reference unit tests
    A, bn = REF.build(1, 2, [0, 0], [0, 1], [3.0, 4.0], True, np.array([10.0]))  # test_kaczmarz.cpp:21-30
    out["kat/rk_step_34/x1"] = REF.rk_step(A, bn, np.zeros(2), 0)
    s = np.sqrt(0.5)
    A3, _ = REF.build(3, 2, [0, 1, 2, 2], [0, 1, 0, 1], [1.0, 1.0, s, s], False, None)
    out["kat/asyrk_update/third_row"] = np.array([REF.asyrk_update(A3, np.zeros(3), 2, 1, 0.5, np.array([1.0, 0.0]))])
    out["kat/asyrk_update/singleton"] = np.array([REF.asyrk_update(A3, np.array([4.0, 0.0, 0.0]), 0, 0, 1.0,
                                                                   np.array([3.0, 0.0]))])
    # compute_stats known answers (test_stats.cpp:8-44): identity, rows e1, e2, (sqrt(.5), sqrt(.5))
    # (unit rows: normalize_rows leaves them bit-identical and sets the flag)
    I3, _ = REF.build(3, 3, [0, 1, 2], [0, 1, 2], [1.0, 1.0, 1.0], True, None)
    out["kat/stats/identity3"] = stats_vector(REF.stats_full(I3, 1e-9, 200000))
    A3n, _ = REF.build(3, 2, [0, 1, 2, 2], [0, 1, 0, 1], [1.0, 1.0, s, s], True, None)
    out["kat/stats/three_row"] = stats_vector(REF.stats_full(A3n, 1e-9, 200000))
    sim_golden(out)
    lsq_golden(out)
    accept_golden(out)
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.npz")
    np.savez_compressed(path, **out)
    print(f"wrote {path}: {len(out)} arrays, {os.path.getsize(path) / 1e3:.0f} kB")


if __name__ == "__main__":
    main()
