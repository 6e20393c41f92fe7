"""GPU parity of the bounded-delay simulator (ref/src/delay_sim.cpp:71-338)
through the C ABI: simulate's records, events, history, probes and final_x,
and monte_carlo_ratios' means and ratios are BIT-IDENTICAL to the reference
(golden fixtures from oracle/_ref) and to the C restatement at larger sizes."""
import os
import sys

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

capi = pytest.importorskip("paper_1401_4780_b200.capi")
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "golden"))
import make_golden  # noqa: E402  (case tables only)

KEYS = ["epoch_index", "r_sq", "grad_sq", "updates_applied", "final_x", "history", "probe_iteration", "probe_r_sq"]


def sim_csr(golden, nm):
    p = f"sim_inst/{nm}/"
    m, n = (int(v) for v in golden[p + "shape"])
    A = capi.HostCsr(m, n, golden[p + "row_ptr"], golden[p + "col_idx"], golden[p + "values"], golden[p + "row_norm"])
    return A, golden[p + "b"]


def same(r, ref, tag):
    for k in KEYS:
        assert np.array_equal(r[k], ref[k]), (tag, k)
    for k in ref["events"]:
        assert np.array_equal(r["events"][k], ref["events"][k]), (tag, "ev_" + k)


def test_simulate_matches_reference_golden(golden):
    for case, nm, fill, kw in make_golden.SIM_CASES:
        A, b = sim_csr(golden, nm)
        r = capi.simulate(A, b, np.full(A.n, fill), **kw)
        ref = {k: golden[f"sim/{case}/{k}"] for k in KEYS}
        ref["events"] = {k: golden[f"sim/{case}/ev_{k}"] for k in ["j", "i", "t", "k", "step"]}
        same(r, ref, case)
    # the resident-system entry point (b of the system)
    case, nm, fill, kw = make_golden.SIM_CASES[-1]
    A, b = sim_csr(golden, nm)
    with capi.System(A, b) as S:
        r = S.simulate(np.full(A.n, fill), **kw)
    assert np.array_equal(r["probe_r_sq"], golden[f"sim/{case}/probe_r_sq"])
    assert np.array_equal(r["final_x"], golden[f"sim/{case}/final_x"])


def test_monte_carlo_matches_reference_golden(golden):
    for case, nm, fill, kw in make_golden.MC_CASES:
        A, b = sim_csr(golden, nm)
        r = capi.monte_carlo_ratios(A, b, np.full(A.n, fill), **kw)
        assert np.array_equal(r["mean_r_sq"], golden[f"mc/{case}/mean_r_sq"]), case
        assert np.array_equal(r["ratios"], golden[f"mc/{case}/ratios"]), case


def _fixed_theta_pair(m, n, theta, seed):
    A, b, xs = capi.generate_fixed_theta(m, n, theta, seed)
    Ac = oracle.C.from_arrays(m, n, A.row_ptr, A.col_idx, A.values)
    return A, Ac, b


@pytest.mark.parametrize("delay,variant,tau", [("uniform_random", "single_component", 50),
                                               ("max_staleness", "full_row", 7), ("fixed", "full_row", 0)])
def test_simulate_matches_oracle_larger(delay, variant, tau):
    A, Ac, b = _fixed_theta_pair(3000, 1500, 12, 21)
    kw = dict(gamma=0.5 if variant == "full_row" else 0.04, tau=tau, delay=delay, iterations=20000, seed=17,
              variant=variant, probe_every=97, probe_r_sq=True, max_events=300)
    x0 = np.zeros(1500)
    r = capi.simulate(A, b, x0, **kw)
    ref = oracle.C.simulate(Ac, b, x0, **kw)
    same(r, ref, (delay, variant, tau))
    assert r["r_sq"][-1] < r["r_sq"][0]


def test_monte_carlo_matches_oracle_acceptance_shape():
    # acceptance.cpp:137-155 style: many runs, uniform delays, single component
    A, Ac, b = _fixed_theta_pair(200, 80, 6, 5)
    kw = dict(gamma=0.1, tau=6, delay="uniform_random", iterations=400, runs=1000, base_seed=99)
    r = capi.monte_carlo_ratios(A, b, np.zeros(80), **kw)
    ref = oracle.C.monte_carlo(Ac, b, np.zeros(80), **kw)
    assert np.array_equal(r["mean_r_sq"], ref["mean_r_sq"]) and np.array_equal(r["ratios"], ref["ratios"])


def test_rate_fit_matches_reference(golden):
    f = capi.rate_fit(golden["fit/y"], 3.0)
    assert np.array_equal(np.array([f["slope"], f["r2"]]), golden["fit/vals"])
    with pytest.raises(capi.AsyrkError, match="InsufficientData"):
        capi.rate_fit(np.ones(10))
    z = np.ones(25)
    z[7] = 0.0
    with pytest.raises(capi.AsyrkError, match=r"NonPositiveData: .*index 7"):
        capi.rate_fit(z)


def test_simulator_errors(golden):
    A, b = sim_csr(golden, "d10x6")
    x0 = np.zeros(6)
    with pytest.raises(capi.AsyrkError, match="InsufficientData"):
        capi.monte_carlo_ratios(A, b, x0, 0.1, 1, "fixed", 5, 50, 1)
    with pytest.raises(capi.AsyrkError, match="InvalidGamma"):
        capi.simulate(A, b, x0, -0.1, 1, "fixed", 5, 1, "full_row")
    with pytest.raises(capi.AsyrkError, match="InvalidArgument"):
        capi.simulate(A, b, x0, 0.1, 1, "fixed", 0, 1, "full_row")
    with pytest.raises(capi.AsyrkError, match="InvalidArgument"):
        capi.simulate(A, b, x0, 0.1, -1, "fixed", 5, 1, "full_row")
    with pytest.raises(capi.AsyrkError, match="SolutionProjector"):
        capi.simulate(A, b, x0, 0.1, 1, "fixed", 5, 1, "full_row", probe_every=1, probe_dist_sq=True)
    U = capi.HostCsr(2, 2, [0, 1, 2], [0, 1], [2.0, 1.0])
    with pytest.raises(capi.AsyrkError, match="NotNormalized"):
        capi.simulate(U, np.zeros(2), np.zeros(2), 0.1, 1, "fixed", 5, 1, "full_row")
    # a diverging step blows the iterate up: NonFinite, like the reference's record()
    with pytest.raises(capi.AsyrkError, match="NonFinite: iterate became non-finite"):
        capi.simulate(A, b, x0, 1e300, 0, "fixed", 200, 1, "single_component")
    with pytest.raises(oracle.OracleError, match="NonFinite"):
        Ac = oracle.C.from_arrays(A.m, A.n, A.row_ptr, A.col_idx, A.values)
        oracle.C.simulate(Ac, b, x0, 1e300, 0, "fixed", 200, 1, "single_component")


def test_pybind_simulate_matches_oracle(golden):
    # module.cpp:213-238: normalize, step parameters from the statistics,
    # gamma overridden, simulate; the trace is the reference's simulate trace
    import paper_1401_4780_b200 as pkg

    A, b = sim_csr(golden, "d30x20")
    rows = np.repeat(np.arange(A.m), np.diff(A.row_ptr))
    d = pkg.simulate(A.m, A.n, rows, A.col_idx, A.values, b, 500, 3, 0.05, delay="max", variant="single", seed=4)
    Ac = oracle.C.from_arrays(A.m, A.n, A.row_ptr, A.col_idx, A.values)
    ref = oracle.C.simulate(Ac, b, np.zeros(A.n), 0.05, 3, "max_staleness", 500, 4, "single_component")
    for k in ["epoch_index", "r_sq", "grad_sq", "updates_applied", "final_x"]:
        assert np.array_equal(np.asarray(d[k]), ref[k]), k
    assert d["gamma"] == 0.05
    st = oracle.C.stats_full(Ac)
    # compute_stats' default exact_spectral: lambda_max = sigma_max^2 of the dense SVD
    D = np.zeros((A.m, A.n))
    for i in range(A.m):
        D[i, A.col_idx[A.row_ptr[i]:A.row_ptr[i + 1]]] = A.values[A.row_ptr[i]:A.row_ptr[i + 1]]
    lam = np.linalg.svd(D, compute_uv=False)[0] ** 2
    assert abs(lam - st["lambda_max"]) <= 1e-7 * lam  # (power iteration, tol 1e-9 on the quotient)
    cor = oracle.C.corollary(A.m, st["mu"], lam, 3)
    assert abs(d["rho"] - cor["rho"]) <= 1e-12 * cor["rho"] and abs(d["psi"] - cor["psi"]) <= 1e-12 * cor["psi"]
    with pytest.raises(ValueError, match="InvalidArgument"):
        pkg.simulate(A.m, A.n, rows, A.col_idx, A.values, b, 10, 1, 0.1, delay="sometimes")


def test_simulator_projector_distances(golden):
    # SimOptions::projector (delay_sim.cpp:94-123, 154): with the projector's
    # solution point every record carries dist_sq and probe_dist_sq follows
    # ||x - A^+ b||^2 at the probe iterations; the r_sq probes and the trace
    # stay bit-identical to the run without distances
    A, b = sim_csr(golden, "d30x20")
    xp = capi.dense_lstsq(A, b)
    x0 = np.full(A.n, 0.25)
    kw = dict(probe_every=7, probe_r_sq=True)
    plain = capi.simulate(A, b, x0, 0.05, 3, "uniform_random", 400, 11, "single_component", **kw)
    d = capi.simulate(A, b, x0, 0.05, 3, "uniform_random", 400, 11, "single_component", probe_dist_sq=True,
                      dist_point=xp, **kw)
    for k in ["epoch_index", "r_sq", "grad_sq", "final_x", "probe_r_sq", "probe_iteration"]:
        assert np.array_equal(d[k], plain[k]), k
    assert len(d["dist_sq"]) == len(d["r_sq"]) and len(d["probe_dist_sq"]) == len(d["probe_iteration"])
    f = d["final_x"] - xp
    assert abs(d["dist_sq"][-1] - f @ f) <= 1e-12 * (f @ f)
    assert abs(d["probe_dist_sq"][0] - (x0 - xp) @ (x0 - xp)) <= 1e-12 * ((x0 - xp) @ (x0 - xp))
    with pytest.raises(capi.AsyrkError, match="InvalidArgument"):
        capi.simulate(A, b, x0, 0.05, 3, "uniform_random", 40, 11, "single_component", probe_every=7,
                      probe_dist_sq=True)
