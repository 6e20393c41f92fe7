"""GPU parity of compute_stats (ref/src/stats.cpp:52-130, exact_spectral=false)
through the C ABI: mu, nu, delta, theta, alpha, frob_sq, l_max and l_res are
BIT-IDENTICAL to the reference (golden fixtures from oracle/_ref) and to the C
restatement at larger sizes; lambda_max (power iteration, tol 1e-9) agrees
within 1e-8 relative (the device dot products use a fixed tree order)."""
import numpy as np
import pytest

import oracle
from conftest import triplets

pytestmark = pytest.mark.gpu

capi = pytest.importorskip("paper_1401_4780_b200.capi")
FIELDS = ["mu", "nu", "delta", "alpha", "lambda_max", "frob_sq", "l_max", "l_res"]
EXACT = ["mu", "nu", "delta", "alpha", "frob_sq", "l_max", "l_res"]
LAMBDA_RTOL = 1e-8


def host_csr(inst):
    return capi.HostCsr(inst["m"], inst["n"], inst["row_ptr"], inst["col_idx"], inst["values"], inst["row_norm"])


def check_against(st, ref_vec, ref_theta=None, tag=""):
    ref = dict(zip(FIELDS, ref_vec))
    for k in EXACT:
        assert float(st[k]) == ref[k], (tag, k, st[k], ref[k])
    assert abs(st["lambda_max"] - ref["lambda_max"]) <= LAMBDA_RTOL * ref["lambda_max"], tag
    if ref_theta is not None:
        assert np.array_equal(st["theta"], ref_theta), tag


def test_compute_stats_matches_reference_golden(golden, instances):
    for nm, inst in instances.items():
        key = f"stats/{nm}/"
        if key + "error" in golden.files:
            with pytest.raises(capi.AsyrkError):
                capi.compute_stats(host_csr(inst))
            continue
        st = capi.compute_stats(host_csr(inst), 1e-9, 200000)
        check_against(st, golden[key + "vals"], golden[key + "theta"], nm)
        with capi.System(host_csr(inst), inst["b"]) as S:  # resident-handle entry point
            check_against(S.compute_stats(1e-9, 200000), golden[key + "vals"], golden[key + "theta"], nm)


def test_compute_stats_known_answers(golden):
    # test_stats.cpp:8-44: the identity and rows e1, e2, (sqrt(.5), sqrt(.5))
    I3 = capi.HostCsr(3, 3, [0, 1, 2, 3], [0, 1, 2], [1.0, 1.0, 1.0])
    st = capi.compute_stats(I3)
    check_against(st, golden["kat/stats/identity3"], np.array([1, 1, 1]))
    s = np.sqrt(0.5)
    A3 = capi.HostCsr(3, 2, [0, 1, 2, 4], [0, 1, 0, 1], [1.0, 1.0, s, s])
    st = capi.compute_stats(A3)
    check_against(st, golden["kat/stats/three_row"], np.array([1, 1, 2]))
    assert abs(st["alpha"] - 1.7320508075688772) <= 1.8e-14 and abs(st["l_res"] - 1.5811388300841898) <= 1.6e-14


def _oracle_of(A):
    Ac = oracle.C.from_arrays(A.m, A.n, A.row_ptr, A.col_idx, A.values)
    return oracle.C.stats_full(Ac, 1e-9, 200000)


def _vec(d):
    return np.array([float(d[k]) for k in FIELDS])


@pytest.mark.parametrize("m,n,theta,seed", [(20000, 10000, 20, 5), (30000, 12000, 24, 6)])
def test_compute_stats_matches_oracle_fixed_theta(m, n, theta, seed):
    A, b, xs = capi.generate_fixed_theta(m, n, theta, seed)
    ref = _oracle_of(A)
    check_against(capi.compute_stats(A), _vec(ref), ref["theta"], (m, n))


def test_compute_stats_ragged_rows_and_heavy_column():
    # ragged rows (1..40 nonzeros) plus one column present in every row: the
    # l_res table of that column exceeds shared memory (global-scratch path)
    rng = np.random.default_rng(11)
    m, n = 6000, 5000
    rows, cols = [], []
    for i in range(m):
        k = int(rng.integers(1, 41))
        c = np.unique(np.concatenate([[0], rng.choice(np.arange(1, n), size=k, replace=False)]))
        rows.append(np.full(c.size, i))
        cols.append(c)
    rows, cols = np.concatenate(rows), np.concatenate(cols)
    vals = rng.standard_normal(rows.size)
    Ac, _ = oracle.C.build(m, n, rows, cols, vals, normalize=True)
    e = oracle.C._export(Ac)
    A = capi.HostCsr(m, n, e["row_ptr"], e["col_idx"], e["values"], e["row_norm"], normalized=True)
    ref = oracle.C.stats_full(Ac, 1e-9, 200000)
    st = capi.compute_stats(A)
    check_against(st, _vec(ref), ref["theta"], "ragged")
    assert st["nu"] == m


def test_compute_stats_errors():
    A = capi.HostCsr(2, 2, [0, 1, 2], [0, 1], [2.0, 1.0])  # rows not unit
    with pytest.raises(capi.AsyrkError, match="NotNormalized"):
        capi.compute_stats(A)
    Z = capi.HostCsr(2, 3, [0, 1, 2], [0, 2], [1.0, 1.0])  # column 1 empty
    with pytest.raises(capi.AsyrkError, match="ZeroColumn: column 1"):
        capi.compute_stats(Z)


def test_pybind_system_stats_and_step_params(golden, instances):
    # module.cpp:113-157 with the device statistics; compute_stats' default
    # exact_spectral: lambda_max / lambda_min / sigma_r from the device SVD
    import paper_1401_4780_b200 as pkg

    nm = "stats_200x120"
    inst = instances[nm]
    rows = np.repeat(np.arange(inst["m"]), np.diff(inst["row_ptr"]))
    d = pkg.system_stats(inst["m"], inst["n"], rows, inst["col_idx"], inst["values"])
    ref = dict(zip(FIELDS, golden[f"stats/{nm}/vals"]))
    for k in EXACT:
        assert float(d[k]) == ref[k], k
    assert list(d["theta"]) == list(golden[f"stats/{nm}/theta"])
    D = np.zeros((inst["m"], inst["n"]))
    for i in range(inst["m"]):
        lo, hi = inst["row_ptr"][i], inst["row_ptr"][i + 1]
        D[i, inst["col_idx"][lo:hi]] = inst["values"][lo:hi]
    sv = np.linalg.svd(D, compute_uv=False)
    sr = sv[sv > 1e-10 * sv[0]][-1]
    assert abs(d["lambda_max"] - sv[0] ** 2) <= 1e-12 * sv[0] ** 2
    assert abs(d["lambda_max"] - ref["lambda_max"]) <= 1e-8 * ref["lambda_max"]  # vs the power iteration
    assert abs(d["sigma_r"] - sr) <= 1e-12 * sv[0] and abs(d["lambda_min"] - d["sigma_r"] ** 2) == 0.0
    p = pkg.step_params(inst["m"], inst["n"], rows, inst["col_idx"], inst["values"], 2)
    Ac = oracle.C.from_arrays(inst["m"], inst["n"], inst["row_ptr"], inst["col_idx"], inst["values"])
    cor = oracle.C.corollary(inst["m"], int(ref["mu"]), sv[0] ** 2, 2)  # exact lambda_max, as the reference's SVD
    assert p["feasible"] == cor["feasible"] and abs(p["rho"] - cor["rho"]) <= 1e-12 * cor["rho"]
    assert abs(p["gamma"] - cor["gamma"]) <= 1e-11 * abs(cor["gamma"]) and len(p["bounds"]) == 3
    assert "rate_iteration" in p or not p["feasible"]  # lambda_min is known now
