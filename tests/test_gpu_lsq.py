"""Device dense spectrum and least squares.

lsq_solve with a supplied sigma_r runs the reference's algorithm end to end
— augment (bit-identical, test_lsq.py) then rk_solve on the device's
deterministic worker — so x_ls, y, grad_norm and every record of the
augmented trace are BIT-IDENTICAL to the reference's lsq_solve
(tests/golden lsq/* from oracle/_ref). The dense spectrum is the device
one-sided Jacobi SVD; the reference's Eigen BDCSVD cannot be built here, so
it is checked against LAPACK (numpy) to 1e-12 relative in every singular
value, and the lsq paths that use it against the normal-equations solution
at the reference tests' 1e-6 bar (test_lsq.cpp:128-213, acceptance C7).
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

capi = pytest.importorskip("paper_1401_4780_b200.capi")


def golden_case(golden, nm):
    p = f"lsq/{nm}/"
    m, n = (int(v) for v in golden[p + "shape"])
    A = capi.HostCsr(m, n, golden[p + "row_ptr"], golden[p + "col_idx"], golden[p + "values"], golden[p + "row_norm"],
                     normalized=True)
    return p, A, golden[p + "b"]


def dense(A):
    D = np.zeros((A.m, A.n))
    for i in range(A.m):
        D[i, A.col_idx[A.row_ptr[i]:A.row_ptr[i + 1]]] = A.values[A.row_ptr[i]:A.row_ptr[i + 1]]
    return D


CASES = ["l60x30", "l60x30_shuffle", "l40x16_consistent", "l30x12_explicit", "l200x100_c7"]
KW = {"l60x30": dict(max_epochs=60000, target=1e-18, seed=3),
      "l60x30_shuffle": dict(max_epochs=300, target=0.0, seed=4, sampling=capi.RK_SHUFFLE),
      "l40x16_consistent": dict(max_epochs=40000, target=1e-20),
      "l30x12_explicit": dict(zeta=0.37, phi=1.5, max_epochs=10),
      "l200x100_c7": dict(max_epochs=200000, target=1e-16, seed=17)}


@pytest.mark.parametrize("nm", CASES)
def test_lsq_solve_bit_identical_to_reference(golden, nm):
    p, A, b = golden_case(golden, nm)
    r = capi.lsq_solve(A, b, sigma_r=float(golden[p + "sigma_r"][0]), **KW[nm])
    assert np.array_equal(r["x_ls"], golden[p + "x_ls"]), nm
    assert np.array_equal(r["y"], golden[p + "y"]), nm
    assert np.array_equal(np.array([r["grad_norm"], r["zeta"], r["phi"], r["sigma_r"]]), golden[p + "scal"]), nm
    assert np.array_equal(r["trace"]["r_sq"], golden[p + "r_sq"]), nm
    assert np.array_equal(r["trace"]["epoch_index"], golden[p + "epoch_index"]), nm


def test_dense_svd_matches_lapack(golden, instances):
    rng = np.random.default_rng(5)
    mats = [capi.HostCsr(inst["m"], inst["n"], inst["row_ptr"], inst["col_idx"], inst["values"])
            for inst in instances.values()]
    mats.append(golden_case(golden, "l200x100_c7")[1])
    # a wide matrix (m < n), a tall dense one and one with duplicated columns (rank-deficient)
    for m, n, dup in [(40, 90, False), (300, 120, False), (80, 30, True)]:
        D = rng.standard_normal((m, n))
        if dup:
            D[:, n // 2:] = D[:, :n - n // 2]
        rp = np.arange(m + 1) * n
        mats.append(capi.HostCsr(m, n, rp, np.tile(np.arange(n), m), D.ravel()))
    for A in mats:
        D = dense(A)
        s = np.linalg.svd(D, compute_uv=False)
        got = capi.dense_svd(A, vectors=True)
        assert np.allclose(got["sigma"][: got["rank"]], s[: got["rank"]], rtol=1e-12, atol=0), (A.m, A.n)
        assert got["rank"] == int(np.sum(s > 1e-10 * s[0])), (A.m, A.n)
        r = got["rank"]
        U, V = got["U"][:, :r], got["V"][:, :r]
        assert np.allclose(U.T @ U, np.eye(r), atol=1e-12) and np.allclose(V.T @ V, np.eye(r), atol=1e-12)
        assert np.allclose(U @ np.diag(got["sigma"][:r]) @ V.T, D, atol=1e-12 * s[0])
        sp = capi.dense_spectrum(A)
        assert sp["rank"] == r and sp["lambda_max"] == got["sigma"][0] ** 2
        assert sp["sigma_r"] == got["sigma"][r - 1] and sp["lambda_min"] == sp["sigma_r"] ** 2
        b = rng.standard_normal(A.m)
        x = capi.dense_lstsq(A, b)
        want = np.linalg.lstsq(D, b, rcond=1e-10)[0]
        assert np.linalg.norm(x - want) <= 1e-10 * max(1.0, np.linalg.norm(want)), (A.m, A.n)


def test_lsq_solve_default_sigma_recovers_normal_equations(golden):
    # test_lsq.cpp:128-176 with sigma_r from the device SVD (the reference's
    # dense-SVD branch), plus the substitution identities of the solution
    p, A, b = golden_case(golden, "l60x30")
    r = capi.lsq_solve(A, b, max_epochs=60000, target=1e-18, seed=3)
    D = dense(A)
    xl = np.linalg.lstsq(D, b, rcond=None)[0]
    assert np.linalg.norm(r["x_ls"] - xl) <= 1e-6 and r["grad_norm"] <= 1e-6
    assert r["phi"] == 1.0 and abs(r["zeta"] - r["sigma_r"] / np.sqrt(2.0)) <= 1e-12 * r["zeta"]
    assert abs(r["sigma_r"] - golden[p + "sigma_r"][0]) <= 1e-12 * r["sigma_r"]
    assert np.linalg.norm(D @ (r["zeta"] * r["x_ls"]) - r["zeta"] * r["y"]) <= 1e-5
    assert np.linalg.norm(D.T @ r["y"] - D.T @ b) <= 1e-5


def test_lsq_orthogonal_rhs_and_consistent_system(golden):
    # test_lsq.cpp:178-202: b orthogonal to range(A) -> x_ls = 0; consistent -> x*
    p, A, b = golden_case(golden, "l40x16_consistent")
    D = dense(A)
    w = np.cos(1.0 + np.arange(A.m))
    b_perp = w - D @ np.linalg.lstsq(D, w, rcond=None)[0]
    assert np.linalg.norm(b_perp) > 1e-6
    r = capi.lsq_solve(A, b_perp, max_epochs=40000, target=1e-20)
    assert np.linalg.norm(r["x_ls"]) <= 1e-6
    r = capi.lsq_solve(A, b, max_epochs=40000, target=1e-20)
    assert np.linalg.norm(r["x_ls"] - np.linalg.lstsq(D, b, rcond=None)[0]) <= 1e-6


def test_lsq_async_workers(golden):
    # the augmented system through the async warp workers (threads > 1)
    p, A, b = golden_case(golden, "l200x100_c7")
    D = dense(A)
    xl = np.linalg.lstsq(D, b, rcond=None)[0]
    r = capi.lsq_solve(A, b, sigma_r=float(golden[p + "sigma_r"][0]), max_epochs=200000, target=1e-18, seed=2,
                       threads=8)
    assert np.linalg.norm(r["x_ls"] - xl) <= 1e-6, np.linalg.norm(r["x_ls"] - xl)
    assert r["grad_norm"] <= 1e-6


def test_sigma_required_above_the_dense_cap():
    # test_lsq.cpp:204-224: 2500 x 1700, two shifted diagonals
    m, n = 2500, 1700
    rows = np.repeat(np.arange(m), 2)
    cols = np.stack([np.arange(m) % n, (np.arange(m) + 7) % n], 1).ravel()
    vals = np.tile([1.0, 0.5], m)
    order = np.lexsort((cols, rows))
    rows, cols, vals = rows[order], cols[order], vals[order]
    rp = np.concatenate([[0], np.cumsum(np.bincount(rows, minlength=m))])
    vals = vals / np.repeat(np.sqrt(np.add.reduceat(vals * vals, rp[:-1])), 2)
    A = capi.HostCsr(m, n, rp, cols, vals)
    assert A.normalized
    b = np.ones(m) / np.sqrt(1.25)
    with pytest.raises(capi.AsyrkError, match="SigmaUnavailable"):
        capi.lsq_solve(A, b, max_epochs=1)
    r = capi.lsq_solve(A, b, sigma_r=0.5, max_epochs=1)
    assert r["sigma_r"] == 0.5
    with pytest.raises(capi.AsyrkError, match="NonPositiveSigma"):
        capi.lsq_solve(A, b, sigma_r=-1.0, max_epochs=1)


def test_pybind_lsq_and_exact_stats(golden):
    import paper_1401_4780_b200 as asyrk
    p, A, b = golden_case(golden, "l60x30")
    rows = np.repeat(np.arange(A.m), np.diff(A.row_ptr))
    res = asyrk.lsq(A.m, A.n, rows.tolist(), A.col_idx.tolist(), A.values.tolist(), b.tolist(), epochs=40000,
                    target=1e-18)
    assert res["grad_norm"] <= 1e-5 and len(res["x_ls"]) == A.n and res["phi"] == 1.0
    st = asyrk.system_stats(A.m, A.n, rows.tolist(), A.col_idx.tolist(), A.values.tolist())
    s = np.linalg.svd(dense(A), compute_uv=False)
    assert abs(st["lambda_max"] - s[0] ** 2) <= 1e-12 * s[0] ** 2
    assert abs(st["sigma_r"] - s[-1]) <= 1e-12 * s[0] and abs(st["lambda_min"] - s[-1] ** 2) <= 1e-12 * s[0] ** 2
    sp = asyrk.step_params(A.m, A.n, rows.tolist(), A.col_idx.tolist(), A.values.tolist(), 2)
    assert "rate_iteration" in sp or not sp["feasible"]
