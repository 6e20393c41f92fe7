"""Least-squares host logic (ref src/lsq.cpp:12-101) in the
CPU suite: optimal_params / critical_ratio and the augmented system are
BIT-IDENTICAL to the reference (oracle/_ref, the unmodified lsq.cpp), with
the reference's error behaviour; the cases follow ref tests/test_lsq.cpp.
The augmented solve itself runs on the device: tests/test_gpu_lsq.py."""
import math

import numpy as np
import pytest

import oracle

capi = pytest.importorskip("paper_1401_4780_b200.capi")
R = oracle.REF
needs_ref = pytest.mark.skipif(R is None, reason="oracle/_ref not built")


def host_of(e, m, n):
    return capi.HostCsr(m, n, e["row_ptr"], e["col_idx"], e["values"], e["row_norm"], normalized=e["normalized"])


def bits(a):
    return np.ascontiguousarray(a, dtype=np.float64).view(np.uint64)


@needs_ref
def test_optimal_params_and_critical_ratio_match_reference():
    # test_lsq.cpp:22-96
    assert capi.lsq_optimal_params(math.sqrt(2.0)) == R.optimal_params(math.sqrt(2.0))
    phi, zeta = capi.lsq_optimal_params(1.0)
    assert phi == 1.0 and abs(zeta - 0.70710678118654746) <= 1e-15
    rng = np.random.default_rng(0)
    for _ in range(200):
        sig, frob, m = rng.uniform(0.01, 3), rng.uniform(1, 100), int(rng.integers(1, 500))
        z, f = rng.uniform(0.01, 3), rng.uniform(0.01, 3)
        assert capi.lsq_critical_ratio(sig, frob, m, z, f) == R.critical_ratio(sig, frob, m, z, f)
    # the ratio peaks at the derived parameters (test_lsq.cpp:60-95)
    sigma, frob, m = 0.7, 30.0, 40
    phi_s, zeta_s = capi.lsq_optimal_params(sigma)
    zs = [zeta_s * 10 ** (-1 + 2 * k / 40) for k in range(41)]
    best = int(np.argmax([capi.lsq_critical_ratio(sigma, frob, m, z, phi_s) for z in zs]))
    assert abs(best - 20) <= 1
    fs = [10 ** (-1 + 2 * k / 40) for k in range(41)]
    best = int(np.argmax([capi.lsq_critical_ratio(sigma, frob, m, zeta_s, f) for f in fs]))
    assert abs(best - 20) <= 1
    for bad in (0.0, -1.0):
        with pytest.raises(capi.AsyrkError, match="NonPositiveSigma"):
            capi.lsq_optimal_params(bad)
    with pytest.raises(capi.AsyrkError, match="InvalidArgument"):
        capi.lsq_critical_ratio(0.7, 30.0, 0, 0.5, 1.0)


@needs_ref
@pytest.mark.parametrize("zeta,phi", [(0.5, 1.0), (0.37, 1.5), (2.0, 0.25), (1e-3, 7.0)])
def test_augment_bit_identical(instances, zeta, phi):
    for nm, inst in instances.items():
        Ar, br = R.build(inst["m"], inst["n"], np.repeat(np.arange(inst["m"]), np.diff(inst["row_ptr"])),
                         inst["col_idx"], inst["values"], True, inst["b"])
        e = Ar.export()
        try:
            ref = R.augment(Ar, br, zeta, phi)
        except oracle.OracleError as err:  # an instance with an empty column
            with pytest.raises(capi.AsyrkError) as ours:
                capi.lsq_augment(host_of(e, inst["m"], inst["n"]), br, zeta, phi)
            assert str(err).endswith(str(ours.value).split(": ", 1)[1]), nm
            continue
        got = capi.lsq_augment(host_of(e, inst["m"], inst["n"]), br, zeta, phi)
        ea, G = ref["a_tilde"].export(), got["a_tilde"]
        assert np.array_equal(ea["row_ptr"], G.row_ptr) and np.array_equal(ea["col_idx"], G.col_idx), nm
        assert np.array_equal(bits(ea["values"]), bits(G.values)), nm
        assert np.array_equal(bits(ea["row_norm"]), bits(G.row_norm)) and G.normalized, nm
        assert np.array_equal(bits(ref["b_tilde"]), bits(got["b_tilde"])), nm
        assert np.array_equal(bits(ref["row_scales"]), bits(got["row_scales"])), nm


def test_augment_block_structure():
    # test_lsq.cpp:98-131: identity(2), b = (1, 1), zeta = phi = 1
    I2 = capi.HostCsr(2, 2, [0, 1, 2], [0, 1], [1.0, 1.0])
    aug = capi.lsq_augment(I2, np.array([1.0, 1.0]), 1.0, 1.0)
    A = aug["a_tilde"]
    assert A.m == A.n == 4 and A.normalized
    D = np.zeros((4, 4))
    for i in range(4):
        for k in range(A.row_ptr[i], A.row_ptr[i + 1]):
            D[i, A.col_idx[k]] = A.values[k] * aug["row_scales"][i]
    want = np.array([[0, 0, 1, 0], [0, 0, 0, 1], [1, 0, -1, 0], [0, 1, 0, -1]], float)
    assert np.allclose(D, want, rtol=0, atol=1e-14)
    assert np.allclose(aug["b_tilde"], [1, 1, 0, 0], rtol=0, atol=1e-14)
    assert aug["b_tilde"][2] == 0.0 and aug["b_tilde"][3] == 0.0
    assert abs(float(np.sum(aug["row_scales"] ** 2)) - 6.0) <= 6e-13


@needs_ref
def test_augment_errors_match_reference():
    # test_lsq.cpp:133-138 (empty column) + the augment() argument checks
    Ar, br = R.build(2, 2, [0, 1], [0, 0], [1.0, 1.0], True, np.array([1.0, 1.0]))
    A = host_of(Ar.export(), 2, 2)
    cases = [(A, br, 0.5, 1.0, "ZeroColumn"), (A, br, 0.0, 1.0, "InvalidArgument"),
             (A, br, 0.5, -1.0, "InvalidArgument"), (A, br[:1], 0.5, 1.0, "DimensionMismatch")]
    for M, b, z, f, code in cases:
        with pytest.raises(capi.AsyrkError, match=code) as ours:
            capi.lsq_augment(M, b, z, f)
        if len(b) == 2:
            with pytest.raises(oracle.OracleError, match=code) as ref:
                R.augment(Ar, b, z, f)
            assert str(ref.value).endswith(str(ours.value).split(": ", 1)[1])
    raw = capi.HostCsr(2, 2, [0, 1, 2], [0, 1], [2.0, 1.0])
    with pytest.raises(capi.AsyrkError, match="NotNormalized"):
        capi.lsq_augment(raw, np.ones(2), 0.5, 1.0)


def test_lsq_golden_vectors_pin_the_reference(golden):
    # the committed lsq fixtures come from the reference lsq_solve; the
    # least-squares optimality of their x_ls is checked independently here
    for nm in sorted({k.split("/")[1] for k in golden.files if k.startswith("lsq/")}):
        p = f"lsq/{nm}/"
        m, n = golden[p + "shape"]
        D = np.zeros((m, n))
        rp, ci, v = golden[p + "row_ptr"], golden[p + "col_idx"], golden[p + "values"]
        for i in range(m):
            D[i, ci[rp[i]:rp[i + 1]]] = v[rp[i]:rp[i + 1]]
        x = golden[p + "x_ls"]
        g = np.linalg.norm(D.T @ (D @ x - golden[p + "b"]))
        assert abs(g - golden[p + "scal"][0]) <= 1e-9 + 1e-6 * g, nm
        if nm != "l30x12_explicit":  # (10 epochs: not converged by design)
            assert np.linalg.norm(x - np.linalg.lstsq(D, golden[p + "b"], rcond=None)[0]) <= 1e-6, nm


def test_dense_and_lsq_argument_errors_without_a_gpu():
    # checks that precede any device work (include/asyrk_dense.h): the dense SVD's
    # size cap, lsq_solve's sigma rules (lsq.cpp:110-129) and its input checks
    A, b, _ = capi.generate_fixed_theta(3000, 1500, 4, seed=2)  # 4.5e6 cells > SolutionProjector cap
    with pytest.raises(capi.AsyrkError, match="TooLarge"):
        capi.dense_svd(A, max_cells=1000)
    with pytest.raises(capi.AsyrkError, match="SigmaUnavailable"):
        capi.lsq_solve(A, b, max_epochs=1)
    with pytest.raises(capi.AsyrkError, match="NonPositiveSigma"):
        capi.lsq_solve(A, b, sigma_r=0.0, max_epochs=1)
    with pytest.raises(capi.AsyrkError, match="DimensionMismatch"):
        capi.lsq_solve(A, b[:-1], sigma_r=0.5, max_epochs=1)
    raw = capi.HostCsr(2, 2, [0, 1, 2], [0, 1], [2.0, 1.0])
    with pytest.raises(capi.AsyrkError, match="NotNormalized"):
        capi.lsq_solve(raw, np.ones(2), sigma_r=0.5, max_epochs=1)
