"""oracle — TEST INFRASTRUCTURE ONLY (the parity checker, never the product).

Two CPU checkers for the AsyRK hot path, both reached through ctypes:

* ``C`` — ``oracle/liboracle.so``, a plain-C restatement of the reference
  algorithm (``oracle/oracle.c``; every function cites the reference
  file:line it follows).
* ``REF`` — ``oracle/_ref/libasyrk_ref.so``, the UNMODIFIED reference sources
  (``/root/reference/proj/src``) compiled by ``oracle/Makefile`` with a flat C
  shim (``oracle/ref_shim.cpp``). It is built here; the prebuilt .so travels to
  the GPU box (git-ignored, not gpurun-ignored).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this package. The product package
(``paper_1401_4780_b200``) must never import it.
"""
from __future__ import annotations

import ctypes as C_
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_i64p = C_.POINTER(C_.c_int64)
_u64p = C_.POINTER(C_.c_uint64)
_f64p = C_.POINTER(C_.c_double)


class _Trace(C_.Structure):
    _fields_ = [
        ("cap", C_.c_int64),
        ("count", C_.c_int64),
        ("epoch_index", _i64p),
        ("r_sq", _f64p),
        ("grad_sq", _f64p),
        ("dist_sq", _f64p),
        ("wall", _f64p),
        ("updates", _i64p),
        ("final_x", _f64p),
    ]


class _Instr(C_.Structure):
    _fields_ = [
        ("row_updates", C_.c_int64),
        ("increments", C_.c_int64),
        ("max_abs_error", C_.c_double),
        ("tolerance", C_.c_double),
        ("consistent", C_.c_int32),
    ]


# ErrorCode ordinal + 1 (ref/include/asyrk/error.hpp:8-33)
ERROR_NAMES = [
    "IndexOutOfRange", "DuplicateEntry", "ZeroRow", "ZeroColumn", "NotNormalized",
    "DimensionMismatch", "PowerIterationDiverged", "NonFinite", "ComponentNotInSupport",
    "Inconsistent", "TooLarge", "InvalidRho", "MissingStats", "StepTooLarge", "ZeroLambdaMin",
    "InvalidGamma", "NonPositiveData", "InsufficientData", "NonPositiveSigma", "SigmaUnavailable",
    "InfeasibleSpec", "ThreadSpawnFailure", "IoError", "InvalidArgument",
]


class OracleError(ValueError):
    def __init__(self, code: int, msg: str = ""):
        self.code = code
        self.name = ERROR_NAMES[code - 1] if 1 <= code <= len(ERROR_NAMES) else f"code{code}"
        super().__init__(f"{self.name}: {msg}" if msg else self.name)


class _SimOut(C_.Structure):
    _fields_ = [("ev_cap", C_.c_int64), ("ev_count", C_.c_int64), ("ev_j", C_.POINTER(C_.c_int64)),
                ("ev_i", C_.POINTER(C_.c_int64)), ("ev_t", C_.POINTER(C_.c_int64)), ("ev_k", C_.POINTER(C_.c_int64)),
                ("ev_step", C_.POINTER(C_.c_double)), ("hist_cap", C_.c_int64), ("hist_rows", C_.c_int64),
                ("history", C_.POINTER(C_.c_double)), ("probe_cap", C_.c_int64), ("probe_count", C_.c_int64),
                ("probe_iteration", C_.POINTER(C_.c_int64)), ("probe_r_sq", C_.POINTER(C_.c_double))]


class _RefSimOut(C_.Structure):
    """ref_sim_out (ref_shim.cpp): the trace, then the _SimOut fields."""

    _fields_ = [("trace", _Trace)] + _SimOut._fields_

    def __init__(self, t, o):
        super().__init__()
        self.trace = t
        for f, _ in _SimOut._fields_:
            setattr(self, f, getattr(o, f))


DELAY_KINDS = {"fixed": 0, "uniform_random": 1, "max_staleness": 2}
SIM_VARIANTS = {"single_component": 0, "full_row": 1}


def _sim_buffers(n, iterations, tau, probe_every, max_events):
    ev = {k: np.zeros(max(max_events, 1), np.int64) for k in ["j", "i", "t", "k"]}
    ev["step"] = np.zeros(max(max_events, 1))
    hist = np.zeros((tau + 1, n))
    npr = iterations // probe_every + 1 if probe_every > 0 else 1
    pit, prs = np.zeros(npr, np.int64), np.zeros(npr)
    o = _SimOut(max_events, 0, _p(ev["j"], _i64p), _p(ev["i"], _i64p), _p(ev["t"], _i64p), _p(ev["k"], _i64p),
                _p(ev["step"], _f64p), tau + 1, 0, _p(hist, _f64p), npr, 0, _p(pit, _i64p), _p(prs, _f64p))
    return o, ev, hist, pit, prs


def _sim_result(trace, o, ev, hist, pit, prs):
    ne = min(o.ev_count, o.ev_cap)
    trace["events"] = {k: v[:ne].copy() for k, v in ev.items()}
    trace["history"] = hist[:o.hist_rows].copy()
    trace["probe_iteration"] = pit[:o.probe_count].copy()
    trace["probe_r_sq"] = prs[:o.probe_count].copy()
    return trace


def _stats_dict(mu, nu, d, theta):
    return dict(mu=mu, nu=nu, delta=d[0], alpha=d[1], lambda_max=d[2], frob_sq=d[3], l_max=d[4], l_res=d[5],
                theta=theta)


def _p(a, t):
    return a.ctypes.data_as(t) if a is not None else None


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _i64(a):
    return np.ascontiguousarray(a, dtype=np.int64)


@dataclass
class Csr:
    lib: "_Lib"
    handle: object
    m: int
    n: int

    def export(self):
        return self.lib._export(self)

    def __del__(self):
        try:
            self.lib._free(self)
        except Exception:
            pass


@dataclass
class Instance:
    """Host CSR arrays of a generated instance (the fields of capi.HostCsr)."""

    m: int
    n: int
    row_ptr: np.ndarray
    col_idx: np.ndarray
    values: np.ndarray
    row_norm: np.ndarray
    normalized: bool

    @property
    def nnz(self):
        return int(self.row_ptr[-1])


class _Lib:
    kind = "?"

    def _trace(self, n, cap):
        bufs = dict(
            epoch_index=np.zeros(cap, np.int64), r_sq=np.zeros(cap), grad_sq=np.zeros(cap),
            dist_sq=np.zeros(cap), wall=np.zeros(cap), updates=np.zeros(cap, np.int64),
            final_x=np.zeros(n),
        )
        t = _Trace(cap, 0, _p(bufs["epoch_index"], _i64p), _p(bufs["r_sq"], _f64p),
                   _p(bufs["grad_sq"], _f64p), _p(bufs["dist_sq"], _f64p), _p(bufs["wall"], _f64p),
                   _p(bufs["updates"], _i64p), _p(bufs["final_x"], _f64p))
        return t, bufs

    @staticmethod
    def _trace_dict(t, bufs, has_dist):
        k = min(t.count, t.cap)
        d = dict(
            epoch_index=bufs["epoch_index"][:k].copy(), r_sq=bufs["r_sq"][:k].copy(),
            grad_sq=bufs["grad_sq"][:k].copy(), wall_seconds=bufs["wall"][:k].copy(),
            updates_applied=bufs["updates"][:k].copy(), final_x=bufs["final_x"],
        )
        if has_dist:
            d["dist_sq"] = bufs["dist_sq"][:k].copy()
        return d


class _RefLib(_Lib):
    """The reference library itself (oracle/_ref/libasyrk_ref.so)."""

    kind = "reference"

    def __init__(self, path):
        L = C_.CDLL(path)
        self.L = L
        L.ref_last_error.restype = C_.c_char_p
        L.ref_csr_build.restype = C_.c_void_p
        L.ref_csr_build.argtypes = [C_.c_int64, C_.c_int64, C_.c_int64, _i64p, _i64p, _f64p, C_.c_int,
                                    _f64p, _f64p, C_.POINTER(C_.c_int)]
        L.ref_csr_free.argtypes = [C_.c_void_p]
        L.ref_csr_nnz.restype = C_.c_int64
        L.ref_csr_nnz.argtypes = [C_.c_void_p]
        L.ref_csr_export.argtypes = [C_.c_void_p, _i64p, _i64p, _f64p, _f64p, C_.POINTER(C_.c_int)]
        L.ref_gen_sparse_gaussian.restype = C_.c_void_p
        L.ref_gen_sparse_gaussian.argtypes = [C_.c_int64, C_.c_int64, C_.c_double, C_.c_uint64, _f64p, _f64p,
                                              C_.POINTER(C_.c_int)]
        L.ref_rk_solve.argtypes = [C_.c_void_p, _f64p, _f64p, C_.c_int64, C_.c_double, C_.c_uint64, C_.c_int,
                                   _f64p, C_.POINTER(_Trace)]
        L.ref_solve_parallel.argtypes = [C_.c_void_p, _f64p, _f64p, C_.c_int64, C_.c_double, C_.c_int64,
                                         C_.c_double, C_.c_int, C_.c_int, C_.c_uint64, C_.c_int64, _f64p,
                                         C_.POINTER(_Trace), C_.POINTER(_Instr)]
        L.ref_residuals.argtypes = [C_.c_void_p, _f64p, _f64p, _f64p, _f64p, _f64p]
        L.ref_multiply.argtypes = [C_.c_void_p, _f64p, _f64p]
        L.ref_multiply_transpose.argtypes = [C_.c_void_p, _f64p, _f64p]
        L.ref_power_iteration.argtypes = [C_.c_void_p, C_.c_double, C_.c_int64, _f64p]
        L.ref_stats.argtypes = [C_.c_void_p, C_.c_double, _i64p, _i64p, _f64p, _f64p, _f64p]
        L.ref_stats_full.argtypes = [C_.c_void_p, C_.c_double, C_.c_int64, _i64p, _i64p, _f64p, _i64p]
        L.ref_simulate.argtypes = [C_.c_void_p, _f64p, _f64p, C_.c_double, C_.c_int64, C_.c_int, C_.c_int64,
                                   C_.c_uint64, C_.c_int, C_.c_int64, C_.c_int, C_.c_int64, C_.c_void_p]
        L.ref_monte_carlo.argtypes = [C_.c_void_p, _f64p, _f64p, C_.c_double, C_.c_int64, C_.c_int, C_.c_int64,
                                      C_.c_int64, C_.c_uint64, C_.c_int, _f64p, _f64p]
        L.ref_rate_fit.argtypes = [_f64p, C_.c_int64, C_.c_double, _f64p, _f64p]
        L.ref_csr_dims.argtypes = [C_.c_void_p, _i64p, _i64p]
        L.ref_write_mtx.argtypes = [C_.c_void_p, C_.c_char_p]
        L.ref_read_mtx.restype = C_.c_void_p
        L.ref_read_mtx.argtypes = [C_.c_char_p, C_.POINTER(C_.c_int)]
        L.ref_write_vector.argtypes = [C_.c_char_p, _f64p, C_.c_int64]
        L.ref_read_vector.argtypes = [C_.c_char_p, _f64p, C_.c_int64, _i64p]
        L.ref_write_instance.argtypes = [C_.c_void_p, _f64p, _f64p, C_.c_int64, C_.c_int64, C_.c_double, C_.c_uint64,
                                         C_.c_int, C_.c_double, C_.c_char_p]
        L.ref_read_instance.restype = C_.c_void_p
        L.ref_read_instance.argtypes = [C_.c_char_p, _f64p, C_.c_int64, _f64p, C_.c_int64, C_.POINTER(C_.c_int), _f64p,
                                        C_.POINTER(C_.c_int)]
        L.ref_corollary.argtypes = [C_.c_int64, C_.c_int64, C_.c_double, C_.c_double, C_.c_int64, _f64p, _f64p,
                                    _f64p, C_.POINTER(C_.c_int)]
        L.ref_stream_raw.argtypes = [C_.c_uint64, C_.c_uint64, C_.c_int64, _u64p]
        L.ref_uniform_below_seq.argtypes = [C_.c_uint64, C_.c_uint64, C_.c_uint64, C_.c_int64, _u64p]
        L.ref_normal_seq.argtypes = [C_.c_uint64, C_.c_uint64, C_.c_int64, _f64p]
        L.ref_shuffle_seq.argtypes = [C_.c_uint64, C_.c_uint64, C_.c_int64, C_.c_int64, _i64p]
        L.ref_alias_sample_seq.argtypes = [_f64p, C_.c_int64, C_.c_uint64, C_.c_int64, _i64p]
        L.ref_rk_step.argtypes = [C_.c_void_p, _f64p, _f64p, C_.c_int64, _f64p]
        L.ref_asyrk_update.argtypes = [C_.c_void_p, _f64p, C_.c_int64, C_.c_int64, C_.c_double, _f64p, _f64p]
        L.ref_gen_instance.restype = C_.c_void_p
        L.ref_gen_instance.argtypes = [C_.c_int64, C_.c_int64, C_.c_double, C_.c_uint64, C_.c_int, C_.c_double,
                                       _f64p, _f64p, C_.POINTER(C_.c_int), C_.POINTER(C_.c_int)]
        L.ref_optimal_params.argtypes = [C_.c_double, _f64p, _f64p]
        L.ref_critical_ratio.argtypes = [C_.c_double, C_.c_double, C_.c_int64, C_.c_double, C_.c_double, _f64p]
        L.ref_augment.restype = C_.c_void_p
        L.ref_augment.argtypes = [C_.c_void_p, _f64p, C_.c_double, C_.c_double, _f64p, _f64p, C_.POINTER(C_.c_int)]
        L.ref_lsq_solve.argtypes = [C_.c_void_p, _f64p, C_.c_double, C_.c_double, C_.c_double, C_.c_int64,
                                    C_.c_double, C_.c_uint64, C_.c_int, _f64p, _f64p, _f64p, C_.POINTER(_Trace)]

    def trace_roundtrip(self, jsonl):
        """The reference's Trace::from_jsonl then to_jsonl / to_csv (trace.cpp:33-112)."""
        L = self.L
        L.ref_trace_roundtrip.argtypes = [C_.c_char_p, C_.c_char_p, C_.c_int64, C_.c_char_p, C_.c_int64, _i64p, _i64p]
        cap = 4 * len(jsonl) + 4096
        bj, bc = C_.create_string_buffer(cap), C_.create_string_buffer(cap)
        lj, lc = C_.c_int64(), C_.c_int64()
        self._check(L.ref_trace_roundtrip(jsonl.encode(), bj, cap, bc, cap, C_.byref(lj), C_.byref(lc)))
        assert lj.value <= cap and lc.value <= cap
        return bj.raw[:lj.value].decode(), bc.raw[:lc.value].decode()

    def _check(self, st):
        if st:
            raise OracleError(st, self.L.ref_last_error().decode())

    # -- matrices
    def build(self, m, n, rows, cols, vals, normalize=True, b=None):
        rows, cols, vals = _i64(rows), _i64(cols), _f64(vals)
        bin_ = _f64(b) if b is not None else None
        bout = np.zeros(m) if b is not None else None
        st = C_.c_int(0)
        h = self.L.ref_csr_build(m, n, len(vals), _p(rows, _i64p), _p(cols, _i64p), _p(vals, _f64p),
                                 1 if normalize else 0, _p(bin_, _f64p), _p(bout, _f64p), C_.byref(st))
        self._check(st.value)
        return Csr(self, h, m, n), bout

    def gen_sparse_gaussian(self, m, n, delta, seed):
        b, xs = np.zeros(m), np.zeros(n)
        st = C_.c_int(0)
        h = self.L.ref_gen_sparse_gaussian(m, n, delta, seed, _p(b, _f64p), _p(xs, _f64p), C_.byref(st))
        self._check(st.value)
        return Csr(self, h, m, n), b, xs

    def gen_instance(self, m, n, delta, seed, consistent=True, noise_level=0.0):
        """gen_sparse_gaussian with the full GenSpec (datagen.cpp:13-137)."""
        b, xs = np.zeros(m), np.zeros(n)
        st, has = C_.c_int(0), C_.c_int(0)
        h = self.L.ref_gen_instance(m, n, delta, seed, int(consistent), noise_level, _p(b, _f64p), _p(xs, _f64p),
                                    C_.byref(has), C_.byref(st))
        self._check(st.value)
        return Csr(self, h, m, n), b, (xs if has.value else None)

    # -- least squares (lsq.cpp:12-170)
    def optimal_params(self, sigma_r):
        phi, zeta = C_.c_double(), C_.c_double()
        self._check(self.L.ref_optimal_params(sigma_r, C_.byref(phi), C_.byref(zeta)))
        return phi.value, zeta.value

    def critical_ratio(self, sigma_r, frob_sq, m, zeta, phi):
        r = C_.c_double()
        self._check(self.L.ref_critical_ratio(sigma_r, frob_sq, m, zeta, phi, C_.byref(r)))
        return r.value

    def augment(self, A, b, zeta, phi):
        N = A.m + A.n
        bt, rs = np.zeros(N), np.zeros(N)
        st = C_.c_int(0)
        h = self.L.ref_augment(A.handle, _p(_f64(b), _f64p), zeta, phi, _p(bt, _f64p), _p(rs, _f64p), C_.byref(st))
        self._check(st.value)
        return dict(a_tilde=Csr(self, h, N, N), b_tilde=bt, row_scales=rs)

    def lsq_solve(self, A, b, sigma_r, zeta=0.0, phi=0.0, max_epochs=5000, target=0.0, seed=0, sampling="uniform",
                  cap=100000):
        s = {"uniform": 0, "norm": 1, "norm_proportional": 1, "shuffle": 2}[sampling]
        x_ls, y, scal = np.zeros(A.n), np.zeros(A.m), np.zeros(4)
        t, bufs = self._trace(A.n + A.m, min(cap, max_epochs + 2))
        self._check(self.L.ref_lsq_solve(A.handle, _p(_f64(b), _f64p), zeta, phi, sigma_r, max_epochs, target, seed,
                                         s, _p(x_ls, _f64p), _p(y, _f64p), _p(scal, _f64p), C_.byref(t)))
        return dict(x_ls=x_ls, y=y, grad_norm=scal[0], zeta=scal[1], phi=scal[2], sigma_r=scal[3],
                    trace=self._trace_dict(t, bufs, False))

    def _export(self, A):
        nnz = self.L.ref_csr_nnz(A.handle)
        rp, ci, v, rn = np.zeros(A.m + 1, np.int64), np.zeros(nnz, np.int64), np.zeros(nnz), np.zeros(A.m)
        norm = C_.c_int(0)
        self.L.ref_csr_export(A.handle, _p(rp, _i64p), _p(ci, _i64p), _p(v, _f64p), _p(rn, _f64p), C_.byref(norm))
        return dict(row_ptr=rp, col_idx=ci, values=v, row_norm=rn, normalized=bool(norm.value))

    def _free(self, A):
        if A.handle:
            self.L.ref_csr_free(A.handle)
            A.handle = None

    # -- solvers
    def rk_solve(self, A, b, x0, epochs, target=0.0, seed=0, sampling="uniform", xstar=None, cap=100000):
        s = {"uniform": 0, "norm": 1, "norm_proportional": 1, "shuffle": 2}[sampling]
        b, x0 = _f64(b), _f64(x0)
        xs = _f64(xstar) if xstar is not None else None
        t, bufs = self._trace(A.n, cap)
        self._check(self.L.ref_rk_solve(A.handle, _p(b, _f64p), _p(x0, _f64p), epochs, target, seed, s,
                                        _p(xs, _f64p), C_.byref(t)))
        return self._trace_dict(t, bufs, xs is not None)

    def solve_parallel(self, A, b, x0, threads=1, gamma=1.0, epochs=100, target=0.0, variant="full_row",
                       sampling="slice_shuffle", seed=0, snapshot_interval=1, xstar=None, instrument=False,
                       cap=100000):
        v = 1 if variant in ("full_row", "full-row") else 0
        s = 1 if sampling in ("slice_shuffle", "slice") else 0
        b, x0 = _f64(b), _f64(x0)
        xs = _f64(xstar) if xstar is not None else None
        t, bufs = self._trace(A.n, cap)
        rep = _Instr()
        self._check(self.L.ref_solve_parallel(A.handle, _p(b, _f64p), _p(x0, _f64p), threads, gamma, epochs,
                                              target, v, s, seed, snapshot_interval, _p(xs, _f64p), C_.byref(t),
                                              C_.byref(rep) if instrument else None))
        d = self._trace_dict(t, bufs, xs is not None)
        if instrument:
            d["instrument"] = dict(row_updates=rep.row_updates, increments=rep.increments,
                                   max_abs_error=rep.max_abs_error, tolerance=rep.tolerance,
                                   consistent=bool(rep.consistent))
        return d

    def residuals(self, A, x, b):
        x, b = _f64(x), _f64(b)
        r = np.zeros(A.m)
        rs, gs = C_.c_double(), C_.c_double()
        self._check(self.L.ref_residuals(A.handle, _p(x, _f64p), _p(b, _f64p), _p(r, _f64p), C_.byref(rs),
                                         C_.byref(gs)))
        return rs.value, gs.value

    def multiply(self, A, x):
        x = _f64(x)
        y = np.zeros(A.m)
        self._check(self.L.ref_multiply(A.handle, _p(x, _f64p), _p(y, _f64p)))
        return y

    def multiply_transpose(self, A, x):
        x = _f64(x)
        y = np.zeros(A.n)
        self._check(self.L.ref_multiply_transpose(A.handle, _p(x, _f64p), _p(y, _f64p)))
        return y

    def power_iteration(self, A, tol=1e-6, max_iters=200000):
        lam = C_.c_double()
        self._check(self.L.ref_power_iteration(A.handle, tol, max_iters, C_.byref(lam)))
        return lam.value

    def stats(self, A, tol=1e-9):
        mu, nu = C_.c_int64(), C_.c_int64()
        al, lm, fs = C_.c_double(), C_.c_double(), C_.c_double()
        self._check(self.L.ref_stats(A.handle, tol, C_.byref(mu), C_.byref(nu), C_.byref(al), C_.byref(lm),
                                     C_.byref(fs)))
        return dict(mu=mu.value, nu=nu.value, alpha=al.value, lambda_max=lm.value, frob_sq=fs.value)

    def simulate(self, A, b, x0, gamma, tau, delay, iterations, seed, variant, probe_every=0, probe_r_sq=False,
                 max_events=0):
        """simulate (delay_sim.cpp:71-228): trace + events + history + probes."""
        b, x0 = _f64(b), _f64(x0)
        o, ev, hist, pit, prs = _sim_buffers(A.n, iterations, tau, probe_every, max_events)
        t, bufs = self._trace(A.n, iterations // A.m + 3)
        ro = _RefSimOut(t, o)
        self._check(self.L.ref_simulate(A.handle, _p(b, _f64p), _p(x0, _f64p), gamma, tau, DELAY_KINDS[delay],
                                        iterations, seed, SIM_VARIANTS[variant], probe_every, int(probe_r_sq),
                                        max_events, C_.byref(ro)))
        return _sim_result(self._trace_dict(ro.trace, bufs, False), ro, ev, hist, pit, prs)

    def monte_carlo(self, A, b, x0, gamma, tau, delay, iterations, runs, base_seed, variant="single_component"):
        b, x0 = _f64(b), _f64(x0)
        mean, ratios = np.zeros(iterations + 1), np.zeros(iterations)
        self._check(self.L.ref_monte_carlo(A.handle, _p(b, _f64p), _p(x0, _f64p), gamma, tau, DELAY_KINDS[delay],
                                           iterations, runs, base_seed, SIM_VARIANTS[variant], _p(mean, _f64p),
                                           _p(ratios, _f64p)))
        return dict(mean_r_sq=mean, ratios=ratios)

    def write_mtx(self, A, path):
        self._check(self.L.ref_write_mtx(A.handle, path.encode()))

    def read_mtx(self, path):
        st = C_.c_int(0)
        h = self.L.ref_read_mtx(path.encode(), C_.byref(st))
        self._check(st.value)
        return self._csr_from_handle(h)

    def _csr_from_handle(self, h):
        m, n = C_.c_int64(), C_.c_int64()
        self.L.ref_csr_dims(h, C_.byref(m), C_.byref(n))
        return Csr(self, h, m.value, n.value)

    def write_vector(self, path, v):
        v = _f64(v)
        self._check(self.L.ref_write_vector(path.encode(), _p(v, _f64p), len(v)))

    def read_vector(self, path, cap=1 << 22):
        out = np.zeros(cap)
        cnt = C_.c_int64()
        self._check(self.L.ref_read_vector(path.encode(), _p(out, _f64p), cap, C_.byref(cnt)))
        return out[:cnt.value].copy()

    def write_instance(self, A, b, xs, spec, path):
        b = _f64(b)
        xs = _f64(xs) if xs is not None else None
        self._check(self.L.ref_write_instance(A.handle, _p(b, _f64p), _p(xs, _f64p), spec["m"], spec["n"],
                                              spec["delta"], spec["seed"], int(spec["consistent"]),
                                              spec["noise_level"], path.encode()))

    def read_instance(self, path, m_cap=1 << 20, n_cap=1 << 20):
        b, xs, meta = np.zeros(m_cap), np.zeros(n_cap), np.zeros(6)
        has, st = C_.c_int(0), C_.c_int(0)
        h = self.L.ref_read_instance(path.encode(), _p(b, _f64p), m_cap, _p(xs, _f64p), n_cap, C_.byref(has),
                                     _p(meta, _f64p), C_.byref(st))
        self._check(st.value)
        m, n = int(meta[0]), int(meta[1])
        A = Csr(self, h, m, n)
        return dict(A=A, b=b[:m].copy(), x_star=xs[:n].copy() if has.value else None,
                    spec=dict(m=m, n=n, delta=meta[2], seed=int(meta[3]), consistent=bool(meta[4]),
                              noise_level=meta[5]))

    def rate_fit(self, y, stride=1.0):
        y = _f64(y)
        sl, r2 = C_.c_double(), C_.c_double()
        self._check(self.L.ref_rate_fit(_p(y, _f64p), len(y), stride, C_.byref(sl), C_.byref(r2)))
        return dict(slope=sl.value, r2=r2.value)

    def stats_full(self, A, tol=1e-9, max_iters=200000):
        """compute_stats(exact_spectral=false): every scalar field and theta."""
        mu, nu = C_.c_int64(), C_.c_int64()
        d = np.zeros(6)
        th = np.zeros(A.m, np.int64)
        self._check(self.L.ref_stats_full(A.handle, tol, max_iters, C_.byref(mu), C_.byref(nu), _p(d, _f64p),
                                          _p(th, _i64p)))
        return _stats_dict(mu.value, nu.value, d, th)

    def corollary(self, m, mu, alpha, lambda_max, tau):
        rho, psi, gam = C_.c_double(), C_.c_double(), C_.c_double()
        f = C_.c_int()
        self._check(self.L.ref_corollary(m, mu, alpha, lambda_max, tau, C_.byref(rho), C_.byref(psi),
                                         C_.byref(gam), C_.byref(f)))
        return dict(rho=rho.value, psi=psi.value, gamma=gam.value, feasible=bool(f.value))

    def stream_raw(self, seed, stream, count):
        out = np.zeros(count, np.uint64)
        self.L.ref_stream_raw(seed, stream, count, _p(out, _u64p))
        return out

    def uniform_below_seq(self, seed, stream, n, count):
        out = np.zeros(count, np.uint64)
        self.L.ref_uniform_below_seq(seed, stream, n, count, _p(out, _u64p))
        return out

    def normal_seq(self, seed, stream, count):
        out = np.zeros(count)
        self.L.ref_normal_seq(seed, stream, count, _p(out, _f64p))
        return out

    def shuffle_seq(self, seed, stream, n, rounds):
        out = np.zeros(n * rounds, np.int64)
        self.L.ref_shuffle_seq(seed, stream, n, rounds, _p(out, _i64p))
        return out.reshape(rounds, n)

    def alias_sample_seq(self, w, seed, count):
        w = _f64(w)
        out = np.zeros(count, np.int64)
        self._check(self.L.ref_alias_sample_seq(_p(w, _f64p), len(w), seed, count, _p(out, _i64p)))
        return out

    def rk_step(self, A, b, x, i):
        b, x = _f64(b), _f64(x)
        out = np.zeros(A.n)
        self._check(self.L.ref_rk_step(A.handle, _p(b, _f64p), _p(x, _f64p), i, _p(out, _f64p)))
        return out

    def asyrk_update(self, A, b, i, t, gamma, x):
        b, x = _f64(b), _f64(x)
        out = C_.c_double()
        self._check(self.L.ref_asyrk_update(A.handle, _p(b, _f64p), i, t, gamma, _p(x, _f64p), C_.byref(out)))
        return out.value


class _OracleLib(_Lib):
    """The plain-C restatement (oracle/liboracle.so)."""

    kind = "port"

    def __init__(self, path):
        L = C_.CDLL(path)
        self.L = L
        L.oc_csr_from_triplets.restype = C_.c_void_p
        L.oc_csr_from_triplets.argtypes = [C_.c_int64, C_.c_int64, C_.c_int64, _i64p, _i64p, _f64p,
                                           C_.POINTER(C_.c_int)]
        L.oc_csr_from_arrays.restype = C_.c_void_p
        L.oc_csr_from_arrays.argtypes = [C_.c_int64, C_.c_int64, _i64p, _i64p, _f64p]
        L.oc_csr_free.argtypes = [C_.c_void_p]
        L.oc_csr_nnz.restype = C_.c_int64
        L.oc_csr_nnz.argtypes = [C_.c_void_p]
        L.oc_normalize_rows.argtypes = [C_.c_void_p, _f64p]
        L.oc_csr_export.argtypes = [C_.c_void_p, _i64p, _i64p, _f64p, _f64p]
        L.oc_rk_solve.argtypes = [C_.c_void_p, _f64p, _f64p, C_.c_int64, C_.c_double, C_.c_uint64, C_.c_int,
                                  _f64p, C_.POINTER(_Trace)]
        L.oc_solve_single.argtypes = [C_.c_void_p, _f64p, _f64p, C_.c_double, C_.c_int64, C_.c_double, C_.c_int,
                                      C_.c_int, C_.c_uint64, C_.c_int64, _f64p, C_.POINTER(_Trace),
                                      C_.POINTER(_Instr)]
        L.oc_residuals.argtypes = [C_.c_void_p, _f64p, _f64p, _f64p, _f64p]
        L.oc_multiply.argtypes = [C_.c_void_p, _f64p, _f64p]
        L.oc_multiply_transpose.argtypes = [C_.c_void_p, _f64p, _f64p]
        L.oc_power_iteration.argtypes = [C_.c_void_p, C_.c_double, C_.c_int64, _f64p, _i64p]
        L.oc_corollary.argtypes = [C_.c_int64, C_.c_int64, C_.c_double, C_.c_int64, _f64p, _f64p, _f64p,
                                   C_.POINTER(C_.c_int)]
        L.oc_stream_raw.argtypes = [C_.c_uint64, C_.c_uint64, C_.c_int64, _u64p]
        L.oc_uniform_below_seq.argtypes = [C_.c_uint64, C_.c_uint64, C_.c_uint64, C_.c_int64, _u64p]
        L.oc_normal_seq.argtypes = [C_.c_uint64, C_.c_uint64, C_.c_int64, _f64p]
        L.oc_shuffle_seq.argtypes = [C_.c_uint64, C_.c_uint64, C_.c_int64, C_.c_int64, _i64p]
        L.oc_alias_sample_seq.argtypes = [_f64p, C_.c_int64, C_.c_uint64, C_.c_int64, _i64p]
        L.oc_alias_sample_seq.restype = C_.c_int
        L.oc_rk_step.argtypes = [C_.c_void_p, _f64p, _f64p, C_.c_int64, _f64p]
        L.oc_compute_stats.argtypes = [C_.c_void_p, C_.c_double, C_.c_int64, _i64p, _i64p, _f64p, _i64p, _i64p]
        L.oc_simulate.argtypes = [C_.c_void_p, _f64p, _f64p, C_.c_double, C_.c_int64, C_.c_int, C_.c_int64,
                                  C_.c_uint64, C_.c_int, C_.c_int64, C_.c_int, C_.c_int64, C_.POINTER(_Trace),
                                  C_.POINTER(_SimOut)]
        L.oc_monte_carlo.argtypes = [C_.c_void_p, _f64p, _f64p, C_.c_double, C_.c_int64, C_.c_int, C_.c_int64,
                                     C_.c_int64, C_.c_uint64, C_.c_int, _f64p, _f64p]
        L.oc_rate_fit.argtypes = [_f64p, C_.c_int64, C_.c_double, _f64p, _f64p]
        L.oc_generate_fixed_theta.argtypes = [C_.c_int64, C_.c_int64, C_.c_int64, C_.c_uint64, C_.c_int32,
                                              C_.c_double, C_.c_int64, C_.c_int32, _i64p, _i64p, _f64p, _f64p,
                                              _f64p, _f64p, C_.POINTER(C_.c_int32)]
        L.oc_generate_fixed_theta.restype = C_.c_int

    @staticmethod
    def _check(st):
        if st:
            raise OracleError(st)

    def generate_fixed_theta(self, m, n, theta, seed, dist="normal", scale_decades=0.0, k=1, threads=0):
        """The benchmark instance generator restated in C (oracle/workload.c), so the
        reference arm builds its instance without the product library. Returns
        (Instance, b, x_star) with the arrays of capi.generate_fixed_theta."""
        nnz = m * theta
        rp = np.zeros(m + 1, np.int64)
        ci = np.zeros(nnz, np.int64)
        v = np.zeros(nnz)
        rn = np.zeros(m)
        b = np.zeros(m * k)
        xs = np.zeros(n * k)
        norm = C_.c_int32(0)
        self._check(self.L.oc_generate_fixed_theta(m, n, theta, seed, 1 if dist == "uniform" else 0, scale_decades,
                                                   k, threads, _p(rp, _i64p), _p(ci, _i64p), _p(v, _f64p),
                                                   _p(rn, _f64p), _p(b, _f64p), _p(xs, _f64p), C_.byref(norm)))
        A = Instance(m, n, rp, ci, v, rn, bool(norm.value))
        if k > 1:
            return A, b.reshape(m, k), xs.reshape(n, k)
        return A, b, xs

    def build(self, m, n, rows, cols, vals, normalize=True, b=None):
        rows, cols, vals = _i64(rows), _i64(cols), _f64(vals)
        st = C_.c_int(0)
        h = self.L.oc_csr_from_triplets(m, n, len(vals), _p(rows, _i64p), _p(cols, _i64p), _p(vals, _f64p),
                                        C_.byref(st))
        self._check(st.value)
        bout = _f64(b).copy() if b is not None else None
        if normalize:
            self._check(self.L.oc_normalize_rows(h, _p(bout, _f64p)))
        return Csr(self, h, m, n), bout

    def from_arrays(self, m, n, row_ptr, col_idx, values):
        rp, ci, v = _i64(row_ptr), _i64(col_idx), _f64(values)
        h = self.L.oc_csr_from_arrays(m, n, _p(rp, _i64p), _p(ci, _i64p), _p(v, _f64p))
        return Csr(self, h, m, n)

    def _export(self, A):
        nnz = self.L.oc_csr_nnz(A.handle)
        rp, ci, v, rn = np.zeros(A.m + 1, np.int64), np.zeros(nnz, np.int64), np.zeros(nnz), np.zeros(A.m)
        self.L.oc_csr_export(A.handle, _p(rp, _i64p), _p(ci, _i64p), _p(v, _f64p), _p(rn, _f64p))
        return dict(row_ptr=rp, col_idx=ci, values=v, row_norm=rn)

    def _free(self, A):
        if A.handle:
            self.L.oc_csr_free(A.handle)
            A.handle = None

    def rk_solve(self, A, b, x0, epochs, target=0.0, seed=0, sampling="uniform", xstar=None, cap=100000):
        s = {"uniform": 0, "norm": 1, "norm_proportional": 1, "shuffle": 2}[sampling]
        b, x0 = _f64(b), _f64(x0)
        xs = _f64(xstar) if xstar is not None else None
        t, bufs = self._trace(A.n, cap)
        self._check(self.L.oc_rk_solve(A.handle, _p(b, _f64p), _p(x0, _f64p), epochs, target, seed, s,
                                       _p(xs, _f64p), C_.byref(t)))
        return self._trace_dict(t, bufs, xs is not None)

    def solve_parallel(self, A, b, x0, threads=1, gamma=1.0, epochs=100, target=0.0, variant="full_row",
                       sampling="slice_shuffle", seed=0, snapshot_interval=1, xstar=None, instrument=False,
                       cap=100000):
        if threads != 1:
            raise NotImplementedError("the C restatement covers the deterministic threads == 1 path")
        v = 1 if variant in ("full_row", "full-row") else 0
        s = 1 if sampling in ("slice_shuffle", "slice") else 0
        b, x0 = _f64(b), _f64(x0)
        xs = _f64(xstar) if xstar is not None else None
        t, bufs = self._trace(A.n, cap)
        rep = _Instr()
        self._check(self.L.oc_solve_single(A.handle, _p(b, _f64p), _p(x0, _f64p), gamma, epochs, target, v, s,
                                           seed, snapshot_interval, _p(xs, _f64p), C_.byref(t),
                                           C_.byref(rep) if instrument else None))
        d = self._trace_dict(t, bufs, xs is not None)
        if instrument:
            d["instrument"] = dict(row_updates=rep.row_updates, increments=rep.increments,
                                   max_abs_error=rep.max_abs_error, tolerance=rep.tolerance,
                                   consistent=bool(rep.consistent))
        return d

    def residuals(self, A, x, b):
        x, b = _f64(x), _f64(b)
        rs, gs = C_.c_double(), C_.c_double()
        self.L.oc_residuals(A.handle, _p(x, _f64p), _p(b, _f64p), C_.byref(rs), C_.byref(gs))
        return rs.value, gs.value

    def multiply(self, A, x):
        x = _f64(x)
        y = np.zeros(A.m)
        self.L.oc_multiply(A.handle, _p(x, _f64p), _p(y, _f64p))
        return y

    def multiply_transpose(self, A, x):
        x = _f64(x)
        y = np.zeros(A.n)
        self.L.oc_multiply_transpose(A.handle, _p(x, _f64p), _p(y, _f64p))
        return y

    def power_iteration(self, A, tol=1e-6, max_iters=200000, return_iters=False):
        lam, it = C_.c_double(), C_.c_int64()
        self._check(self.L.oc_power_iteration(A.handle, tol, max_iters, C_.byref(lam), C_.byref(it)))
        return (lam.value, it.value) if return_iters else lam.value

    def simulate(self, A, b, x0, gamma, tau, delay, iterations, seed, variant, probe_every=0, probe_r_sq=False,
                 max_events=0):
        b, x0 = _f64(b), _f64(x0)
        o, ev, hist, pit, prs = _sim_buffers(A.n, iterations, tau, probe_every, max_events)
        t, bufs = self._trace(A.n, iterations // A.m + 3)
        self._check(self.L.oc_simulate(A.handle, _p(b, _f64p), _p(x0, _f64p), gamma, tau, DELAY_KINDS[delay],
                                       iterations, seed, SIM_VARIANTS[variant], probe_every, int(probe_r_sq),
                                       max_events, C_.byref(t), C_.byref(o)))
        return _sim_result(self._trace_dict(t, bufs, False), o, ev, hist, pit, prs)

    def monte_carlo(self, A, b, x0, gamma, tau, delay, iterations, runs, base_seed, variant="single_component"):
        b, x0 = _f64(b), _f64(x0)
        mean, ratios = np.zeros(iterations + 1), np.zeros(iterations)
        self._check(self.L.oc_monte_carlo(A.handle, _p(b, _f64p), _p(x0, _f64p), gamma, tau, DELAY_KINDS[delay],
                                          iterations, runs, base_seed, SIM_VARIANTS[variant], _p(mean, _f64p),
                                          _p(ratios, _f64p)))
        return dict(mean_r_sq=mean, ratios=ratios)

    def rate_fit(self, y, stride=1.0):
        y = _f64(y)
        sl, r2 = C_.c_double(), C_.c_double()
        self._check(self.L.oc_rate_fit(_p(y, _f64p), len(y), stride, C_.byref(sl), C_.byref(r2)))
        return dict(slope=sl.value, r2=r2.value)

    def stats_full(self, A, tol=1e-9, max_iters=200000):
        """oc_compute_stats: the same fields as REF.stats_full."""
        mu, nu, zc = C_.c_int64(), C_.c_int64(), C_.c_int64(-1)
        d = np.zeros(6)
        th = np.zeros(A.m, np.int64)
        self._check(self.L.oc_compute_stats(A.handle, tol, max_iters, C_.byref(mu), C_.byref(nu), _p(d, _f64p),
                                            _p(th, _i64p), C_.byref(zc)))
        return _stats_dict(mu.value, nu.value, d, th)

    def corollary(self, m, mu, lambda_max, tau):
        rho, psi, gam = C_.c_double(), C_.c_double(), C_.c_double()
        f = C_.c_int()
        self.L.oc_corollary(m, mu, lambda_max, tau, C_.byref(rho), C_.byref(psi), C_.byref(gam), C_.byref(f))
        return dict(rho=rho.value, psi=psi.value, gamma=gam.value, feasible=bool(f.value))

    def stream_raw(self, seed, stream, count):
        out = np.zeros(count, np.uint64)
        self.L.oc_stream_raw(seed, stream, count, _p(out, _u64p))
        return out

    def uniform_below_seq(self, seed, stream, n, count):
        out = np.zeros(count, np.uint64)
        self.L.oc_uniform_below_seq(seed, stream, n, count, _p(out, _u64p))
        return out

    def normal_seq(self, seed, stream, count):
        out = np.zeros(count)
        self.L.oc_normal_seq(seed, stream, count, _p(out, _f64p))
        return out

    def shuffle_seq(self, seed, stream, n, rounds):
        out = np.zeros(n * rounds, np.int64)
        self.L.oc_shuffle_seq(seed, stream, n, rounds, _p(out, _i64p))
        return out.reshape(rounds, n)

    def alias_sample_seq(self, w, seed, count):
        w = _f64(w)
        out = np.zeros(count, np.int64)
        self._check(self.L.oc_alias_sample_seq(_p(w, _f64p), len(w), seed, count, _p(out, _i64p)))
        return out

    def rk_step(self, A, b, x, i):
        b, x = _f64(b), _f64(x)
        out = np.zeros(A.n)
        self._check(self.L.oc_rk_step(A.handle, _p(b, _f64p), _p(x, _f64p), i, _p(out, _f64p)))
        return out


def build_oracle():
    """Compile oracle/liboracle.so (and oracle/_ref when /root/reference exists)."""
    import subprocess

    subprocess.run(["make", "-s", "-C", _HERE, "all"], check=True)


def _load(cls, rel):
    path = os.path.join(_HERE, rel)
    if not os.path.exists(path):
        return None
    return cls(path)


C = _load(_OracleLib, "liboracle.so")
REF = _load(_RefLib, os.path.join("_ref", "libasyrk_ref.so"))
