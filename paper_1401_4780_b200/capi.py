"""ctypes view of the C ABI (include/asyrk_cuda.h, include/asyrk_datagen.h).

This is the binding a ctypes-based host would write against the drop-in
library (INTEGRATION.md shows the same for cgo/JNI-style hosts). bench.py and
the GPU parity tests drive the hot path through it. Loading fails loudly if
``libasyrk_b200.so`` has not been built; there is no fallback.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# (ASYRK_LIB: an alternative build of the same library, for A/B experiments)
LIB_PATH = os.environ.get("ASYRK_LIB") or os.path.join(_HERE, "libasyrk_b200.so")

_i64p = C.POINTER(C.c_int64)
_f64p = C.POINTER(C.c_double)
_i32p = C.POINTER(C.c_int32)

ERROR_NAMES = [
    "IndexOutOfRange", "DuplicateEntry", "ZeroRow", "ZeroColumn", "NotNormalized",
    "DimensionMismatch", "PowerIterationDiverged", "NonFinite", "ComponentNotInSupport",
    "Inconsistent", "TooLarge", "InvalidRho", "MissingStats", "StepTooLarge", "ZeroLambdaMin",
    "InvalidGamma", "NonPositiveData", "InsufficientData", "NonPositiveSigma", "SigmaUnavailable",
    "InfeasibleSpec", "ThreadSpawnFailure", "IoError", "InvalidArgument",
]

F64, F32, F32X64 = 0, 1, 2
SINGLE_COMPONENT, FULL_ROW = 0, 1
WITH_REPLACEMENT, SLICE_SHUFFLE, NORM_PROPORTIONAL = 0, 1, 2
RK_UNIFORM, RK_NORM_PROPORTIONAL, RK_SHUFFLE = 0, 1, 2


class CsrView(C.Structure):
    _fields_ = [("m", C.c_int64), ("n", C.c_int64), ("nnz", C.c_int64), ("row_ptr", _i64p), ("col_idx", _i64p),
                ("values", _f64p), ("row_norm", _f64p), ("normalized", C.c_int32)]


class RunConfig(C.Structure):
    _fields_ = [("threads", C.c_int64), ("gamma", C.c_double), ("epochs", C.c_int64), ("target_r_sq", C.c_double),
                ("variant", C.c_int32), ("sampling", C.c_int32), ("seed", C.c_uint64),
                ("snapshot_interval", C.c_int64), ("x_star", _f64p), ("precision", C.c_int32),
                ("allow_unnormalized", C.c_int32), ("record_every_boundary", C.c_int32),
                ("det_reassociate", C.c_int32)]


class RkConfig(C.Structure):
    _fields_ = [("max_epochs", C.c_int64), ("target_r_sq", C.c_double), ("seed", C.c_uint64),
                ("sampling", C.c_int32), ("x_star", _f64p), ("det_reassociate", C.c_int32)]


class TraceOut(C.Structure):
    _fields_ = [("cap", C.c_int64), ("count", C.c_int64), ("epoch_index", _i64p), ("r_sq", _f64p),
                ("grad_sq", _f64p), ("dist_sq", _f64p), ("wall_seconds", _f64p), ("updates_applied", _i64p),
                ("final_x", _f64p)]


class InstrumentOut(C.Structure):
    _fields_ = [("row_updates", C.c_int64), ("increments", C.c_int64), ("max_abs_error", C.c_double),
                ("tolerance", C.c_double), ("consistent", C.c_int32)]


class SolveStats(C.Structure):
    _fields_ = [("solve_ms", C.c_double), ("worker_ms", C.c_double), ("monitor_ms", C.c_double),
                ("worker_launches", C.c_int64), ("monitor_launches", C.c_int64), ("kernel_launches", C.c_int64),
                ("projections", C.c_int64), ("resident_warps", C.c_int32), ("warps", C.c_int32)]


class StatsOut(C.Structure):
    """asyrk_stats_out (include/asyrk_cuda.h; SystemStats, ref stats.hpp:18-37)."""

    _fields_ = [("m", C.c_int64), ("n", C.c_int64), ("delta", C.c_double), ("mu", C.c_int64), ("nu", C.c_int64),
                ("alpha", C.c_double), ("lambda_max", C.c_double), ("frob_sq", C.c_double), ("l_max", C.c_double),
                ("l_res", C.c_double), ("power_iterations", C.c_int64), ("theta", C.POINTER(C.c_int64))]


def _stats_result(o, theta):
    d = {f: getattr(o, f) for f, _ in StatsOut._fields_ if f != "theta"}
    d["theta"] = theta
    return d


class SimConfig(C.Structure):
    """asyrk_sim_config (include/asyrk_cuda.h; DelayModel + StepParams.gamma + SimOptions)."""

    _fields_ = [("gamma", C.c_double), ("tau", C.c_int64), ("delay", C.c_int32), ("variant", C.c_int32),
                ("iterations", C.c_int64), ("seed", C.c_uint64), ("probe_every", C.c_int64),
                ("probe_r_sq", C.c_int32), ("probe_dist_sq", C.c_int32), ("max_events", C.c_int64),
                ("dist_point", _f64p)]


class SimOut(C.Structure):
    _fields_ = [("trace", TraceOut), ("ev_cap", C.c_int64), ("ev_count", C.c_int64), ("ev_j", _i64p),
                ("ev_i", _i64p), ("ev_t", _i64p), ("ev_k", _i64p), ("ev_step", _f64p), ("history_cap", C.c_int64),
                ("history_rows", C.c_int64), ("history", _f64p), ("probe_cap", C.c_int64),
                ("probe_count", C.c_int64), ("probe_iteration", _i64p), ("probe_r_sq", _f64p),
                ("probe_dist_sq", _f64p)]


DELAY = {"fixed": 0, "uniform_random": 1, "max_staleness": 2}
SIM_VARIANT = {"single_component": 0, "full_row": 1}


def _sim_config(gamma, tau, delay, iterations, seed, variant, probe_every=0, probe_r_sq=False, probe_dist_sq=False,
                max_events=0, dist_point=None):
    """dist_point: the SolutionProjector's solution point A^+ b (e.g. dense_lstsq(A, b)), which
    adds dist_sq to the records and enables probe_dist_sq."""
    dp = np.ascontiguousarray(dist_point, dtype=np.float64) if dist_point is not None else None
    c = SimConfig(gamma, tau, DELAY[delay], SIM_VARIANT[variant], iterations, seed, probe_every,
                  int(probe_r_sq), int(probe_dist_sq), max_events, _ptr(dp, _f64p))
    c._keep = dp  # the pointer's owner lives as long as the config
    return c


def _sim_call(fn, n, m, cfg: SimConfig):
    """Run asyrk_(system_)simulate through fn(out) and collect SimRun-like dicts."""
    K = max(cfg.iterations, 0)
    tr = _Trace(n, K // max(m, 1) + 3)
    ne = max(min(cfg.max_events, K), 1)
    ev = {k: np.zeros(ne, np.int64) for k in ["j", "i", "t", "k"]}
    ev["step"] = np.zeros(ne)
    hist = np.zeros((max(cfg.tau, 0) + 1, n))
    npr = K // cfg.probe_every + 1 if cfg.probe_every > 0 else 1
    pit, prs, pds = np.zeros(npr, np.int64), np.zeros(npr), np.zeros(npr)
    o = SimOut(tr.out, min(cfg.max_events, K), 0, _ptr(ev["j"], _i64p), _ptr(ev["i"], _i64p), _ptr(ev["t"], _i64p),
               _ptr(ev["k"], _i64p), _ptr(ev["step"], _f64p), hist.shape[0], 0, _ptr(hist, _f64p), npr, 0,
               _ptr(pit, _i64p), _ptr(prs, _f64p), _ptr(pds, _f64p))
    check(fn(o))
    tr.out = o.trace
    d = tr.result(bool(cfg.dist_point))
    nev = min(o.ev_count, o.ev_cap)
    d["events"] = {k: v[:nev].copy() for k, v in ev.items()}
    d["history"] = hist[:o.history_rows].copy()
    d["probe_iteration"] = pit[:o.probe_count].copy()
    d["probe_r_sq"] = prs[:o.probe_count].copy() if cfg.probe_r_sq else np.zeros(0)
    if cfg.probe_dist_sq:
        d["probe_dist_sq"] = pds[:o.probe_count].copy()
    return d


class HostCsrInfo(C.Structure):
    _fields_ = [("m", C.c_int64), ("n", C.c_int64), ("nnz", C.c_int64), ("normalized", C.c_int32)]


class InstanceMeta(C.Structure):
    """asyrk_instance_meta (include/asyrk_io.h; ref GenSpec, datagen.hpp:11-18)."""

    _fields_ = [("m", C.c_int64), ("n", C.c_int64), ("delta", C.c_double), ("seed", C.c_uint64),
                ("consistent", C.c_int32), ("noise_level", C.c_double), ("has_x_star", C.c_int32)]


class Spectrum(C.Structure):
    """asyrk_spectrum (include/asyrk_dense.h; Spectrum, ref dense.hpp:15-20)."""

    _fields_ = [("lambda_max", C.c_double), ("lambda_min", C.c_double), ("sigma_r", C.c_double),
                ("rank", C.c_int32)]


class LsqConfig(C.Structure):
    """asyrk_lsq_config (include/asyrk_dense.h; LsqConfig, ref lsq.hpp:40-50 + device solver choice)."""

    _fields_ = [("zeta", C.c_double), ("phi", C.c_double), ("has_sigma_r", C.c_int32), ("sigma_r", C.c_double),
                ("max_epochs", C.c_int64), ("target_r_sq", C.c_double), ("seed", C.c_uint64),
                ("sampling", C.c_int32), ("threads", C.c_int64), ("gamma", C.c_double)]


class LsqOut(C.Structure):
    """asyrk_lsq_out (include/asyrk_dense.h; LsqResult, ref lsq.hpp:52-60)."""

    _fields_ = [("x_ls", _f64p), ("y", _f64p), ("grad_norm", C.c_double), ("zeta", C.c_double),
                ("phi", C.c_double), ("sigma_r", C.c_double), ("trace", TraceOut)]


class AsyrkError(ValueError):
    def __init__(self, status: int, msg: str):
        self.status = status
        self.name = ERROR_NAMES[status - 1] if 1 <= status <= len(ERROR_NAMES) else f"status{status}"
        super().__init__(f"{self.name}: {msg}")


def _ptr(a, t):
    return a.ctypes.data_as(t) if a is not None else None


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is not built; run __graft_entry__.build() (make -C "
                              "paper_1401_4780_b200/csrc)")
        L = C.CDLL(LIB_PATH)
        L.asyrk_last_error.restype = C.c_char_p
        L.asyrk_set_device.argtypes = [C.c_int32]
        sp = C.c_void_p
        L.asyrk_system_create.argtypes = [C.POINTER(CsrView), _f64p, C.c_int32, C.c_void_p, C.POINTER(sp)]
        L.asyrk_system_destroy.argtypes = [sp]
        L.asyrk_system_solve.argtypes = [sp, _f64p, C.POINTER(RunConfig), C.POINTER(TraceOut),
                                         C.POINTER(InstrumentOut)]
        L.asyrk_system_rk_solve.argtypes = [sp, _f64p, C.POINTER(RkConfig), C.POINTER(TraceOut)]
        L.asyrk_system_residuals.argtypes = [sp, _f64p, _f64p, _f64p]
        L.asyrk_system_set_rhs.argtypes = [sp, _f64p]
        L.asyrk_system_multiply.argtypes = [sp, _f64p, _f64p]
        L.asyrk_system_multiply_transpose.argtypes = [sp, _f64p, _f64p]
        L.asyrk_system_power_iteration.argtypes = [sp, C.c_double, C.c_int64, _f64p, _i64p]
        L.asyrk_system_last_stats.argtypes = [sp, C.POINTER(SolveStats)]
        L.asyrk_system_max_resident_warps.argtypes = [sp, C.c_int32, _i32p]
        L.asyrk_system_compute_stats.argtypes = [sp, C.c_double, C.c_int64, C.POINTER(StatsOut)]
        L.asyrk_compute_stats.argtypes = [C.POINTER(CsrView), C.c_double, C.c_int64, C.POINTER(StatsOut)]
        L.asyrk_simulate.argtypes = [C.POINTER(CsrView), _f64p, _f64p, C.POINTER(SimConfig), C.POINTER(SimOut)]
        L.asyrk_system_simulate.argtypes = [sp, _f64p, C.POINTER(SimConfig), C.POINTER(SimOut)]
        L.asyrk_monte_carlo_ratios.argtypes = [C.POINTER(CsrView), _f64p, _f64p, C.POINTER(SimConfig), C.c_int64,
                                               _f64p, _f64p]
        L.asyrk_system_monte_carlo_ratios.argtypes = [sp, _f64p, C.POINTER(SimConfig), C.c_int64, _f64p, _f64p]
        L.asyrk_rate_fit.argtypes = [_f64p, C.c_int64, C.c_double, _f64p, _f64p]
        L.asyrk_read_matrix_market.argtypes = [C.c_char_p, C.POINTER(sp), C.POINTER(HostCsrInfo)]
        L.asyrk_write_matrix_market.argtypes = [C.c_char_p, C.POINTER(CsrView)]
        L.asyrk_read_csr_cache.argtypes = [C.c_char_p, C.POINTER(sp), C.POINTER(HostCsrInfo)]
        L.asyrk_write_csr_cache.argtypes = [C.c_char_p, C.POINTER(CsrView)]
        L.asyrk_host_csr_copy.argtypes = [sp, _i64p, _i64p, _f64p, _f64p]
        L.asyrk_host_csr_free.argtypes = [sp]
        L.asyrk_host_csr_get_info.argtypes = [sp, C.POINTER(HostCsrInfo)]
        L.asyrk_read_vector.argtypes = [C.c_char_p, C.POINTER(_f64p), _i64p]
        L.asyrk_write_vector.argtypes = [C.c_char_p, _f64p, C.c_int64]
        L.asyrk_free.argtypes = [C.c_void_p]
        L.asyrk_write_instance.argtypes = [C.c_char_p, C.POINTER(CsrView), _f64p, _f64p, C.POINTER(InstanceMeta)]
        L.asyrk_read_instance.argtypes = [C.c_char_p, C.POINTER(sp), C.POINTER(_f64p), C.POINTER(_f64p),
                                          C.POINTER(InstanceMeta)]
        L.asyrk_dense_svd.argtypes = [C.POINTER(CsrView), C.c_int64, _f64p, _f64p, _f64p, C.POINTER(C.c_int32),
                                      C.POINTER(C.c_int32)]
        L.asyrk_dense_spectrum.argtypes = [C.POINTER(CsrView), C.POINTER(Spectrum)]
        L.asyrk_dense_lstsq.argtypes = [C.POINTER(CsrView), _f64p, _f64p]
        L.asyrk_lsq_optimal_params.argtypes = [C.c_double, _f64p, _f64p]
        L.asyrk_lsq_critical_ratio.argtypes = [C.c_double, C.c_double, C.c_int64, C.c_double, C.c_double, _f64p]
        L.asyrk_lsq_augment.argtypes = [C.POINTER(CsrView), _f64p, C.c_double, C.c_double, C.POINTER(sp), _f64p,
                                        _f64p]
        L.asyrk_lsq_solve.argtypes = [C.POINTER(CsrView), _f64p, C.POINTER(LsqConfig), C.POINTER(LsqOut)]
        L.asyrk_solve_parallel.argtypes = [C.POINTER(CsrView), _f64p, _f64p, C.POINTER(RunConfig),
                                           C.POINTER(TraceOut), C.POINTER(InstrumentOut)]
        L.asyrk_rk_solve.argtypes = [C.POINTER(CsrView), _f64p, _f64p, C.POINTER(RkConfig), C.POINTER(TraceOut)]
        L.asyrk_residuals.argtypes = [C.POINTER(CsrView), _f64p, _f64p, _f64p, _f64p]
        L.asyrk_power_iteration_lambda_max.argtypes = [C.POINTER(CsrView), C.c_double, C.c_int64, _f64p]
        L.asyrk_sweep_threads.argtypes = [C.POINTER(CsrView), _f64p, _f64p, C.POINTER(RunConfig), _i64p, C.c_int64,
                                          _f64p, _i64p, _f64p, _f64p]
        _f32p = C.POINTER(C.c_float)
        L.asyrk_mrhs_create.argtypes = [C.POINTER(CsrView), _f32p, C.c_int64, C.c_int64, C.c_int64, C.c_void_p,
                                        C.POINTER(sp)]
        L.asyrk_mrhs_destroy.argtypes = [sp]
        L.asyrk_mrhs_begin.argtypes = [sp, C.POINTER(RunConfig), _f32p, _f64p]
        L.asyrk_mrhs_norms.argtypes = [sp, C.POINTER(C.c_void_p)]
        L.asyrk_mrhs_commit.argtypes = [sp, C.c_int32]
        L.asyrk_mrhs_step.argtypes = [sp]
        L.asyrk_mrhs_stopped.argtypes = [sp, _i32p]
        L.asyrk_mrhs_finish.argtypes = [sp, C.POINTER(TraceOut), _f32p]
        L.asyrk_mrhs_solve.argtypes = [sp, C.POINTER(RunConfig), _f32p, _f64p, C.POINTER(TraceOut), _f32p]
        L.asyrk_mrhs_last_stats.argtypes = [sp, C.POINTER(SolveStats)]
        L.asyrk_mrhs_due.argtypes = [sp, _i32p]
        L.asyrk_mrhs_max_resident_warps.argtypes = [sp, _i32p]
        L.asyrk_mrhs_microbench_xside.argtypes = [sp, C.c_int32, C.c_int64, _f64p, _f64p]
        L.asyrk_microbench_xside_mrhs.argtypes = [C.c_int64, C.c_int32, C.c_int32, C.c_int32, C.c_int64, _f64p, _f64p]
        L.asyrk_monitor_schedule_next.argtypes = [C.c_double, C.c_int32, C.c_int64, _i64p, _f64p, C.c_int64, _i64p]
        L.asyrk_system_rk_solve_multi.argtypes = [sp, _f64p, C.c_int64, _f64p, C.POINTER(RkConfig), _f64p,
                                                  C.POINTER(TraceOut)]
        L.asyrk_system_microbench_xside.argtypes = [sp, C.c_int32, C.c_int64, C.c_int32, _f64p, _f64p]
        L.asyrk_system_sample_rows.argtypes = [sp, C.c_int32, C.c_uint64, C.c_int64, C.c_int64, C.c_int64, _i32p]
        L.asyrk_nccl_available.argtypes = [_i32p]
        L.asyrk_nccl_get_unique_id.argtypes = [C.c_char_p]
        L.asyrk_nccl_comm_init_rank.argtypes = [C.POINTER(C.c_void_p), C.c_int32, C.c_char_p, C.c_int32]
        L.asyrk_nccl_comm_destroy.argtypes = [C.c_void_p]
        L.asyrk_mrhs_solve_nccl.argtypes = [sp, C.POINTER(RunConfig), C.c_void_p, _f32p, _f64p, C.POINTER(TraceOut),
                                            _f32p]
        L.asyrk_mrhs_solve_devices.argtypes = [C.POINTER(CsrView), _f32p, C.c_int64, _i32p, C.c_int32,
                                               C.POINTER(RunConfig), _f32p, _f64p, C.POINTER(TraceOut), _f32p,
                                               C.POINTER(SolveStats)]
        L.asyrk_microbench_xside.argtypes = [C.c_int64, C.c_int32, C.c_int32, C.c_int32, C.c_int64, C.c_int32,
                                             _f64p, _f64p]
        L.asyrk_generate_fixed_theta.argtypes = [C.c_int64, C.c_int64, C.c_int64, C.c_uint64, C.c_int32, C.c_double,
                                                 C.c_int64, C.c_int32, _i64p, _i64p, _f64p, _f64p, _f64p, _f64p,
                                                 _i32p]
        _lib = L
    return _lib


# every symbol include/asyrk_cuda.h and include/asyrk_datagen.h declare
EXPORTED = [
    "asyrk_last_error", "asyrk_abi_version", "asyrk_set_device", "asyrk_solve_parallel", "asyrk_rk_solve", "asyrk_residuals",
    "asyrk_power_iteration_lambda_max", "asyrk_sweep_threads", "asyrk_system_create", "asyrk_system_destroy",
    "asyrk_system_solve", "asyrk_system_rk_solve", "asyrk_system_residuals", "asyrk_system_set_rhs",
    "asyrk_system_multiply", "asyrk_system_multiply_transpose", "asyrk_system_power_iteration",
    "asyrk_system_last_stats", "asyrk_system_max_resident_warps", "asyrk_generate_fixed_theta",
    "asyrk_microbench_xside", "asyrk_mrhs_create", "asyrk_mrhs_destroy", "asyrk_mrhs_begin", "asyrk_mrhs_norms",
    "asyrk_mrhs_commit", "asyrk_mrhs_step", "asyrk_mrhs_stopped", "asyrk_mrhs_finish", "asyrk_mrhs_solve",
    "asyrk_mrhs_last_stats", "asyrk_mrhs_due", "asyrk_mrhs_max_resident_warps", "asyrk_mrhs_microbench_xside", "asyrk_microbench_xside_mrhs", "asyrk_monitor_schedule_next", "asyrk_system_rk_solve_multi", "asyrk_system_microbench_xside", "asyrk_system_sample_rows", "asyrk_nccl_available", "asyrk_nccl_get_unique_id",
    "asyrk_nccl_comm_init_rank", "asyrk_nccl_comm_destroy", "asyrk_mrhs_solve_nccl", "asyrk_mrhs_solve_devices",
    "asyrk_compute_stats", "asyrk_system_compute_stats", "asyrk_simulate",
    "asyrk_system_simulate", "asyrk_monte_carlo_ratios", "asyrk_system_monte_carlo_ratios", "asyrk_rate_fit",
    "asyrk_read_matrix_market", "asyrk_write_matrix_market", "asyrk_read_csr_cache", "asyrk_write_csr_cache",
    "asyrk_host_csr_copy", "asyrk_host_csr_free", "asyrk_host_csr_get_info", "asyrk_read_vector", "asyrk_write_vector", "asyrk_free",
    "asyrk_write_instance", "asyrk_read_instance", "asyrk_dense_svd", "asyrk_dense_spectrum", "asyrk_dense_lstsq",
    "asyrk_lsq_optimal_params", "asyrk_lsq_critical_ratio", "asyrk_lsq_augment", "asyrk_lsq_solve",
]


class MultiRHS:
    """Device-resident multi-RHS shard (asyrk_mrhs_*): A replicated, columns [c0, c1) of B/X."""

    def __init__(self, A: "HostCsr", B, c0, c1, stream=None):
        B = np.ascontiguousarray(B, dtype=np.float32)
        if B.ndim != 2 or B.shape[0] != A.m:
            raise AsyrkError(6, f"B has shape {B.shape}, expected ({A.m}, k)")
        self.m, self.n = A.m, A.n
        self.k_total = B.shape[1]
        self.c0, self.c1 = c0, c1
        h = C.c_void_p()
        check(lib().asyrk_mrhs_create(C.byref(A.view()), B.ctypes.data_as(C.POINTER(C.c_float)), self.k_total, c0,
                                      c1, C.c_void_p(stream) if stream else None, C.byref(h)))
        self.h = h

    def close(self):
        if getattr(self, "h", None):
            lib().asyrk_mrhs_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def begin(self, X0=None, X_star=None, **cfg):
        self._cfg = _run_config(**cfg)
        self._x0 = _mat(X0, (self.n, self.k_total), np.float32, "X0") if X0 is not None else None
        self._xs = _mat(X_star, (self.n, self.k_total), np.float64, "X_star") if X_star is not None else None
        check(lib().asyrk_mrhs_begin(self.h, C.byref(self._cfg),
                                     self._x0.ctypes.data_as(C.POINTER(C.c_float)) if self._x0 is not None else None,
                                     _ptr(self._xs, _f64p)))
        self._cap = max(self._cfg.epochs, 0) // max(self._cfg.snapshot_interval, 1) + 2

    def norms_ptr(self):
        p = C.c_void_p()
        check(lib().asyrk_mrhs_norms(self.h, C.byref(p)))
        return p.value

    def commit(self, advance):
        check(lib().asyrk_mrhs_commit(self.h, 1 if advance else 0))

    def step(self):
        check(lib().asyrk_mrhs_step(self.h))

    def max_resident_warps(self):
        w = C.c_int32()
        check(lib().asyrk_mrhs_max_resident_warps(self.h, C.byref(w)))
        return w.value

    def microbench_xside(self, warps, proj_per_warp=64):
        """R_x of this shard's pattern on its own X (asyrk_mrhs_microbench_xside): row projections/s."""
        rate, ms = C.c_double(), C.c_double()
        check(lib().asyrk_mrhs_microbench_xside(self.h, warps, proj_per_warp, C.byref(rate), C.byref(ms)))
        return rate.value

    def due(self):
        """True when the last begin/step ended at an evaluated boundary (all-reduce the norms, then commit)."""
        d = C.c_int32()
        check(lib().asyrk_mrhs_due(self.h, C.byref(d)))
        return bool(d.value)

    def stopped(self):
        s = C.c_int32()
        check(lib().asyrk_mrhs_stopped(self.h, C.byref(s)))
        return bool(s.value)

    def finish(self):
        tr = _Trace(0, self._cap, want_x=False)
        X = np.zeros((self.n, self.c1 - self.c0), np.float32)
        check(lib().asyrk_mrhs_finish(self.h, C.byref(tr.out), X.ctypes.data_as(C.POINTER(C.c_float))))
        d = tr.result(self._xs is not None)
        d["X"] = X
        return d

    def solve(self, X0=None, X_star=None, want_x=True, **cfg):
        c = _run_config(**cfg)
        cap = max(c.epochs, 0) // max(c.snapshot_interval, 1) + 2
        tr = _Trace(0, cap, want_x=False)
        X = np.zeros((self.n, self.c1 - self.c0), np.float32) if want_x else None
        x0 = _mat(X0, (self.n, self.k_total), np.float32, "X0") if X0 is not None else None
        xs = _mat(X_star, (self.n, self.k_total), np.float64, "X_star") if X_star is not None else None
        check(lib().asyrk_mrhs_solve(self.h, C.byref(c), x0.ctypes.data_as(C.POINTER(C.c_float)) if x0 is not None
                                     else None, _ptr(xs, _f64p), C.byref(tr.out), _ptr(X, C.POINTER(C.c_float))))
        d = tr.result(xs is not None)
        d["X"] = X
        return d

    def solve_nccl(self, comm, X0=None, X_star=None, want_x=True, **cfg):
        """This rank's shard of a sharded solve, the loop in C++ with one ncclAllReduce of the
        shard norms per evaluated boundary (asyrk_mrhs_solve_nccl); comm from NcclComm."""
        c = _run_config(**cfg)
        cap = max(c.epochs, 0) // max(c.snapshot_interval, 1) + 2
        tr = _Trace(0, cap, want_x=False)
        X = np.zeros((self.n, self.c1 - self.c0), np.float32) if want_x else None
        x0 = _mat(X0, (self.n, self.k_total), np.float32, "X0") if X0 is not None else None
        xs = _mat(X_star, (self.n, self.k_total), np.float64, "X_star") if X_star is not None else None
        check(lib().asyrk_mrhs_solve_nccl(self.h, C.byref(c), C.c_void_p(comm.handle),
                                          x0.ctypes.data_as(C.POINTER(C.c_float)) if x0 is not None else None,
                                          _ptr(xs, _f64p), C.byref(tr.out), _ptr(X, C.POINTER(C.c_float))))
        d = tr.result(xs is not None)
        d["X"] = X
        return d

    def stats(self):
        s = SolveStats()
        check(lib().asyrk_mrhs_last_stats(self.h, C.byref(s)))
        return {f: getattr(s, f) for f, _ in SolveStats._fields_}


NCCL_UNIQUE_ID_BYTES = 128


def nccl_version():
    """NCCL version code of the libnccl.so.2 the library resolves at run time (raises if none)."""
    v = C.c_int32()
    check(lib().asyrk_nccl_available(C.byref(v)))
    return v.value


def nccl_unique_id():
    buf = C.create_string_buffer(NCCL_UNIQUE_ID_BYTES)
    check(lib().asyrk_nccl_get_unique_id(buf))
    return buf.raw


class NcclComm:
    """An NCCL communicator created by the library (asyrk_nccl_comm_init_rank) on the current device."""

    def __init__(self, nranks, unique_id, rank):
        if len(unique_id) != NCCL_UNIQUE_ID_BYTES:
            raise ValueError("InvalidArgument: the NCCL unique id is 128 bytes")
        h = C.c_void_p()
        check(lib().asyrk_nccl_comm_init_rank(C.byref(h), nranks, unique_id, rank))
        self.handle = h.value

    def close(self):
        if getattr(self, "handle", None):
            lib().asyrk_nccl_comm_destroy(C.c_void_p(self.handle))
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def mrhs_solve_devices(A, B, devices, X0=None, X_star=None, **cfg):
    """One process, several GPUs (asyrk_mrhs_solve_devices): the k columns of B split evenly
    over `devices`, ncclCommInitAll, grouped all-reduces of the shard norms. Returns the
    global trace, X (n x k fp32) and device 0's solve stats."""
    B = np.ascontiguousarray(B, dtype=np.float32)
    k = B.shape[1]
    devs = np.ascontiguousarray(devices, dtype=np.int32)
    c = _run_config(**cfg)
    cap = max(c.epochs, 0) // max(c.snapshot_interval, 1) + 2
    tr = _Trace(0, cap, want_x=False)
    if B.ndim != 2 or B.shape[0] != A.m:
        raise AsyrkError(6, f"B has shape {B.shape}, expected ({A.m}, k)")
    X = np.zeros((A.n, k), np.float32)
    x0 = _mat(X0, (A.n, k), np.float32, "X0") if X0 is not None else None
    xs = _mat(X_star, (A.n, k), np.float64, "X_star") if X_star is not None else None
    st = SolveStats()
    check(lib().asyrk_mrhs_solve_devices(C.byref(A.view()), B.ctypes.data_as(C.POINTER(C.c_float)), k,
                                         devs.ctypes.data_as(_i32p), len(devs), C.byref(c),
                                         x0.ctypes.data_as(C.POINTER(C.c_float)) if x0 is not None else None,
                                         _ptr(xs, _f64p), C.byref(tr.out), X.ctypes.data_as(C.POINTER(C.c_float)),
                                         C.byref(st)))
    d = tr.result(xs is not None)
    d["X"] = X
    d["stats"] = {f: getattr(st, f) for f, _ in SolveStats._fields_}
    return d


def microbench_xside(n, theta, precision=F64, warps=4736, proj_per_warp=256, mode=0):
    """R_x: projections/s of the x-side traffic alone (see asyrk_microbench_xside)."""
    rate, ms = C.c_double(), C.c_double()
    check(lib().asyrk_microbench_xside(n, theta, precision, warps, proj_per_warp, mode, C.byref(rate),
                                       C.byref(ms)))
    return rate.value


def _mat(a, shape, dtype, name):
    """Contiguous host matrix of exactly `shape` (DimensionMismatch otherwise)."""
    v = np.ascontiguousarray(a, dtype=dtype)
    if v.shape != tuple(shape):
        raise AsyrkError(6, f"{name} has shape {v.shape}, expected {tuple(shape)}")
    return v


def _vec(a, n, name):
    """Contiguous float64 host vector of exactly n entries (the C ABI copies n
    doubles from it): DimensionMismatch otherwise, like the reference
    (parallel.cpp:57-61)."""
    v = np.ascontiguousarray(a, dtype=np.float64)
    if v.ndim != 1 or v.shape[0] != n:
        raise AsyrkError(6, f"{name} has {v.size} entries, expected {n}")
    return v


def microbench_xside_mrhs(n, theta, kl, warps=4096, proj_per_warp=64):
    """R_x of the multi-RHS pattern (asyrk_microbench_xside_mrhs): row projections/s."""
    rate, ms = C.c_double(), C.c_double()
    check(lib().asyrk_microbench_xside_mrhs(n, theta, kl, warps, proj_per_warp, C.byref(rate), C.byref(ms)))
    return rate.value


def check(status: int):
    if status:
        raise AsyrkError(status, lib().asyrk_last_error().decode())


def serial_row_sumsq(row_ptr, values):
    """sum_k v_k^2 per row in storage order from 0.0 — the reference's cached
    row norms are sqrt of exactly this (csr.cpp:53-61); np.add.reduceat sums in
    a different order and can differ by an ulp, which changes every projection
    coefficient gamma*res/(nrm*nrm). Vectorized across rows, serial within."""
    lens = np.diff(row_ptr)
    acc = np.zeros(len(lens))
    sq = values * values
    start = row_ptr[:-1]
    live = np.arange(len(lens))
    for k in range(int(lens.max()) if len(lens) else 0):
        live = live[lens[live] > k]
        acc[live] += sq[start[live] + k]
    return acc


class HostCsr:
    """Host CSR arrays in the reference's layout (int64 indices, fp64 values)."""

    def __init__(self, m, n, row_ptr, col_idx, values, row_norm=None, normalized=None):
        self.m, self.n = int(m), int(n)
        self.row_ptr = np.ascontiguousarray(row_ptr, dtype=np.int64)
        self.col_idx = np.ascontiguousarray(col_idx, dtype=np.int64)
        self.values = np.ascontiguousarray(values, dtype=np.float64)
        if row_norm is None:
            row_norm = np.sqrt(serial_row_sumsq(self.row_ptr, self.values))
        self.row_norm = np.ascontiguousarray(row_norm, dtype=np.float64)
        if normalized is None:
            normalized = bool(np.all(np.abs(self.row_norm - 1.0) <= 1e-12))
        self.normalized = bool(normalized)

    @property
    def nnz(self):
        return int(self.row_ptr[-1])

    def view(self):
        return CsrView(self.m, self.n, self.nnz, _ptr(self.row_ptr, _i64p), _ptr(self.col_idx, _i64p),
                       _ptr(self.values, _f64p), _ptr(self.row_norm, _f64p), 1 if self.normalized else 0)


def generate_fixed_theta(m, n, theta, seed, dist="normal", scale_decades=0.0, k=1, threads=0):
    """Seeded fixed-theta system (include/asyrk_datagen.h). Returns (HostCsr, b, x_star)."""
    nnz = m * theta
    rp = np.zeros(m + 1, np.int64)
    ci = np.zeros(nnz, np.int64)
    v = np.zeros(nnz)
    rn = np.zeros(m)
    b = np.zeros(m * k)
    xs = np.zeros(n * k)
    norm = C.c_int32(0)
    check(lib().asyrk_generate_fixed_theta(m, n, theta, seed, 1 if dist == "uniform" else 0, scale_decades, k,
                                           threads, _ptr(rp, _i64p), _ptr(ci, _i64p), _ptr(v, _f64p),
                                           _ptr(rn, _f64p), _ptr(b, _f64p), _ptr(xs, _f64p), C.byref(norm)))
    A = HostCsr(m, n, rp, ci, v, rn, bool(norm.value))
    if k > 1:
        return A, b.reshape(m, k), xs.reshape(n, k)
    return A, b, xs


class _Trace:
    def __init__(self, n, cap, want_x=True):
        self.b = dict(epoch_index=np.zeros(cap, np.int64), r_sq=np.zeros(cap), grad_sq=np.zeros(cap),
                      dist_sq=np.zeros(cap), wall_seconds=np.zeros(cap), updates_applied=np.zeros(cap, np.int64),
                      final_x=np.zeros(n) if want_x else None)
        b = self.b
        self.out = TraceOut(cap, 0, _ptr(b["epoch_index"], _i64p), _ptr(b["r_sq"], _f64p),
                            _ptr(b["grad_sq"], _f64p), _ptr(b["dist_sq"], _f64p), _ptr(b["wall_seconds"], _f64p),
                            _ptr(b["updates_applied"], _i64p), _ptr(b["final_x"], _f64p))

    def result(self, has_dist):
        k = min(self.out.count, self.out.cap)
        d = {key: (val[:k].copy() if key != "final_x" else val) for key, val in self.b.items()
             if key != "dist_sq" or has_dist}
        return d


def _run_config(threads=1, gamma=1.0, epochs=100, target=0.0, variant=FULL_ROW, sampling=SLICE_SHUFFLE, seed=0,
                snapshot_interval=1, x_star=None, precision=F64, allow_unnormalized=0, record_every_boundary=0,
                det_reassociate=0):
    return RunConfig(threads, gamma, epochs, target, variant, sampling, seed, snapshot_interval,
                     _ptr(x_star, _f64p), precision, allow_unnormalized, int(record_every_boundary),
                     int(det_reassociate))


class System:
    """Device-resident A (+ b): asyrk_system_* of the C ABI."""

    def __init__(self, A: HostCsr, b=None, precision=F64, stream=None):
        self.A = A
        self.m, self.n = A.m, A.n
        self.precision = precision
        self._traces = {}
        self._b = _vec(b, A.m, "b") if b is not None else None
        h = C.c_void_p()
        check(lib().asyrk_system_create(C.byref(A.view()), _ptr(self._b, _f64p), precision,
                                        C.c_void_p(stream) if stream else None, C.byref(h)))
        self.h = h

    def close(self):
        if getattr(self, "h", None):
            lib().asyrk_system_destroy(self.h)
            self.h = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_rhs(self, b):
        self._b = _vec(b, self.m, "b")
        check(lib().asyrk_system_set_rhs(self.h, _ptr(self._b, _f64p)))

    def solve(self, x0=None, instrument=False, want_x=True, **cfg):
        xs = cfg.pop("x_star", None)
        xs = _vec(xs, self.n, "x_star") if xs is not None else None
        c = _run_config(x_star=xs, **cfg)
        cap = max(c.epochs, 0) // max(c.snapshot_interval, 1) + 2
        # trace buffers are reused across solves of this system (result() copies them out)
        key = (cap, bool(want_x))
        tr = self._traces.get(key) if want_x is False else None
        if tr is None:
            tr = _Trace(self.n, cap, want_x)
            if not want_x:
                self._traces[key] = tr
        x0a = _vec(x0, self.n, "x0") if x0 is not None else None
        rep = InstrumentOut()
        check(lib().asyrk_system_solve(self.h, _ptr(x0a, _f64p), C.byref(c), C.byref(tr.out),
                                       C.byref(rep) if instrument else None))
        d = tr.result(xs is not None)
        if instrument:
            d["instrument"] = dict(row_updates=rep.row_updates, increments=rep.increments,
                                   max_abs_error=rep.max_abs_error, tolerance=rep.tolerance,
                                   consistent=bool(rep.consistent))
        return d

    def rk_solve_multi(self, B, X0=None, max_epochs=100, target=0.0, seed=0, sampling=RK_UNIFORM, X_star=None,
                       reassociate=False):
        """Deterministic multi-RHS rk_solve (asyrk_system_rk_solve_multi): B (m x k); column j
        of the result is rk_solve(A, B[:, j]) with the same seed, bit for bit."""
        B = np.ascontiguousarray(B, dtype=np.float64)
        if B.ndim != 2 or B.shape[0] != self.m:
            raise AsyrkError(6, f"B has shape {B.shape}, expected ({self.m}, k)")
        k = B.shape[1]
        x0 = _mat(X0, (self.n, k), np.float64, "X0") if X0 is not None else None
        xs = _mat(X_star, (self.n, k), np.float64, "X_star") if X_star is not None else None
        c = RkConfig(max_epochs, target, seed, sampling, _ptr(xs, _f64p), int(reassociate))
        tr = _Trace(0, max(max_epochs, 0) + 2, want_x=False)
        X = np.zeros((self.n, k))
        check(lib().asyrk_system_rk_solve_multi(self.h, _ptr(B, _f64p), k, _ptr(x0, _f64p), C.byref(c),
                                                _ptr(X, _f64p), C.byref(tr.out)))
        d = tr.result(xs is not None)
        d["X"] = X
        return d

    def microbench_xside(self, warps, proj_per_warp=1024, mode=0):
        """R_x on this system's own x buffer (asyrk_system_microbench_xside): proj/s."""
        rate, ms = C.c_double(), C.c_double()
        check(lib().asyrk_system_microbench_xside(self.h, warps, proj_per_warp, mode, C.byref(rate), C.byref(ms)))
        return rate.value

    def sample_rows(self, sampling, seed, warps, per_warp, epoch=0):
        """The async workers' own row draws: (warps, per_warp) int32 array (asyrk_system_sample_rows)."""
        out = np.zeros((warps, per_warp), np.int32)
        check(lib().asyrk_system_sample_rows(self.h, sampling, seed, warps, epoch, per_warp,
                                             out.ctypes.data_as(_i32p)))
        return out

    def rk_solve(self, x0=None, max_epochs=100, target=0.0, seed=0, sampling=RK_UNIFORM, x_star=None,
                 reassociate=False):
        xs = _vec(x_star, self.n, "x_star") if x_star is not None else None
        c = RkConfig(max_epochs, target, seed, sampling, _ptr(xs, _f64p), int(reassociate))
        tr = _Trace(self.n, max(max_epochs, 0) + 2)
        x0a = _vec(x0, self.n, "x0") if x0 is not None else None
        check(lib().asyrk_system_rk_solve(self.h, _ptr(x0a, _f64p), C.byref(c), C.byref(tr.out)))
        return tr.result(xs is not None)

    def residuals(self, x):
        x = _vec(x, self.n, "x")
        rs, gs = C.c_double(), C.c_double()
        check(lib().asyrk_system_residuals(self.h, _ptr(x, _f64p), C.byref(rs), C.byref(gs)))
        return rs.value, gs.value

    def multiply(self, x):
        x = _vec(x, self.n, "x")
        y = np.zeros(self.m)
        check(lib().asyrk_system_multiply(self.h, _ptr(x, _f64p), _ptr(y, _f64p)))
        return y

    def multiply_transpose(self, x):
        x = _vec(x, self.m, "x")
        y = np.zeros(self.n)
        check(lib().asyrk_system_multiply_transpose(self.h, _ptr(x, _f64p), _ptr(y, _f64p)))
        return y

    def power_iteration(self, tol=1e-6, max_iters=200000):
        lam, it = C.c_double(), C.c_int64()
        check(lib().asyrk_system_power_iteration(self.h, tol, max_iters, C.byref(lam), C.byref(it)))
        return lam.value, it.value

    def simulate(self, x0, gamma, tau, delay, iterations, seed, variant, **opts):
        """simulate (ref delay_sim.cpp:71-228) with the system's b."""
        x0 = _vec(x0, self.n, "x0")
        cfg = _sim_config(gamma, tau, delay, iterations, seed, variant, **opts)
        return _sim_call(lambda o: lib().asyrk_system_simulate(self.h, _ptr(x0, _f64p), C.byref(cfg), C.byref(o)),
                         self.n, self.m, cfg)

    def monte_carlo_ratios(self, x0, gamma, tau, delay, iterations, runs, base_seed, variant="single_component"):
        x0 = _vec(x0, self.n, "x0")
        cfg = _sim_config(gamma, tau, delay, iterations, base_seed, variant)
        mean, ratios = np.zeros(iterations + 1), np.zeros(max(iterations, 1))
        check(lib().asyrk_system_monte_carlo_ratios(self.h, _ptr(x0, _f64p), C.byref(cfg), runs, _ptr(mean, _f64p),
                                                    _ptr(ratios, _f64p)))
        return dict(mean_r_sq=mean, ratios=ratios[:iterations])

    def compute_stats(self, tol=1e-9, max_iters=200000):
        """compute_stats(exact_spectral=false) on the device (ref stats.cpp:52-130)."""
        theta = np.zeros(self.m, np.int64)
        o = StatsOut()
        o.theta = theta.ctypes.data_as(C.POINTER(C.c_int64))
        check(lib().asyrk_system_compute_stats(self.h, tol, max_iters, C.byref(o)))
        return _stats_result(o, theta)

    def stats(self):
        s = SolveStats()
        check(lib().asyrk_system_last_stats(self.h, C.byref(s)))
        return {f: getattr(s, f) for f, _ in SolveStats._fields_}

    def max_resident_warps(self, precision=None):
        out = C.c_int32()
        check(lib().asyrk_system_max_resident_warps(self.h, self.precision if precision is None else precision,
                                                    C.byref(out)))
        return out.value


def solve_parallel_host(A: HostCsr, b, x0=None, instrument=False, want_x=True, **cfg):
    """One-shot asyrk_solve_parallel with host buffers (upload, solve, download)."""
    xs = cfg.pop("x_star", None)
    xs = _vec(xs, A.n, "x_star") if xs is not None else None
    c = _run_config(x_star=xs, **cfg)
    cap = max(c.epochs, 0) // max(c.snapshot_interval, 1) + 2
    tr = _Trace(A.n, cap, want_x)
    b = _vec(b, A.m, "b")
    x0a = _vec(x0, A.n, "x0") if x0 is not None else None
    rep = InstrumentOut()
    check(lib().asyrk_solve_parallel(C.byref(A.view()), _ptr(b, _f64p), _ptr(x0a, _f64p), C.byref(c),
                                     C.byref(tr.out), C.byref(rep) if instrument else None))
    d = tr.result(xs is not None)
    if instrument:
        d["instrument"] = dict(row_updates=rep.row_updates, increments=rep.increments,
                               max_abs_error=rep.max_abs_error, tolerance=rep.tolerance,
                               consistent=bool(rep.consistent))
    return d


def monitor_schedule_next(target, boundaries, r_sq, every=False, max_gap=0):
    """The next boundary the async solves evaluate after these records (asyrk_monitor_schedule_next)."""
    bd = np.ascontiguousarray(boundaries, dtype=np.int64)
    rs = np.ascontiguousarray(r_sq, dtype=np.float64)
    out = C.c_int64()
    check(lib().asyrk_monitor_schedule_next(target, 1 if every else 0, max_gap, _ptr(bd, _i64p), _ptr(rs, _f64p),
                                            len(bd), C.byref(out)))
    return out.value


def sweep_threads(A: HostCsr, b, thread_list, x0=None, **cfg):
    """asyrk_sweep_threads (ref parallel.cpp:447-481): one solve per worker count,
    speedup = wall(threads=1) / wall(threads). Returns a list of entry dicts."""
    b = _vec(b, A.m, "b")
    x0a = _vec(x0, A.n, "x0") if x0 is not None else None
    c = _run_config(**cfg)
    tl = np.ascontiguousarray(thread_list, dtype=np.int64)
    k = len(tl)
    wall, ep, rs, sp = np.zeros(k), np.zeros(k, np.int64), np.zeros(k), np.zeros(k)
    check(lib().asyrk_sweep_threads(C.byref(A.view()), _ptr(b, _f64p), _ptr(x0a, _f64p), C.byref(c),
                                    _ptr(tl, _i64p) if k else None, k, _ptr(wall, _f64p), _ptr(ep, _i64p),
                                    _ptr(rs, _f64p), _ptr(sp, _f64p)))
    return [dict(threads=int(tl[i]), wall_seconds=float(wall[i]), epochs=int(ep[i]), final_r_sq=float(rs[i]),
                 speedup=float(sp[i])) for i in range(k)]


def simulate(A: HostCsr, b, x0, gamma, tau, delay, iterations, seed, variant, **opts):
    """One-shot asyrk_simulate (ref delay_sim.cpp:71-228); opts = probe_every, probe_r_sq, max_events,
    probe_dist_sq + dist_point (the projector's A^+ b)."""
    b = _vec(b, A.m, "b")
    x0 = _vec(x0, A.n, "x0")
    cfg = _sim_config(gamma, tau, delay, iterations, seed, variant, **opts)
    return _sim_call(lambda o: lib().asyrk_simulate(C.byref(A.view()), _ptr(b, _f64p), _ptr(x0, _f64p), C.byref(cfg),
                                                    C.byref(o)), A.n, A.m, cfg)


def monte_carlo_ratios(A: HostCsr, b, x0, gamma, tau, delay, iterations, runs, base_seed,
                       variant="single_component"):
    """One-shot asyrk_monte_carlo_ratios (ref delay_sim.cpp:230-270)."""
    b = _vec(b, A.m, "b")
    x0 = _vec(x0, A.n, "x0")
    cfg = _sim_config(gamma, tau, delay, iterations, base_seed, variant)
    mean, ratios = np.zeros(iterations + 1), np.zeros(max(iterations, 1))
    check(lib().asyrk_monte_carlo_ratios(C.byref(A.view()), _ptr(b, _f64p), _ptr(x0, _f64p), C.byref(cfg), runs,
                                         _ptr(mean, _f64p), _ptr(ratios, _f64p)))
    return dict(mean_r_sq=mean, ratios=ratios[:iterations])


def rate_fit(y, stride=1.0):
    y = np.ascontiguousarray(y, dtype=np.float64)
    sl, r2 = C.c_double(), C.c_double()
    check(lib().asyrk_rate_fit(_ptr(y, _f64p), len(y), stride, C.byref(sl), C.byref(r2)))
    return dict(slope=sl.value, r2=r2.value)


# ---- dense spectrum and least squares (include/asyrk_dense.h; ref dense.hpp, lsq.hpp)
DENSE_CAP_DEFAULT = 4000000     # SolutionProjector::kDefaultDenseCap
DENSE_DEVICE_CAP = 67108864


def dense_svd(A: "HostCsr", vectors=False, max_cells=0):
    """Thin SVD of A on the device (one-sided Jacobi; replaces ref dense.cpp:27-50).
    Returns dict(sigma (descending), rank, sweeps[, U (m x k), V (n x k)])."""
    k = min(A.m, A.n)
    sigma = np.zeros(k)
    U = np.zeros((k, A.m)) if vectors else None   # column-major m x k == row-major k x m
    V = np.zeros((k, A.n)) if vectors else None
    rank, sweeps = C.c_int32(), C.c_int32()
    check(lib().asyrk_dense_svd(C.byref(A.view()), max_cells, _ptr(sigma, _f64p), _ptr(U, _f64p), _ptr(V, _f64p),
                                C.byref(rank), C.byref(sweeps)))
    d = dict(sigma=sigma, rank=rank.value, sweeps=sweeps.value)
    if vectors:
        d["U"], d["V"] = U.T.copy(), V.T.copy()
    return d


def dense_spectrum(A: "HostCsr"):
    """dense_spectrum (ref dense.cpp:62-64): lambda_max, lambda_min, sigma_r, rank."""
    o = Spectrum()
    check(lib().asyrk_dense_spectrum(C.byref(A.view()), C.byref(o)))
    return {f: getattr(o, f) for f, _ in Spectrum._fields_}


def dense_lstsq(A: "HostCsr", b):
    """dense_min_norm_lstsq (ref dense.cpp:110-117): A^+ b from the device SVD."""
    b = _vec(b, A.m, "b")
    x = np.zeros(A.n)
    check(lib().asyrk_dense_lstsq(C.byref(A.view()), _ptr(b, _f64p), _ptr(x, _f64p)))
    return x


def lsq_optimal_params(sigma_r):
    """optimal_params (ref lsq.cpp:12-18) -> (phi, zeta)."""
    phi, zeta = C.c_double(), C.c_double()
    check(lib().asyrk_lsq_optimal_params(sigma_r, C.byref(phi), C.byref(zeta)))
    return phi.value, zeta.value


def lsq_critical_ratio(sigma_r, frob_sq, m, zeta, phi):
    """critical_ratio (ref lsq.cpp:20-34)."""
    r = C.c_double()
    check(lib().asyrk_lsq_critical_ratio(sigma_r, frob_sq, m, zeta, phi, C.byref(r)))
    return r.value


def lsq_augment(A: "HostCsr", b, zeta, phi):
    """augment (ref lsq.cpp:36-101) -> dict(a_tilde HostCsr, b_tilde, row_scales, zeta, phi)."""
    b = np.ascontiguousarray(b, dtype=np.float64)
    if len(b) != A.m:  # (the C ABI takes m entries by pointer)
        raise AsyrkError(6, "augment: b size mismatch")
    N = A.m + A.n
    bt, rs = np.zeros(N), np.zeros(N)
    h = C.c_void_p()
    check(lib().asyrk_lsq_augment(C.byref(A.view()), _ptr(b, _f64p), zeta, phi, C.byref(h), _ptr(bt, _f64p),
                                  _ptr(rs, _f64p)))
    info = HostCsrInfo()
    check(lib().asyrk_host_csr_get_info(h, C.byref(info)))
    return dict(a_tilde=_take_host_csr(h, info), b_tilde=bt, row_scales=rs, zeta=zeta, phi=phi)


def lsq_solve(A: "HostCsr", b, zeta=0.0, phi=0.0, sigma_r=None, max_epochs=5000, target=0.0, seed=0,
              sampling=RK_UNIFORM, threads=1, gamma=1.0, cap=None):
    """lsq_solve (ref lsq.cpp:103-170): min ||Ax - b|| through the augmented
    system, solved by the device rk_solve (threads <= 1) or the async warp
    workers (threads > 1). Returns dict(x_ls, y, grad_norm, zeta, phi, sigma_r, trace)."""
    b = np.ascontiguousarray(b, dtype=np.float64)
    if len(b) != A.m:
        raise AsyrkError(6, "lsq_solve: b size mismatch")
    c = LsqConfig(zeta, phi, 1 if sigma_r is not None else 0, sigma_r or 0.0, max_epochs, target, seed, sampling,
                  threads, gamma)
    x_ls, y = np.zeros(A.n), np.zeros(A.m)
    tr = _Trace(A.n + A.m, cap or (max_epochs + 2))
    o = LsqOut(_ptr(x_ls, _f64p), _ptr(y, _f64p), 0.0, 0.0, 0.0, 0.0, tr.out)
    check(lib().asyrk_lsq_solve(C.byref(A.view()), _ptr(b, _f64p), C.byref(c), C.byref(o)))
    tr.out.count = o.trace.count
    return dict(x_ls=x_ls, y=y, grad_norm=o.grad_norm, zeta=o.zeta, phi=o.phi, sigma_r=o.sigma_r,
                trace=tr.result(False))


# ---- instance I/O (include/asyrk_io.h; ref io.hpp:12-33)
def _take_host_csr(h, info):
    m, n, nnz = info.m, info.n, info.nnz
    rp, ci = np.zeros(m + 1, np.int64), np.zeros(nnz, np.int64)
    v, rn = np.zeros(nnz), np.zeros(m)
    try:
        check(lib().asyrk_host_csr_copy(h, _ptr(rp, _i64p), _ptr(ci, _i64p), _ptr(v, _f64p), _ptr(rn, _f64p)))
    finally:
        lib().asyrk_host_csr_free(h)
    return HostCsr(m, n, rp, ci, v, rn, normalized=bool(info.normalized))


def read_matrix_market(path):
    """read_matrix_market (ref io.cpp:60-96): Matrix Market coordinate file -> HostCsr."""
    h, info = C.c_void_p(), HostCsrInfo()
    check(lib().asyrk_read_matrix_market(os.fsencode(path), C.byref(h), C.byref(info)))
    return _take_host_csr(h, info)


def write_matrix_market(path, A: HostCsr):
    check(lib().asyrk_write_matrix_market(os.fsencode(path), C.byref(A.view())))


def read_csr_cache(path):
    h, info = C.c_void_p(), HostCsrInfo()
    check(lib().asyrk_read_csr_cache(os.fsencode(path), C.byref(h), C.byref(info)))
    return _take_host_csr(h, info)


def write_csr_cache(path, A: HostCsr):
    check(lib().asyrk_write_csr_cache(os.fsencode(path), C.byref(A.view())))


def _take_vec(p, count):
    try:
        return np.ctypeslib.as_array(p, shape=(count,)).copy() if count else np.zeros(0)
    finally:
        lib().asyrk_free(p)


def read_vector(path):
    p, cnt = _f64p(), C.c_int64()
    check(lib().asyrk_read_vector(os.fsencode(path), C.byref(p), C.byref(cnt)))
    return _take_vec(p, cnt.value)


def write_vector(path, v):
    v = np.ascontiguousarray(v, dtype=np.float64)
    check(lib().asyrk_write_vector(os.fsencode(path), _ptr(v, _f64p), len(v)))


def write_instance(path, A: HostCsr, b, x_star=None, spec=None):
    """write_instance (ref io.cpp:125-150): A.mtx, b.txt, xstar.txt, meta.json."""
    spec = dict(spec or {})
    b = np.ascontiguousarray(b, dtype=np.float64)
    xs = np.ascontiguousarray(x_star, dtype=np.float64) if x_star is not None else None
    meta = InstanceMeta(spec.get("m", A.m), spec.get("n", A.n), spec.get("delta", A.nnz / (A.m * A.n)),
                        spec.get("seed", 0), int(spec.get("consistent", xs is not None)),
                        spec.get("noise_level", 0.0), int(xs is not None))
    check(lib().asyrk_write_instance(os.fsencode(path), C.byref(A.view()), _ptr(b, _f64p), _ptr(xs, _f64p),
                                     C.byref(meta)))


def read_instance(path):
    """read_instance (ref io.cpp:152-183) -> dict(A, b, x_star, spec)."""
    h, pb, px, meta = C.c_void_p(), _f64p(), _f64p(), InstanceMeta()
    check(lib().asyrk_read_instance(os.fsencode(path), C.byref(h), C.byref(pb), C.byref(px), C.byref(meta)))
    info = HostCsrInfo()
    check(lib().asyrk_host_csr_get_info(h, C.byref(info)))
    A = _take_host_csr(h, info)
    b = _take_vec(pb, meta.m)
    xs = _take_vec(px, meta.n) if meta.has_x_star else None
    spec = dict(m=meta.m, n=meta.n, delta=meta.delta, seed=meta.seed, consistent=bool(meta.consistent),
                noise_level=meta.noise_level)
    return dict(A=A, b=b, x_star=xs, spec=spec)


def compute_stats(A: HostCsr, tol=1e-9, max_iters=200000):
    """One-shot asyrk_compute_stats with host buffers (exact_spectral=false)."""
    theta = np.zeros(A.m, np.int64)
    o = StatsOut()
    o.theta = theta.ctypes.data_as(C.POINTER(C.c_int64))
    check(lib().asyrk_compute_stats(C.byref(A.view()), tol, max_iters, C.byref(o)))
    return _stats_result(o, theta)


def rk_solve_host(A: HostCsr, b, x0=None, max_epochs=100, target=0.0, seed=0, sampling=RK_UNIFORM, x_star=None,
                  reassociate=False):
    xs = np.ascontiguousarray(x_star, dtype=np.float64) if x_star is not None else None
    c = RkConfig(max_epochs, target, seed, sampling, _ptr(xs, _f64p), int(reassociate))
    tr = _Trace(A.n, max(max_epochs, 0) + 2)
    b = np.ascontiguousarray(b, dtype=np.float64)
    x0a = np.ascontiguousarray(x0, dtype=np.float64) if x0 is not None else None
    check(lib().asyrk_rk_solve(C.byref(A.view()), _ptr(b, _f64p), _ptr(x0a, _f64p), C.byref(c), C.byref(tr.out)))
    return tr.result(xs is not None)
