// pybind11 module `_asyrk` with the reference's Python signatures
// (ref/bindings/module.cpp:281-318: solve_rk, solve_parallel, system_stats,
// step_params, simulate): dict in / dict out, triplets -> CSR ->
// normalize_rows inside, errors as ValueError("<ErrorCodeName>: message")
// (module.cpp:271-279). Statistics use the device compute_stats with the
// dense spectrum from the device Jacobi SVD (exact_spectral, the reference
// default) up to ASYRK_DENSE_DEVICE_CAP cells, power iteration beyond.
#include <pybind11/numpy.h>
#include <pybind11/pybind11.h>
#include <pybind11/stl.h>

#include <optional>
#include <span>
#include <string>
#include <vector>

#include "asyrk/delay_sim.hpp"
#include "host/csr_coo.hpp"
#include "asyrk/dense.hpp"
#include "asyrk/lsq.hpp"
#include "asyrk_dense.h"
#include "asyrk/error.hpp"
#include "asyrk/kaczmarz.hpp"
#include "asyrk/parallel.hpp"
#include "asyrk/stats.hpp"
#include "asyrk/stepsize.hpp"
#include "asyrk/trace.hpp"

namespace py = pybind11;
using namespace asyrk;

// A 1-D host array argument (triplets, b): numpy arrays pass without a
// per-element Python conversion (the reference's std::vector arguments,
// module.cpp, convert element by element: ~2 s for config 2's 6M triplets);
// lists and other sequences are converted by numpy (forcecast).
namespace {
template <class T>
struct Arr {
    py::array_t<T, py::array::c_style | py::array::forcecast> a;
    std::size_t size() const { return static_cast<std::size_t>(a.size()); }
    const T& operator[](std::size_t i) const { return a.data()[i]; }
    const T* data() const { return a.data(); }
    operator std::vector<T>() const { return std::vector<T>(a.data(), a.data() + a.size()); }
    operator std::span<const T>() const { return std::span<const T>(a.data(), size()); }
};
}  // namespace

namespace pybind11::detail {
template <class T>
struct type_caster<Arr<T>> {
    PYBIND11_TYPE_CASTER(Arr<T>, const_name("numpy.ndarray"));
    bool load(handle src, bool) {
        auto arr = py::array_t<T, py::array::c_style | py::array::forcecast>::ensure(src);
        if (!arr || arr.ndim() != 1) return false;
        value.a = std::move(arr);
        return true;
    }
};
}  // namespace pybind11::detail

namespace {

CsrMatrix triplets_to_csr(index_t m, index_t n, const Arr<index_t>& rows, const Arr<index_t>& cols,
                          const Arr<double>& vals) {
    if (rows.size() != cols.size() || rows.size() != vals.size())
        fail(ErrorCode::DimensionMismatch, "triplet lists differ in length");
    // from_triplets' semantics straight from the arrays (host/csr_coo.hpp)
    return csr_from_coo(m, n, rows.data(), cols.data(), vals.data(), rows.size());
}

py::dict to_dict(const Trace& tr) {
    std::vector<index_t> ep, upd;
    std::vector<double> rs, gs, wall, dist;
    const bool has_dist = !tr.epochs.empty() && tr.epochs.front().dist_sq.has_value();
    for (const EpochRecord& e : tr.epochs) {
        ep.push_back(e.epoch_index);
        rs.push_back(e.r_sq);
        gs.push_back(e.grad_sq);
        wall.push_back(e.wall_seconds);
        upd.push_back(e.updates_applied);
        if (has_dist && e.dist_sq) dist.push_back(*e.dist_sq);
    }
    py::dict d;
    d["epoch_index"] = ep;
    d["r_sq"] = rs;
    d["grad_sq"] = gs;
    if (has_dist) d["dist_sq"] = dist;
    d["wall_seconds"] = wall;
    d["updates_applied"] = upd;
    d["final_x"] = tr.final_x;
    d["config"] = tr.config_echo;
    return d;
}

Sampling parse_sampling(const std::string& s) {
    if (s == "uniform") return Sampling::uniform;
    if (s == "norm" || s == "norm-proportional") return Sampling::norm_proportional;
    if (s == "shuffle") return Sampling::shuffle;
    fail(ErrorCode::InvalidArgument, "sampling: expected uniform|norm|shuffle");
}

UpdateVariant parse_variant(const std::string& s) {
    if (s == "full-row" || s == "full_row") return UpdateVariant::full_row;
    if (s == "single" || s == "single_component") return UpdateVariant::single_component;
    fail(ErrorCode::InvalidArgument, "variant: expected full-row|single");
}

py::dict solve_rk_py(index_t m, index_t n, const Arr<index_t>& rows, const Arr<index_t>& cols,
                     const Arr<double>& vals, const Arr<double>& b, index_t epochs, double target,
                     std::uint64_t seed, const std::string& sampling) {
    CsrMatrix A0 = triplets_to_csr(m, n, rows, cols, vals);
    auto [A, bn] = normalize_rows(A0, b);
    RkConfig cfg;
    cfg.max_epochs = epochs;
    cfg.target_r_sq = target;
    cfg.seed = seed;
    cfg.sampling = parse_sampling(sampling);
    std::vector<double> x0(static_cast<std::size_t>(n), 0.0);
    Trace tr;
    {
        py::gil_scoped_release nogil;
        tr = rk_solve(A, bn, x0, cfg);
    }
    return to_dict(tr);
}

py::dict solve_parallel_core(index_t m, index_t n, const Arr<index_t>& rows, const Arr<index_t>& cols,
                             const Arr<double>& vals, const Arr<double>& b, index_t threads,
                             double gamma, index_t epochs, double target, std::uint64_t seed,
                             const std::string& variant, const std::string& sampling, index_t snapshot_interval,
                             int precision, bool instrumented, const std::vector<double>* x_star) {
    DeviceOptions dev;
    dev.precision = precision;
    dev.norm_proportional = sampling == "norm" || sampling == "norm-proportional";
    // the reference normalizes before every parallel solve (module.cpp:179);
    // norm-proportional sampling is the device extension for raw rows
    CsrMatrix A;
    std::vector<double> bn;
    if (dev.norm_proportional) {
        A = triplets_to_csr(m, n, rows, cols, vals);
        bn = b;
    } else {
        if (rows.size() != cols.size() || rows.size() != vals.size())
            fail(ErrorCode::DimensionMismatch, "triplet lists differ in length");
        // triplets -> CSR -> normalize_rows, the arrays scaled in place (host/csr_coo.hpp)
        auto pr = csr_from_coo_normalized(m, n, rows.data(), cols.data(), vals.data(), rows.size(), b);
        A = std::move(pr.first);
        bn = std::move(pr.second);
    }
    RunConfig cfg;
    cfg.threads = threads;
    cfg.gamma = gamma;
    cfg.epochs = epochs;
    cfg.target_r_sq = target;
    cfg.seed = seed;
    cfg.variant = parse_variant(variant);
    cfg.sampling = (sampling == "slice" || sampling == "slice_shuffle") ? ParSampling::slice_shuffle
                                                                       : ParSampling::with_replacement;
    cfg.snapshot_interval = snapshot_interval;
    cfg.x_star = x_star;
    std::vector<double> x0(static_cast<std::size_t>(n), 0.0);
    InstrumentReport rep;
    Trace tr;
    {
        py::gil_scoped_release nogil;
        tr = solve_parallel(A, bn, x0, cfg, instrumented ? &rep : nullptr, dev);
    }
    py::dict d = to_dict(tr);
    if (instrumented)
        d["instrument"] = py::dict(py::arg("row_updates") = rep.row_updates, py::arg("increments") = rep.increments,
                                   py::arg("max_abs_error") = rep.max_abs_error, py::arg("tolerance") = rep.tolerance,
                                   py::arg("consistent") = rep.consistent);
    return d;
}

// compute_stats(N) with the reference default exact_spectral = true: the
// dense spectrum is the device Jacobi SVD (csrc/dense.cu). Past the device
// SVD cap the power-iteration lambda_max stands in (lambda_min / sigma_r
// then absent), where the reference would attempt a dense SVD it cannot hold.
SystemStats device_stats(const CsrMatrix& N) {
    StatsOptions o;
    o.exact_spectral = static_cast<double>(N.rows()) * static_cast<double>(N.cols()) <= ASYRK_DENSE_DEVICE_CAP;
    return compute_stats(N, o);
}

// module.cpp:113-135
py::dict system_stats_py(index_t m, index_t n, const Arr<index_t>& rows, const Arr<index_t>& cols,
                         const Arr<double>& vals) {
    CsrMatrix A = triplets_to_csr(m, n, rows, cols, vals);
    std::vector<double> dummy(static_cast<std::size_t>(m), 0.0);
    auto [N, ignored] = normalize_rows(A, dummy);
    SystemStats st;
    {
        py::gil_scoped_release nogil;
        st = device_stats(N);
    }
    py::dict d;
    d["m"] = st.m;
    d["n"] = st.n;
    d["delta"] = st.delta;
    d["theta"] = st.theta;
    d["mu"] = st.mu;
    d["nu"] = st.nu;
    d["alpha"] = st.alpha;
    d["lambda_max"] = st.lambda_max;
    if (st.lambda_min) d["lambda_min"] = *st.lambda_min;
    if (st.sigma_r) d["sigma_r"] = *st.sigma_r;
    d["frob_sq"] = st.frob_sq;
    d["l_max"] = st.l_max;
    d["l_res"] = st.l_res;
    return d;
}

// module.cpp:137-157
py::dict step_params_py(index_t m, index_t n, const Arr<index_t>& rows, const Arr<index_t>& cols,
                        const Arr<double>& vals, index_t tau) {
    CsrMatrix A = triplets_to_csr(m, n, rows, cols, vals);
    std::vector<double> dummy(static_cast<std::size_t>(m), 0.0);
    auto [N, ignored] = normalize_rows(A, dummy);
    SystemStats st;
    {
        py::gil_scoped_release nogil;
        st = device_stats(N);
    }
    StepParams p = corollary_params(st, tau);
    py::dict d;
    d["tau"] = p.tau;
    d["rho"] = p.rho;
    d["psi"] = p.psi;
    d["feasible"] = p.feasible;
    d["gamma"] = p.gamma;
    d["bounds"] = py::make_tuple(p.gamma_bounds.b1, p.gamma_bounds.b2, p.gamma_bounds.b3);
    if (p.rate_iter) d["rate_iteration"] = *p.rate_iter;
    if (p.rate_simplified) d["rate_simplified"] = *p.rate_simplified;
    return d;
}

// module.cpp:213-238: step parameters from the statistics, gamma overridden,
// then the device bounded-delay simulation
py::dict simulate_py(index_t m, index_t n, const Arr<index_t>& rows, const Arr<index_t>& cols,
                     const Arr<double>& vals, const Arr<double>& b, index_t iterations, index_t tau,
                     double gamma, const std::string& delay, const std::string& variant, std::uint64_t seed) {
    CsrMatrix A0 = triplets_to_csr(m, n, rows, cols, vals);
    auto [A, bn] = normalize_rows(A0, b);
    SimRun run;
    StepParams p;
    {
        py::gil_scoped_release nogil;
        p = corollary_params(device_stats(A), tau);
        p.gamma = gamma;
        DelayModel dm;
        if (delay == "fixed")
            dm = DelayModel::fixed(tau);
        else if (delay == "uniform")
            dm = DelayModel::uniform_random(tau);
        else if (delay == "max")
            dm = DelayModel::max_staleness(tau);
        else
            fail(ErrorCode::InvalidArgument, "delay: expected fixed|uniform|max");
        std::vector<double> x0(static_cast<std::size_t>(n), 0.0);
        run = simulate(A, bn, x0, p, dm, iterations, seed, parse_variant(variant), {});
    }
    py::dict d = to_dict(run.trace);
    d["gamma"] = p.gamma;
    d["rho"] = p.rho;
    d["psi"] = p.psi;
    return d;
}

// module.cpp:227-246: triplets -> normalize_rows(A0, b) -> lsq_solve with the
// derived (phi, zeta); the augmented solve runs on the device
py::dict lsq_py(index_t m, index_t n, const Arr<index_t>& rows, const Arr<index_t>& cols,
                const Arr<double>& vals, const Arr<double>& b, index_t epochs, double target,
                std::uint64_t seed, std::optional<double> sigma_r, index_t threads, double gamma) {
    CsrMatrix A0 = triplets_to_csr(m, n, rows, cols, vals);
    auto [A, bn] = normalize_rows(A0, b);
    LsqConfig cfg;
    cfg.max_epochs = epochs;
    cfg.target_r_sq = target;
    cfg.seed = seed;
    cfg.sigma_r = sigma_r;
    cfg.threads = threads;
    cfg.gamma = gamma;
    LsqResult res;
    {
        py::gil_scoped_release nogil;
        res = lsq_solve(A, bn, cfg);
    }
    py::dict d;
    d["x_ls"] = res.x_ls;
    d["grad_norm"] = res.grad_norm;
    d["zeta"] = res.zeta;
    d["phi"] = res.phi;
    d["sigma_r"] = res.sigma_r;
    d["trace"] = to_dict(res.trace);
    return d;
}

}  // namespace

PYBIND11_MODULE(_asyrk, mod) {
    mod.doc() = "B200-native AsyRK: sm_100a row-projection solvers behind the reference's signatures.";

    py::register_exception_translator([](std::exception_ptr p) {
        try {
            if (p) std::rethrow_exception(p);
        } catch (const Error& e) {
            const std::string text = std::string(error_code_name(e.code())) + ": " + e.what();
            PyErr_SetString(PyExc_ValueError, text.c_str());
        }
    });

    mod.def("solve_rk", &solve_rk_py, py::arg("m"), py::arg("n"), py::arg("rows"), py::arg("cols"), py::arg("vals"),
            py::arg("b"), py::arg("epochs") = 100, py::arg("target") = 0.0, py::arg("seed") = 0,
            py::arg("sampling") = "uniform",
            "Serial randomized row-projection solve from x0 = 0 (deterministic device worker, "
            "bit-identical to the reference).");
    mod.def(
        "solve_parallel",
        [](index_t m, index_t n, const Arr<index_t>& rows, const Arr<index_t>& cols,
           const Arr<double>& vals, const Arr<double>& b, index_t threads, double gamma,
           index_t epochs, double target, std::uint64_t seed, const std::string& variant) {
            // reference: slice_shuffle, snapshot_interval 1, always instrumented (module.cpp:182-191)
            return solve_parallel_core(m, n, rows, cols, vals, b, threads, gamma, epochs, target, seed, variant,
                                       "slice", 1, 0, true, nullptr);
        },
        py::arg("m"), py::arg("n"), py::arg("rows"), py::arg("cols"), py::arg("vals"), py::arg("b"),
        py::arg("threads") = 1, py::arg("gamma") = 1.0, py::arg("epochs") = 100, py::arg("target") = 0.0,
        py::arg("seed") = 0, py::arg("variant") = "full-row",
        "Lock-free solve with `threads` warp-workers; returns the trace plus an instrument report.");
    mod.def(
        "solve_parallel_device",
        [](index_t m, index_t n, const Arr<index_t>& rows, const Arr<index_t>& cols,
           const Arr<double>& vals, const Arr<double>& b, index_t threads, double gamma,
           index_t epochs, double target, std::uint64_t seed, const std::string& variant, const std::string& sampling,
           index_t snapshot_interval, int precision, bool instrument, std::optional<std::vector<double>> x_star) {
            return solve_parallel_core(m, n, rows, cols, vals, b, threads, gamma, epochs, target, seed, variant,
                                       sampling, snapshot_interval, precision, instrument,
                                       x_star ? &*x_star : nullptr);
        },
        py::arg("m"), py::arg("n"), py::arg("rows"), py::arg("cols"), py::arg("vals"), py::arg("b"),
        py::arg("threads") = 1, py::arg("gamma") = 1.0, py::arg("epochs") = 100, py::arg("target") = 0.0,
        py::arg("seed") = 0, py::arg("variant") = "full-row", py::arg("sampling") = "slice",
        py::arg("snapshot_interval") = 1, py::arg("precision") = 0, py::arg("instrument") = false,
        py::arg("x_star") = py::none(),
        "solve_parallel with the device options: sampling slice|replacement|norm, precision 0/1/2.");
    mod.def("system_stats", &system_stats_py, py::arg("m"), py::arg("n"), py::arg("rows"), py::arg("cols"),
            py::arg("vals"),
            "Structural and spectral statistics (rows normalized first; device compute_stats, "
            "dense spectrum from the device Jacobi SVD).");
    mod.def("step_params", &step_params_py, py::arg("m"), py::arg("n"), py::arg("rows"), py::arg("cols"),
            py::arg("vals"), py::arg("tau"), "Staleness-aware step size and rate bounds for delay bound tau.");
    mod.def("simulate", &simulate_py, py::arg("m"), py::arg("n"), py::arg("rows"), py::arg("cols"), py::arg("vals"),
            py::arg("b"), py::arg("iterations"), py::arg("tau"), py::arg("gamma"), py::arg("delay") = "uniform",
            py::arg("variant") = "single", py::arg("seed") = 0,
            "Deterministic bounded-delay simulation of the asynchronous update recursion (device replay, "
            "bit-identical to the reference).");
    mod.def("lsq", &lsq_py, py::arg("m"), py::arg("n"), py::arg("rows"), py::arg("cols"), py::arg("vals"),
            py::arg("b"), py::arg("epochs") = 5000, py::arg("target") = 0.0, py::arg("seed") = 0,
            py::arg("sigma_r") = py::none(), py::arg("threads") = 1, py::arg("gamma") = 1.0,
            "Least squares through the square augmented encoding with the optimal coupling parameters "
            "(device rk_solve; threads > 1: async warp workers; sigma_r skips the dense SVD).");
    mod.def(
        "dense_spectrum",
        [](index_t m, index_t n, const Arr<index_t>& rows, const Arr<index_t>& cols,
           const Arr<double>& vals) {
            CsrMatrix A = triplets_to_csr(m, n, rows, cols, vals);
            Spectrum sp;
            {
                py::gil_scoped_release nogil;
                sp = dense_spectrum(A);
            }
            return py::dict(py::arg("lambda_max") = sp.lambda_max, py::arg("lambda_min") = sp.lambda_min,
                            py::arg("sigma_r") = sp.sigma_r, py::arg("rank") = sp.rank);
        },
        py::arg("m"), py::arg("n"), py::arg("rows"), py::arg("cols"), py::arg("vals"),
        "Dense spectrum of the raw matrix (device one-sided Jacobi SVD; ref dense_spectrum).");
    mod.def(
        "lambda_max",
        [](index_t m, index_t n, const Arr<index_t>& rows, const Arr<index_t>& cols,
           const Arr<double>& vals, double tol, index_t max_iters) {
            CsrMatrix A0 = triplets_to_csr(m, n, rows, cols, vals);
            auto [A, ignored] = normalize_rows(A0, {});
            py::gil_scoped_release nogil;
            return power_iteration_lambda_max(A, tol, max_iters);
        },
        py::arg("m"), py::arg("n"), py::arg("rows"), py::arg("cols"), py::arg("vals"), py::arg("tol") = 1e-9,
        py::arg("max_iters") = 200000, "lambda_max(A^T A) of the row-normalized matrix (device power iteration).");
    mod.def(
        "residuals",
        [](index_t m, index_t n, const Arr<index_t>& rows, const Arr<index_t>& cols,
           const Arr<double>& vals, const Arr<double>& b, const std::vector<double>& x) {
            CsrMatrix A = triplets_to_csr(m, n, rows, cols, vals);
            Residuals r = residuals(A, x, b);
            return py::dict(py::arg("r_sq") = r.r_sq, py::arg("grad_sq") = r.grad_sq);
        },
        py::arg("m"), py::arg("n"), py::arg("rows"), py::arg("cols"), py::arg("vals"), py::arg("b"), py::arg("x"),
        "||Ax-b||^2 and ||A^T(Ax-b)||^2 of the raw (unnormalized) system, reference summation order.");
    mod.def(
        "max_feasible_tau", [](index_t m, double lambda_max) { return max_feasible_tau(m, lambda_max); },
        py::arg("m"), py::arg("lambda_max"), "Largest tau with 2e*lambda_max*(tau+1)/m <= 1.");
}
