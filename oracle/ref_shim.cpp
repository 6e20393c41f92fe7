// Test infrastructure only: a flat C shim over the UNMODIFIED reference
// library, compiled from /root/reference/proj/src by oracle/Makefile into
// oracle/_ref/libasyrk_ref.so. It lets pytest (ctypes) and bench.py's
// reference arm drive the reference's own code path:
//   CsrMatrix::from_triplets / normalize_rows  (ref/src/csr.cpp:9-63,113-138)
//   rk_solve                                   (ref/src/kaczmarz.cpp:128-227)
//   solve_parallel (+InstrumentReport)         (ref/src/parallel.cpp:220-445)
//   residuals                                  (ref/src/csr.cpp:140-160)
//   power_iteration_lambda_max                 (ref/src/stats.cpp:15-50)
//   corollary_params                           (ref/src/stepsize.cpp:59-82)
//   gen_sparse_gaussian                        (ref/src/datagen.cpp:13-137)
//   AliasTable, make_stream/uniform_below      (ref/src/kaczmarz.cpp:14-61, rng.hpp)
//   simulate / monte_carlo_ratios / rate_fit   (ref/src/delay_sim.cpp:71-338)
//   Matrix Market / vector / instance I/O      (ref/src/io.cpp:41-183)
//   augment / lsq_solve / optimal_params       (ref/src/lsq.cpp:12-170)
// Nothing here is shipped; the product never links this library.
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "asyrk/csr.hpp"
#include "asyrk/datagen.hpp"
#include "asyrk/delay_sim.hpp"
#include "asyrk/io.hpp"
#include "asyrk/error.hpp"
#include "asyrk/kaczmarz.hpp"
#include "asyrk/lsq.hpp"
#include "asyrk/parallel.hpp"
#include "asyrk/rng.hpp"
#include "asyrk/stats.hpp"
#include "asyrk/stepsize.hpp"

using namespace asyrk;

namespace {
thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const Error& e) {
        g_err = std::string(error_code_name(e.code())) + ": " + e.what();
        return 1 + static_cast<int>(e.code());
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1000;
    }
}

struct Handle {
    CsrMatrix A;
};
}  // namespace

extern "C" {

struct ref_trace {
    int64_t cap;
    int64_t count;
    int64_t* epoch_index;
    double* r_sq;
    double* grad_sq;
    double* dist_sq;  // may be null
    double* wall;
    int64_t* updates;
    double* final_x;  // n entries, may be null
};

struct ref_instrument {
    int64_t row_updates;
    int64_t increments;
    double max_abs_error;
    double tolerance;
    int32_t consistent;
};

const char* ref_last_error() { return g_err.c_str(); }

static void dump_trace(const Trace& tr, ref_trace* out) {
    out->count = static_cast<int64_t>(tr.epochs.size());
    const int64_t k = std::min<int64_t>(out->cap, out->count);
    for (int64_t i = 0; i < k; ++i) {
        const auto& e = tr.epochs[static_cast<std::size_t>(i)];
        if (out->epoch_index) out->epoch_index[i] = e.epoch_index;
        if (out->r_sq) out->r_sq[i] = e.r_sq;
        if (out->grad_sq) out->grad_sq[i] = e.grad_sq;
        if (out->dist_sq) out->dist_sq[i] = e.dist_sq ? *e.dist_sq : -1.0;
        if (out->wall) out->wall[i] = e.wall_seconds;
        if (out->updates) out->updates[i] = e.updates_applied;
    }
    if (out->final_x)
        std::memcpy(out->final_x, tr.final_x.data(), tr.final_x.size() * sizeof(double));
}

// Triplets -> reference CsrMatrix; normalize != 0 applies normalize_rows with
// b_in (m entries, may be null) and writes the rescaled b to b_out.
void* ref_csr_build(int64_t m, int64_t n, int64_t nnz, const int64_t* rows, const int64_t* cols,
                    const double* vals, int normalize, const double* b_in, double* b_out, int* status) {
    Handle* h = nullptr;
    *status = guarded([&] {
        std::vector<Triplet> t(static_cast<std::size_t>(nnz));
        for (int64_t k = 0; k < nnz; ++k) t[static_cast<std::size_t>(k)] = {rows[k], cols[k], vals[k]};
        CsrMatrix A = CsrMatrix::from_triplets(t, m, n);
        if (normalize) {
            std::vector<double> b(b_in ? b_in : nullptr, b_in ? b_in + m : nullptr);
            auto [N, nb] = normalize_rows(A, b);
            if (b_out && !nb.empty()) std::memcpy(b_out, nb.data(), nb.size() * sizeof(double));
            h = new Handle{std::move(N)};
        } else {
            h = new Handle{std::move(A)};
        }
    });
    return h;
}

void ref_csr_free(void* h) { delete static_cast<Handle*>(h); }

int64_t ref_csr_nnz(void* h) { return static_cast<Handle*>(h)->A.nnz(); }

void ref_csr_dims(void* h, int64_t* m, int64_t* n) {
    *m = static_cast<Handle*>(h)->A.rows();
    *n = static_cast<Handle*>(h)->A.cols();
}

void ref_csr_export(void* hp, int64_t* row_ptr, int64_t* col_idx, double* vals, double* row_norm,
                    int* normalized) {
    const CsrMatrix& A = static_cast<Handle*>(hp)->A;
    if (row_ptr) std::memcpy(row_ptr, A.row_ptr().data(), A.row_ptr().size() * 8);
    if (col_idx) std::memcpy(col_idx, A.col_idx().data(), A.col_idx().size() * 8);
    if (vals) std::memcpy(vals, A.values().data(), A.values().size() * 8);
    if (row_norm) std::memcpy(row_norm, A.row_norm().data(), A.row_norm().size() * 8);
    if (normalized) *normalized = A.is_normalized() ? 1 : 0;
}

// gen_sparse_gaussian(consistent=true): returns the normalized A; b (m), x* (n).
void* ref_gen_sparse_gaussian(int64_t m, int64_t n, double delta, uint64_t seed, double* b_out,
                              double* xstar_out, int* status) {
    Handle* h = nullptr;
    *status = guarded([&] {
        Instance inst = gen_sparse_gaussian({m, n, delta, seed, true, 0.0});
        std::memcpy(b_out, inst.b.data(), inst.b.size() * 8);
        std::memcpy(xstar_out, inst.x_star->data(), inst.x_star->size() * 8);
        h = new Handle{std::move(inst.A)};
    });
    return h;
}

// sampling: 0 uniform, 1 norm_proportional, 2 shuffle (kaczmarz.hpp:89-93)
int ref_rk_solve(void* hp, const double* b, const double* x0, int64_t max_epochs, double target,
                 uint64_t seed, int sampling, const double* xstar, ref_trace* out) {
    return guarded([&] {
        const CsrMatrix& A = static_cast<Handle*>(hp)->A;
        std::vector<double> xs;
        RkConfig cfg;
        cfg.max_epochs = max_epochs;
        cfg.target_r_sq = target;
        cfg.seed = seed;
        cfg.sampling = sampling == 0 ? Sampling::uniform
                                     : (sampling == 1 ? Sampling::norm_proportional : Sampling::shuffle);
        if (xstar) {
            xs.assign(xstar, xstar + A.cols());
            cfg.x_star = &xs;
        }
        Trace tr = rk_solve(A, {b, static_cast<std::size_t>(A.rows())},
                            {x0, static_cast<std::size_t>(A.cols())}, cfg);
        dump_trace(tr, out);
    });
}

// variant: 0 single_component, 1 full_row; sampling: 0 with_replacement, 1 slice_shuffle
int ref_solve_parallel(void* hp, const double* b, const double* x0, int64_t threads, double gamma,
                       int64_t epochs, double target, int variant, int sampling, uint64_t seed,
                       int64_t snapshot_interval, const double* xstar, ref_trace* out,
                       ref_instrument* rep) {
    return guarded([&] {
        const CsrMatrix& A = static_cast<Handle*>(hp)->A;
        std::vector<double> xs;
        RunConfig cfg;
        cfg.threads = threads;
        cfg.gamma = gamma;
        cfg.epochs = epochs;
        cfg.target_r_sq = target;
        cfg.variant = variant == 1 ? UpdateVariant::full_row : UpdateVariant::single_component;
        cfg.sampling = sampling == 1 ? ParSampling::slice_shuffle : ParSampling::with_replacement;
        cfg.seed = seed;
        cfg.snapshot_interval = snapshot_interval;
        if (xstar) {
            xs.assign(xstar, xstar + A.cols());
            cfg.x_star = &xs;
        }
        InstrumentReport r;
        Trace tr = solve_parallel(A, {b, static_cast<std::size_t>(A.rows())},
                                  {x0, static_cast<std::size_t>(A.cols())}, cfg, rep ? &r : nullptr);
        dump_trace(tr, out);
        if (rep) {
            rep->row_updates = r.row_updates;
            rep->increments = r.increments;
            rep->max_abs_error = r.max_abs_error;
            rep->tolerance = r.tolerance;
            rep->consistent = r.consistent ? 1 : 0;
        }
    });
}

int ref_residuals(void* hp, const double* x, const double* b, double* r_out, double* r_sq,
                  double* grad_sq) {
    return guarded([&] {
        const CsrMatrix& A = static_cast<Handle*>(hp)->A;
        Residuals r = residuals(A, {x, static_cast<std::size_t>(A.cols())},
                                {b, static_cast<std::size_t>(A.rows())});
        if (r_out) std::memcpy(r_out, r.r.data(), r.r.size() * 8);
        *r_sq = r.r_sq;
        *grad_sq = r.grad_sq;
    });
}

int ref_multiply(void* hp, const double* x, double* y) {
    return guarded([&] {
        const CsrMatrix& A = static_cast<Handle*>(hp)->A;
        std::vector<double> out;
        A.multiply({x, static_cast<std::size_t>(A.cols())}, out);
        std::memcpy(y, out.data(), out.size() * 8);
    });
}

int ref_multiply_transpose(void* hp, const double* x, double* y) {
    return guarded([&] {
        const CsrMatrix& A = static_cast<Handle*>(hp)->A;
        std::vector<double> out;
        A.multiply_transpose({x, static_cast<std::size_t>(A.rows())}, out);
        std::memcpy(y, out.data(), out.size() * 8);
    });
}

int ref_power_iteration(void* hp, double tol, int64_t max_iters, double* lambda) {
    return guarded([&] {
        *lambda = power_iteration_lambda_max(static_cast<Handle*>(hp)->A, tol, max_iters);
    });
}

// compute_stats with exact_spectral=false (power-iteration lambda_max).
int ref_stats(void* hp, double tol, int64_t* mu, int64_t* nu, double* alpha, double* lambda_max,
              double* frob_sq) {
    return guarded([&] {
        StatsOptions o;
        o.exact_spectral = false;
        o.tol = tol;
        SystemStats s = compute_stats(static_cast<Handle*>(hp)->A, o);
        *mu = s.mu;
        *nu = s.nu;
        *alpha = s.alpha;
        *lambda_max = s.lambda_max;
        *frob_sq = s.frob_sq;
    });
}

// compute_stats with exact_spectral=false, every scalar field + theta.
// d[6] = {delta, alpha, lambda_max, frob_sq, l_max, l_res}
int ref_stats_full(void* hp, double tol, int64_t max_iters, int64_t* mu, int64_t* nu, double* d, int64_t* theta) {
    return guarded([&] {
        StatsOptions o;
        o.exact_spectral = false;
        o.tol = tol;
        o.max_power_iters = max_iters;
        SystemStats s = compute_stats(static_cast<Handle*>(hp)->A, o);
        *mu = s.mu;
        *nu = s.nu;
        d[0] = s.delta;
        d[1] = s.alpha;
        d[2] = s.lambda_max;
        d[3] = s.frob_sq;
        d[4] = s.l_max;
        d[5] = s.l_res;
        if (theta)
            for (std::size_t i = 0; i < s.theta.size(); ++i) theta[i] = s.theta[i];
    });
}

int ref_corollary(int64_t m, int64_t mu, double alpha, double lambda_max, int64_t tau, double* rho,
                  double* psi, double* gamma, int* feasible) {
    return guarded([&] {
        SystemStats s;
        s.m = m;
        s.mu = mu;
        s.alpha = alpha;
        s.lambda_max = lambda_max;
        StepParams p = corollary_params(s, tau);
        *rho = p.rho;
        *psi = p.psi;
        *gamma = p.gamma;
        *feasible = p.feasible ? 1 : 0;
    });
}

// Raw mt19937_64 outputs of make_stream(seed, stream) (rng.hpp:14-25).
void ref_stream_raw(uint64_t seed, uint64_t stream, int64_t count, uint64_t* out) {
    auto g = make_stream(seed, stream);
    for (int64_t k = 0; k < count; ++k) out[k] = g();
}

void ref_uniform_below_seq(uint64_t seed, uint64_t stream, uint64_t n, int64_t count, uint64_t* out) {
    auto g = make_stream(seed, stream);
    for (int64_t k = 0; k < count; ++k) out[k] = uniform_below(g, n);
}

void ref_normal_seq(uint64_t seed, uint64_t stream, int64_t count, double* out) {
    auto g = make_stream(seed, stream);
    for (int64_t k = 0; k < count; ++k) out[k] = standard_normal(g);
}

// `rounds` cumulative Fisher-Yates shuffles of the identity of size n
// (parallel.cpp:119-123,160-162 / kaczmarz.cpp:157-160,203).
void ref_shuffle_seq(uint64_t seed, uint64_t stream, int64_t n, int64_t rounds, int64_t* out) {
    auto g = make_stream(seed, stream);
    std::vector<int64_t> p(static_cast<std::size_t>(n));
    for (int64_t i = 0; i < n; ++i) p[static_cast<std::size_t>(i)] = i;
    for (int64_t r = 0; r < rounds; ++r) {
        shuffle_in_place(p, g);
        std::memcpy(out + r * n, p.data(), static_cast<std::size_t>(n) * 8);
    }
}

int ref_alias_sample_seq(const double* w, int64_t n, uint64_t seed, int64_t count, int64_t* out) {
    return guarded([&] {
        AliasTable t({w, static_cast<std::size_t>(n)});
        auto g = make_stream(seed, 0);
        for (int64_t k = 0; k < count; ++k) out[k] = t.sample(g);
    });
}

int ref_rk_step(void* hp, const double* b, const double* x, int64_t i, double* out) {
    return guarded([&] {
        const CsrMatrix& A = static_cast<Handle*>(hp)->A;
        auto y = rk_step(A, {b, static_cast<std::size_t>(A.rows())},
                         {x, static_cast<std::size_t>(A.cols())}, i);
        std::memcpy(out, y.data(), y.size() * 8);
    });
}

int ref_asyrk_update(void* hp, const double* b, int64_t i, int64_t t, double gamma, const double* x,
                     double* out) {
    return guarded([&] {
        const CsrMatrix& A = static_cast<Handle*>(hp)->A;
        *out = asyrk_update(A, {b, static_cast<std::size_t>(A.rows())}, i, t, gamma,
                            {x, static_cast<std::size_t>(A.cols())});
    });
}

// ---- bounded-delay simulator (delay_sim.hpp:13-96)
struct ref_sim_out {
    ref_trace trace;
    int64_t ev_cap, ev_count;
    int64_t *ev_j, *ev_i, *ev_t, *ev_k;
    double* ev_step;
    int64_t hist_cap, hist_rows;  // rows of n
    double* history;
    int64_t probe_cap, probe_count;
    int64_t* probe_iteration;
    double* probe_r_sq;
};

static DelayModel delay_of(int kind, int64_t tau) {
    if (kind == 1) return DelayModel::uniform_random(tau);
    if (kind == 2) return DelayModel::max_staleness(tau);
    return DelayModel::fixed(tau);
}

static StepParams params_of(double gamma, int64_t tau) {
    StepParams p;
    p.tau = tau;
    p.gamma = gamma;
    p.feasible = true;
    return p;
}

// variant: 0 single_component, 1 full_row (UpdateVariant order, kaczmarz.hpp:20)
int ref_simulate(void* hp, const double* b, const double* x0, double gamma, int64_t tau, int kind,
                 int64_t iterations, uint64_t seed, int variant, int64_t probe_every, int probe_r_sq,
                 int64_t max_events, ref_sim_out* out) {
    return guarded([&] {
        const CsrMatrix& A = static_cast<Handle*>(hp)->A;
        SimOptions o;
        o.probe_every = probe_every;
        o.probe_r_sq = probe_r_sq != 0;
        o.max_events = max_events;
        SimRun r = simulate(A, std::span<const double>(b, (size_t)A.rows()),
                            std::span<const double>(x0, (size_t)A.cols()), params_of(gamma, tau), delay_of(kind, tau),
                            iterations, seed, variant ? SimVariant::full_row : SimVariant::single_component, o);
        dump_trace(r.trace, &out->trace);
        out->ev_count = (int64_t)r.events.size();
        for (int64_t k = 0; k < std::min(out->ev_cap, out->ev_count); ++k) {
            const auto& e = r.events[(size_t)k];
            out->ev_j[k] = e.j;
            out->ev_i[k] = e.i;
            out->ev_t[k] = e.t;
            out->ev_k[k] = e.k;
            out->ev_step[k] = e.step;
        }
        out->hist_rows = (int64_t)r.history.size();
        for (int64_t k = 0; k < std::min(out->hist_cap, out->hist_rows); ++k)
            std::memcpy(out->history + k * A.cols(), r.history[(size_t)k].data(), (size_t)A.cols() * 8);
        out->probe_count = (int64_t)r.probe_iteration.size();
        for (int64_t k = 0; k < std::min(out->probe_cap, out->probe_count); ++k) {
            out->probe_iteration[k] = r.probe_iteration[(size_t)k];
            if (o.probe_r_sq) out->probe_r_sq[k] = r.probe_r_sq[(size_t)k];
        }
    });
}

int ref_monte_carlo(void* hp, const double* b, const double* x0, double gamma, int64_t tau, int kind,
                    int64_t iterations, int64_t runs, uint64_t base_seed, int variant, double* mean_r_sq,
                    double* ratios) {
    return guarded([&] {
        const CsrMatrix& A = static_cast<Handle*>(hp)->A;
        MonteCarloRatios mc = monte_carlo_ratios(
            A, std::span<const double>(b, (size_t)A.rows()), std::span<const double>(x0, (size_t)A.cols()),
            params_of(gamma, tau), delay_of(kind, tau), iterations, runs, base_seed,
            variant ? SimVariant::full_row : SimVariant::single_component);
        std::memcpy(mean_r_sq, mc.mean_r_sq.data(), mc.mean_r_sq.size() * 8);
        std::memcpy(ratios, mc.ratios.data(), mc.ratios.size() * 8);
    });
}

int ref_rate_fit(const double* y, int64_t n, double stride, double* slope, double* r2) {
    return guarded([&] {
        RateFit f = rate_fit(std::span<const double>(y, (size_t)n), stride);
        *slope = f.slope;
        *r2 = f.r2;
    });
}

// ---- instance I/O (io.hpp:12-33)
int ref_write_mtx(void* hp, const char* path) {
    return guarded([&] { write_matrix_market(path, static_cast<Handle*>(hp)->A); });
}

void* ref_read_mtx(const char* path, int* status) {
    Handle* h = nullptr;
    *status = guarded([&] { h = new Handle{read_matrix_market(path)}; });
    return h;
}

int ref_write_vector(const char* path, const double* v, int64_t n) {
    return guarded([&] { write_vector(path, std::span<const double>(v, (size_t)n)); });
}

// count = the vector length; at most cap values copied
int ref_read_vector(const char* path, double* out, int64_t cap, int64_t* count) {
    return guarded([&] {
        std::vector<double> v = read_vector(path);
        *count = (int64_t)v.size();
        std::memcpy(out, v.data(), (size_t)std::min<int64_t>(cap, *count) * 8);
    });
}

int ref_write_instance(void* hp, const double* b, const double* xs, int64_t m, int64_t n, double delta, uint64_t seed,
                       int consistent, double noise_level, const char* dir) {
    return guarded([&] {
        Instance inst;
        inst.A = static_cast<Handle*>(hp)->A;
        inst.b.assign(b, b + inst.A.rows());
        if (xs) inst.x_star = std::vector<double>(xs, xs + inst.A.cols());
        inst.spec = GenSpec{m, n, delta, seed, consistent != 0, noise_level};
        write_instance(dir, inst);
    });
}

// b_out: m values, xs_out: n values (has_xs = 0 when absent); meta6 = {m, n, delta, seed, consistent, noise}
void* ref_read_instance(const char* dir, double* b_out, int64_t b_cap, double* xs_out, int64_t xs_cap, int* has_xs,
                        double* meta6, int* status) {
    Handle* h = nullptr;
    *status = guarded([&] {
        Instance inst = read_instance(dir);
        std::memcpy(b_out, inst.b.data(), (size_t)std::min<int64_t>(b_cap, (int64_t)inst.b.size()) * 8);
        *has_xs = inst.x_star ? 1 : 0;
        if (inst.x_star)
            std::memcpy(xs_out, inst.x_star->data(), (size_t)std::min<int64_t>(xs_cap, (int64_t)inst.x_star->size()) * 8);
        meta6[0] = (double)inst.spec.m;
        meta6[1] = (double)inst.spec.n;
        meta6[2] = inst.spec.delta;
        meta6[3] = (double)inst.spec.seed;
        meta6[4] = inst.spec.consistent ? 1.0 : 0.0;
        meta6[5] = inst.spec.noise_level;
        h = new Handle{std::move(inst.A)};
    });
    return h;
}

}  // extern "C"

// ---- least squares (ref/src/lsq.cpp:12-170) and general instances
extern "C" {

// gen_sparse_gaussian with the full GenSpec (datagen.hpp:11-18): consistent
// or noisy b; x* written only when present (*has_xs).
void* ref_gen_instance(int64_t m, int64_t n, double delta, uint64_t seed, int consistent, double noise,
                       double* b_out, double* xstar_out, int* has_xs, int* status) {
    Handle* h = nullptr;
    *status = guarded([&] {
        Instance inst = gen_sparse_gaussian({m, n, delta, seed, consistent != 0, noise});
        std::memcpy(b_out, inst.b.data(), inst.b.size() * 8);
        *has_xs = inst.x_star ? 1 : 0;
        if (inst.x_star && xstar_out) std::memcpy(xstar_out, inst.x_star->data(), inst.x_star->size() * 8);
        h = new Handle{std::move(inst.A)};
    });
    return h;
}

int ref_optimal_params(double sigma_r, double* phi, double* zeta) {
    return guarded([&] {
        auto p = optimal_params(sigma_r);
        *phi = p.first;
        *zeta = p.second;
    });
}

int ref_critical_ratio(double sigma_r, double frob_sq, int64_t m, double zeta, double phi, double* out) {
    return guarded([&] { *out = critical_ratio(sigma_r, frob_sq, m, zeta, phi); });
}

// augment: returns a_tilde as a handle; b_tilde / row_scales (n+m entries)
void* ref_augment(void* hp, const double* b, double zeta, double phi, double* b_tilde, double* row_scales,
                  int* status) {
    Handle* h = nullptr;
    *status = guarded([&] {
        const CsrMatrix& A = static_cast<Handle*>(hp)->A;
        AugmentedSystem aug = augment(A, std::span<const double>(b, (size_t)A.rows()), zeta, phi);
        std::memcpy(b_tilde, aug.b_tilde.data(), aug.b_tilde.size() * 8);
        std::memcpy(row_scales, aug.row_scales.data(), aug.row_scales.size() * 8);
        h = new Handle{std::move(aug.a_tilde)};
    });
    return h;
}

// lsq_solve with a supplied sigma_r (> 0; <= 0 leaves it unset, which needs
// the dense SVD the stub refuses). scal <- {grad_norm, zeta, phi, sigma_r}.
int ref_lsq_solve(void* hp, const double* b, double zeta, double phi, double sigma_r, int64_t max_epochs,
                  double target, uint64_t seed, int sampling, double* x_ls, double* y, double* scal, ref_trace* tr) {
    return guarded([&] {
        const CsrMatrix& A = static_cast<Handle*>(hp)->A;
        LsqConfig cfg;
        cfg.zeta = zeta;
        cfg.phi = phi;
        if (sigma_r > 0.0) cfg.sigma_r = sigma_r;
        cfg.max_epochs = max_epochs;
        cfg.target_r_sq = target;
        cfg.seed = seed;
        cfg.sampling = sampling == 1 ? Sampling::norm_proportional : sampling == 2 ? Sampling::shuffle
                                                                                   : Sampling::uniform;
        LsqResult r = lsq_solve(A, std::span<const double>(b, (size_t)A.rows()), cfg);
        std::memcpy(x_ls, r.x_ls.data(), r.x_ls.size() * 8);
        if (y) std::memcpy(y, r.y.data(), r.y.size() * 8);
        scal[0] = r.grad_norm;
        scal[1] = r.zeta;
        scal[2] = r.phi;
        scal[3] = r.sigma_r;
        if (tr) dump_trace(r.trace, tr);
    });
}

// Trace serialization (ref/src/trace.cpp:33-112): parse a JSONL trace with
// the reference's Trace::from_jsonl and write it back with its to_jsonl and
// to_csv, so the product's serializers can be byte-compared on the same
// content. out buffers: cap bytes each; *len_* = the full lengths.
int ref_trace_roundtrip(const char* text, char* out_jsonl, int64_t cap_j, char* out_csv, int64_t cap_c,
                        int64_t* len_j, int64_t* len_c) {
    return guarded([&] {
        const Trace t = Trace::from_jsonl(text);
        const std::string j = t.to_jsonl(), c = t.to_csv();
        *len_j = (int64_t)j.size();
        *len_c = (int64_t)c.size();
        if (cap_j > 0) std::memcpy(out_jsonl, j.data(), std::min<size_t>(j.size(), (size_t)cap_j));
        if (cap_c > 0) std::memcpy(out_csv, c.data(), std::min<size_t>(c.size(), (size_t)cap_c));
    });
}

}  // extern "C"
