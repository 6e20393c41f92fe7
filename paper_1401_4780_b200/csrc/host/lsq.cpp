// Drop-in least squares (ref/src/lsq.cpp:12-170).
//
// augment() builds the (n+m)-square system directly in CSR, O(nnz): the top
// block's row t is column t of A scaled by phi (a counting-sort transpose
// visits rows in ascending order, which is the column order from_triplets
// would produce), the bottom block's row n+i is row i of A followed by
// -zeta on the diagonal. Row norms and normalization are the reference's
// (compute_norms / normalize_rows), so a_tilde, b_tilde and row_scales are
// bit-identical to the reference's. lsq_solve then runs the augmented solve
// on the device: rk_solve (the reference's own path, bit-identical iterates)
// or, with LsqConfig::threads > 1, the async warp workers.
#include "asyrk/lsq.hpp"

#include <cmath>
#include <cstring>
#include <string>

#include "../capi_common.h"
#include "asyrk/dense.hpp"
#include "asyrk/error.hpp"
#include "asyrk/parallel.hpp"
#include "asyrk_dense.h"
#include "common.hpp"

namespace asyrk {

std::pair<double, double> optimal_params(double sigma_r) {
    if (!(sigma_r > 0.0)) fail(ErrorCode::NonPositiveSigma, "the smallest nonzero singular value must be positive");
    return {1.0, sigma_r / std::sqrt(2.0)};
}

double critical_ratio(double sigma_r, double frob_sq, index_t m, double zeta, double phi) {
    if (!(sigma_r > 0.0) || !(frob_sq > 0.0) || m < 1 || !(zeta > 0.0) || !(phi > 0.0))
        fail(ErrorCode::InvalidArgument, "critical_ratio needs positive inputs");
    const double balanced = -zeta / 2.0 + std::sqrt(zeta * zeta + 4.0 * phi * sigma_r * sigma_r) / 2.0;
    const double lam = std::min(zeta, balanced);
    return lam * lam / ((1.0 + phi * phi) * frob_sq + static_cast<double>(m) * zeta * zeta);
}

AugmentedSystem augment(const CsrMatrix& A, std::span<const double> b, double zeta, double phi) {
    const index_t m = A.rows(), n = A.cols();
    if (static_cast<index_t>(b.size()) != m) fail(ErrorCode::DimensionMismatch, "augment: b size mismatch");
    if (!A.is_normalized()) fail(ErrorCode::NotNormalized, "augment expects normalized rows");
    if (!(zeta > 0.0) || !(phi > 0.0)) fail(ErrorCode::InvalidArgument, "zeta and phi must be positive");

    const auto& rp = A.row_ptr();
    const auto& ci = A.col_idx();
    const auto& va = A.values();
    const std::size_t nnz = va.size();
    // CSC by counting sort; entries of a column in ascending row order
    std::vector<index_t> cp(static_cast<std::size_t>(n) + 1, 0);
    for (std::size_t e = 0; e < nnz; ++e) ++cp[static_cast<std::size_t>(ci[e]) + 1];
    for (index_t t = 0; t < n; ++t) {
        if (cp[static_cast<std::size_t>(t) + 1] == 0)
            fail(ErrorCode::ZeroColumn, "column " + std::to_string(t) +
                                            " is empty: its augmented row would read 0 = 0; drop the variable first");
        cp[static_cast<std::size_t>(t) + 1] += cp[static_cast<std::size_t>(t)];
    }
    std::vector<index_t> crow(nnz);
    std::vector<double> cval(nnz);
    {
        std::vector<index_t> cur(cp.begin(), cp.end() - 1);
        for (index_t i = 0; i < m; ++i)
            for (index_t e = rp[static_cast<std::size_t>(i)]; e < rp[static_cast<std::size_t>(i) + 1]; ++e) {
                const std::size_t pos = static_cast<std::size_t>(cur[static_cast<std::size_t>(ci[e])]++);
                crow[pos] = i;
                cval[pos] = va[static_cast<std::size_t>(e)];
            }
    }

    const index_t N = n + m;
    std::vector<index_t> arp(static_cast<std::size_t>(N) + 1, 0);
    std::vector<index_t> aci;
    std::vector<double> av;
    aci.reserve(2 * nnz + static_cast<std::size_t>(m));
    av.reserve(2 * nnz + static_cast<std::size_t>(m));
    bool underflow = false;
    for (index_t t = 0; t < n; ++t) {  // top block: phi * A^T against y
        for (index_t e = cp[static_cast<std::size_t>(t)]; e < cp[static_cast<std::size_t>(t) + 1]; ++e) {
            const double v = phi * cval[static_cast<std::size_t>(e)];
            if (v == 0.0) {
                underflow = true;  // from_triplets drops explicit zeros
                continue;
            }
            aci.push_back(n + crow[static_cast<std::size_t>(e)]);
            av.push_back(v);
        }
        arp[static_cast<std::size_t>(t) + 1] = static_cast<index_t>(av.size());
    }
    for (index_t i = 0; i < m; ++i) {  // bottom block: A against x, -zeta I against y
        for (index_t e = rp[static_cast<std::size_t>(i)]; e < rp[static_cast<std::size_t>(i) + 1]; ++e) {
            aci.push_back(ci[static_cast<std::size_t>(e)]);
            av.push_back(va[static_cast<std::size_t>(e)]);
        }
        aci.push_back(n + i);
        av.push_back(-zeta);
        arp[static_cast<std::size_t>(n + i) + 1] = static_cast<index_t>(av.size());
    }
    CsrMatrix raw;
    if (!underflow) {
        raw = CsrMatrix::from_csr(N, N, std::move(arp), std::move(aci), std::move(av));
    } else {  // rare: a phi*a product underflowed; defer to the triplet builder's exact semantics
        std::vector<Triplet> trip;
        for (index_t t = 0; t < n; ++t)
            for (index_t e = cp[static_cast<std::size_t>(t)]; e < cp[static_cast<std::size_t>(t) + 1]; ++e)
                trip.push_back({t, n + crow[static_cast<std::size_t>(e)], phi * cval[static_cast<std::size_t>(e)]});
        for (index_t i = 0; i < m; ++i) {
            for (index_t e = rp[static_cast<std::size_t>(i)]; e < rp[static_cast<std::size_t>(i) + 1]; ++e)
                trip.push_back({n + i, ci[static_cast<std::size_t>(e)], va[static_cast<std::size_t>(e)]});
            trip.push_back({n + i, n + i, -zeta});
        }
        raw = CsrMatrix::from_triplets(trip, N, N);
    }

    // phi * A^T b, multiply_transpose's row-order accumulation (csr.cpp:80-92)
    std::vector<double> bt(static_cast<std::size_t>(N), 0.0);
    for (index_t i = 0; i < m; ++i) {
        const double xi = b[static_cast<std::size_t>(i)];
        if (xi == 0.0) continue;
        for (index_t e = rp[static_cast<std::size_t>(i)]; e < rp[static_cast<std::size_t>(i) + 1]; ++e)
            bt[static_cast<std::size_t>(ci[static_cast<std::size_t>(e)])] += va[static_cast<std::size_t>(e)] * xi;
    }
    for (index_t t = 0; t < n; ++t) bt[static_cast<std::size_t>(t)] = phi * bt[static_cast<std::size_t>(t)];

    AugmentedSystem aug;
    aug.zeta = zeta;
    aug.phi = phi;
    aug.row_scales = raw.row_norm();
    auto [scaled, scaled_b] = normalize_rows(raw, bt);
    aug.a_tilde = std::move(scaled);
    aug.b_tilde = std::move(scaled_b);
    return aug;
}

LsqResult lsq_solve(const CsrMatrix& A, std::span<const double> b, const LsqConfig& cfg) {
    const index_t m = A.rows(), n = A.cols();
    if (static_cast<index_t>(b.size()) != m) fail(ErrorCode::DimensionMismatch, "lsq_solve: b size mismatch");
    if (!A.is_normalized()) fail(ErrorCode::NotNormalized, "lsq_solve expects normalized rows");

    double sigma_r;
    if (cfg.sigma_r) {
        if (!(*cfg.sigma_r > 0.0)) fail(ErrorCode::NonPositiveSigma, "supplied sigma_r must be > 0");
        sigma_r = *cfg.sigma_r;
    } else {
        if (m * n > SolutionProjector::kDefaultDenseCap)
            fail(ErrorCode::SigmaUnavailable, "matrix too large for the dense spectrum; pass sigma_r");
        sigma_r = dense_spectrum(A).sigma_r;
        if (!(sigma_r > 0.0)) fail(ErrorCode::SigmaUnavailable, "could not extract a positive smallest singular value");
    }

    const auto [phi_opt, zeta_opt] = optimal_params(sigma_r);
    const double phi = cfg.phi > 0.0 ? cfg.phi : phi_opt;
    const double zeta = cfg.zeta > 0.0 ? cfg.zeta : zeta_opt;

    const AugmentedSystem aug = augment(A, b, zeta, phi);
    std::vector<double> x0(static_cast<std::size_t>(n + m), 0.0);
    Trace trace;
    if (cfg.threads <= 1) {
        RkConfig rk;
        rk.max_epochs = cfg.max_epochs;
        rk.target_r_sq = cfg.target_r_sq;
        rk.seed = cfg.seed;
        rk.sampling = cfg.sampling;
        trace = rk_solve(aug.a_tilde, aug.b_tilde, x0, rk);
    } else {
        RunConfig rc;
        rc.threads = cfg.threads;
        rc.gamma = cfg.gamma;
        rc.epochs = cfg.max_epochs;
        rc.target_r_sq = cfg.target_r_sq;
        rc.seed = cfg.seed;
        rc.sampling = ParSampling::with_replacement;
        trace = solve_parallel(aug.a_tilde, aug.b_tilde, x0, rc);
    }

    LsqResult out;
    out.zeta = zeta;
    out.phi = phi;
    out.sigma_r = sigma_r;
    out.x_ls.resize(static_cast<std::size_t>(n));
    for (index_t t = 0; t < n; ++t)  // the x block is zeta * x_ls
        out.x_ls[static_cast<std::size_t>(t)] = trace.final_x[static_cast<std::size_t>(t)] / zeta;
    out.y.assign(trace.final_x.begin() + n, trace.final_x.end());

    std::vector<double> ax;
    A.multiply(out.x_ls, ax);  // device SpMV, reference summation order
    for (index_t i = 0; i < m; ++i) ax[static_cast<std::size_t>(i)] -= b[static_cast<std::size_t>(i)];
    std::vector<double> grad;
    A.multiply_transpose(ax, grad);
    double g = 0.0;
    for (double v : grad) g += v * v;
    out.grad_norm = std::sqrt(g);
    out.trace = std::move(trace);
    return out;
}

}  // namespace asyrk

// ---- C ABI (include/asyrk_dense.h)
namespace {

template <class F>
asyrk_status lsq_guarded(F&& f) {
    try {
        return f();
    } catch (const asyrk::Error& e) {
        return ak::fail((asyrk_status)(static_cast<int>(e.code()) + 1), e.what());
    } catch (const std::bad_alloc&) {
        return ak::fail(ASYRK_E_TooLarge, "host allocation failed");
    } catch (const std::exception& e) {
        return ak::fail(ASYRK_E_InvalidArgument, e.what());
    }
}

asyrk::CsrMatrix matrix_of(const asyrk_csr_view* A) {
    if (!A || !A->row_ptr || !A->col_idx || !A->values || A->m < 1 || A->n < 1 || A->row_ptr[A->m] != A->nnz)
        asyrk::fail(asyrk::ErrorCode::InvalidArgument, "bad csr view");
    asyrk::CsrMatrix M = asyrk::CsrMatrix::from_csr(
        A->m, A->n, std::vector<int64_t>(A->row_ptr, A->row_ptr + A->m + 1),
        std::vector<int64_t>(A->col_idx, A->col_idx + A->nnz), std::vector<double>(A->values, A->values + A->nnz));
    if (A->normalized) M.flag_normalized();
    return M;
}

}  // namespace

extern "C" {

asyrk_status asyrk_lsq_optimal_params(double sigma_r, double* phi, double* zeta) {
    if (!phi || !zeta) return ak::fail(ASYRK_E_InvalidArgument, "null argument");
    return lsq_guarded([&] {
        const auto p = asyrk::optimal_params(sigma_r);
        *phi = p.first;
        *zeta = p.second;
        return ASYRK_OK;
    });
}

asyrk_status asyrk_lsq_critical_ratio(double sigma_r, double frob_sq, int64_t m, double zeta, double phi,
                                      double* ratio) {
    if (!ratio) return ak::fail(ASYRK_E_InvalidArgument, "null argument");
    return lsq_guarded([&] {
        *ratio = asyrk::critical_ratio(sigma_r, frob_sq, m, zeta, phi);
        return ASYRK_OK;
    });
}

asyrk_status asyrk_lsq_augment(const asyrk_csr_view* A, const double* b, double zeta, double phi,
                               asyrk_host_csr** a_tilde, double* b_tilde, double* row_scales) {
    if (!A || !b || !a_tilde) return ak::fail(ASYRK_E_InvalidArgument, "null argument");
    return lsq_guarded([&] {
        const asyrk::CsrMatrix M = matrix_of(A);
        asyrk::AugmentedSystem aug = asyrk::augment(M, std::span<const double>(b, (size_t)A->m), zeta, phi);
        if (b_tilde) std::memcpy(b_tilde, aug.b_tilde.data(), aug.b_tilde.size() * 8);
        if (row_scales) std::memcpy(row_scales, aug.row_scales.data(), aug.row_scales.size() * 8);
        auto h = std::make_unique<asyrk_host_csr>();
        h->A = std::move(aug.a_tilde);
        *a_tilde = h.release();
        return ASYRK_OK;
    });
}

asyrk_status asyrk_lsq_solve(const asyrk_csr_view* A, const double* b, const asyrk_lsq_config* cfg,
                             asyrk_lsq_out* out) {
    if (!A || !b || !cfg || !out || !out->x_ls) return ak::fail(ASYRK_E_InvalidArgument, "null argument");
    return lsq_guarded([&] {
        const asyrk::CsrMatrix M = matrix_of(A);
        asyrk::LsqConfig c;
        c.zeta = cfg->zeta;
        c.phi = cfg->phi;
        if (cfg->has_sigma_r) c.sigma_r = cfg->sigma_r;
        c.max_epochs = cfg->max_epochs;
        c.target_r_sq = cfg->target_r_sq;
        c.seed = cfg->seed;
        c.sampling = cfg->sampling == ASYRK_RK_NORM_PROPORTIONAL ? asyrk::Sampling::norm_proportional
                     : cfg->sampling == ASYRK_RK_SHUFFLE         ? asyrk::Sampling::shuffle
                                                                 : asyrk::Sampling::uniform;
        c.threads = cfg->threads;
        c.gamma = cfg->gamma > 0.0 ? cfg->gamma : 1.0;
        asyrk::LsqResult r = asyrk::lsq_solve(M, std::span<const double>(b, (size_t)A->m), c);
        std::memcpy(out->x_ls, r.x_ls.data(), r.x_ls.size() * 8);
        if (out->y) std::memcpy(out->y, r.y.data(), r.y.size() * 8);
        out->grad_norm = r.grad_norm;
        out->zeta = r.zeta;
        out->phi = r.phi;
        out->sigma_r = r.sigma_r;
        asyrk_trace_out& t = out->trace;
        t.count = (int64_t)r.trace.epochs.size();
        const int64_t k = std::min<int64_t>(t.count, t.cap);
        for (int64_t e = 0; e < k; ++e) {
            const asyrk::EpochRecord& rec = r.trace.epochs[(size_t)e];
            if (t.epoch_index) t.epoch_index[e] = rec.epoch_index;
            if (t.r_sq) t.r_sq[e] = rec.r_sq;
            if (t.grad_sq) t.grad_sq[e] = rec.grad_sq;
            if (t.dist_sq) t.dist_sq[e] = rec.dist_sq ? *rec.dist_sq : -1.0;
            if (t.wall_seconds) t.wall_seconds[e] = rec.wall_seconds;
            if (t.updates_applied) t.updates_applied[e] = rec.updates_applied;
        }
        if (t.final_x) std::memcpy(t.final_x, r.trace.final_x.data(), r.trace.final_x.size() * 8);
        return ASYRK_OK;
    });
}

}  // extern "C"
