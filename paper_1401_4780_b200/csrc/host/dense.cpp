// Drop-in dense oracle (ref/src/dense.cpp): the thin SVD comes from the
// device one-sided Jacobi (asyrk_dense_svd, csrc/dense.cu); projector
// arithmetic follows dense.cpp:52-117 on the host (desk scale, <= 4e6 cells).
#include "asyrk/dense.hpp"

#include <algorithm>
#include <cmath>
#include <string>

#include "../capi_common.h"
#include "asyrk/error.hpp"
#include "asyrk_dense.h"

namespace asyrk {

namespace {

asyrk_csr_view view_of(const CsrMatrix& A) {
    asyrk_csr_view v{};
    v.m = A.rows();
    v.n = A.cols();
    v.nnz = A.nnz();
    v.row_ptr = A.row_ptr().data();
    v.col_idx = A.col_idx().data();
    v.values = A.values().data();
    v.row_norm = A.row_norm().data();
    v.normalized = A.is_normalized() ? 1 : 0;
    return v;
}

struct Svd {
    index_t m = 0, n = 0;
    int k = 0, rank = 0;
    std::vector<double> sigma, U, V;  // U: m x k, V: n x k, column-major
};

Svd decompose(const CsrMatrix& A, bool vectors, index_t cap) {
    Svd s;
    s.m = A.rows();
    s.n = A.cols();
    s.k = static_cast<int>(std::min(s.m, s.n));
    s.sigma.resize(static_cast<std::size_t>(s.k));
    if (vectors) {
        s.U.resize(static_cast<std::size_t>(s.m) * s.k);
        s.V.resize(static_cast<std::size_t>(s.n) * s.k);
    }
    const asyrk_csr_view v = view_of(A);
    int32_t rank = 0;
    throw_status(asyrk_dense_svd(&v, cap, s.sigma.data(), vectors ? s.U.data() : nullptr,
                                 vectors ? s.V.data() : nullptr, &rank, nullptr));
    s.rank = rank;
    return s;
}

Spectrum spectrum_of(const Svd& p) {
    Spectrum s;
    s.lambda_max = p.k > 0 ? p.sigma[0] * p.sigma[0] : 0.0;
    s.sigma_r = p.rank > 0 ? p.sigma[static_cast<std::size_t>(p.rank - 1)] : 0.0;
    s.lambda_min = s.sigma_r * s.sigma_r;
    s.rank = p.rank;
    return s;
}

// V_r diag(1/sigma) U_r^T rhs (dense.cpp:52-58)
std::vector<double> pinv_apply(const Svd& p, std::span<const double> rhs) {
    std::vector<double> c(static_cast<std::size_t>(p.rank), 0.0);
    for (int k = 0; k < p.rank; ++k) {
        const double* u = p.U.data() + static_cast<std::size_t>(k) * p.m;
        double s = 0.0;
        for (index_t i = 0; i < p.m; ++i) s += u[i] * rhs[static_cast<std::size_t>(i)];
        c[static_cast<std::size_t>(k)] = s / p.sigma[static_cast<std::size_t>(k)];
    }
    std::vector<double> x(static_cast<std::size_t>(p.n), 0.0);
    for (int k = 0; k < p.rank; ++k) {
        const double* v = p.V.data() + static_cast<std::size_t>(k) * p.n;
        const double ck = c[static_cast<std::size_t>(k)];
        for (index_t j = 0; j < p.n; ++j) x[static_cast<std::size_t>(j)] += v[j] * ck;
    }
    return x;
}

// U_r (S_r (V_r^T x)) (dense.cpp:96-100)
std::vector<double> ax_of(const Svd& p, std::span<const double> x) {
    std::vector<double> ax(static_cast<std::size_t>(p.m), 0.0);
    for (int k = 0; k < p.rank; ++k) {
        const double* v = p.V.data() + static_cast<std::size_t>(k) * p.n;
        double t = 0.0;
        for (index_t j = 0; j < p.n; ++j) t += v[j] * x[static_cast<std::size_t>(j)];
        t *= p.sigma[static_cast<std::size_t>(k)];
        const double* u = p.U.data() + static_cast<std::size_t>(k) * p.m;
        for (index_t i = 0; i < p.m; ++i) ax[static_cast<std::size_t>(i)] += u[i] * t;
    }
    return ax;
}

double norm2(const std::vector<double>& v) {
    double s = 0.0;
    for (double x : v) s += x * x;
    return std::sqrt(s);
}

}  // namespace

Spectrum dense_spectrum(const CsrMatrix& A) { return spectrum_of(decompose(A, false, 0)); }

struct SolutionProjector::Impl {
    Svd svd;
    std::vector<double> point;  // A^+ b when rank == n
};

SolutionProjector::SolutionProjector(const CsrMatrix& A, std::vector<double> b, index_t max_dense_elements) {
    if (A.rows() * A.cols() > max_dense_elements)
        fail(ErrorCode::TooLarge,
             "dense projection oracle capped at " + std::to_string(max_dense_elements) + " elements");
    if (static_cast<index_t>(b.size()) != A.rows()) fail(ErrorCode::DimensionMismatch, "projector: b has wrong length");
    auto impl = std::make_shared<Impl>();
    impl->svd = decompose(A, true, max_dense_elements);
    if (impl->svd.rank == A.cols()) impl->point = pinv_apply(impl->svd, b);
    spectrum_ = spectrum_of(impl->svd);
    b_ = std::move(b);
    impl_ = std::move(impl);
}

std::vector<double> SolutionProjector::project(std::span<const double> x) const {
    const Svd& p = impl_->svd;
    // residual in row space only: A z = b requires b in range(A)
    std::vector<double> r(static_cast<std::size_t>(p.m));
    for (index_t i = 0; i < p.m; ++i) r[static_cast<std::size_t>(i)] = -b_[static_cast<std::size_t>(i)];
    for (int k = 0; k < p.rank; ++k) {
        const double* u = p.U.data() + static_cast<std::size_t>(k) * p.m;
        double c = 0.0;
        for (index_t i = 0; i < p.m; ++i) c += u[i] * b_[static_cast<std::size_t>(i)];
        for (index_t i = 0; i < p.m; ++i) r[static_cast<std::size_t>(i)] += u[i] * c;
    }
    const double bnorm = norm2(b_);
    if (norm2(r) > 1e-8 * std::max(1.0, bnorm))
        fail(ErrorCode::Inconsistent, "b is not in range(A); system inconsistent");
    std::vector<double> ax = ax_of(p, x);
    for (index_t i = 0; i < p.m; ++i) ax[static_cast<std::size_t>(i)] -= b_[static_cast<std::size_t>(i)];
    const std::vector<double> corr = pinv_apply(p, ax);
    std::vector<double> z(x.begin(), x.end());
    for (std::size_t j = 0; j < z.size(); ++j) z[j] -= corr[j];
    return z;
}

double SolutionProjector::dist_sq(std::span<const double> x) const {
    const Svd& p = impl_->svd;
    std::vector<double> ax = ax_of(p, x);
    for (index_t i = 0; i < p.m; ++i) ax[static_cast<std::size_t>(i)] -= b_[static_cast<std::size_t>(i)];
    const std::vector<double> corr = pinv_apply(p, ax);
    double s = 0.0;
    for (double c : corr) s += c * c;
    return s;
}

const std::vector<double>& SolutionProjector::solution_point() const { return impl_->point; }

const std::vector<double>& projector_point(const SolutionProjector& p, index_t n) {
    const std::vector<double>& pt = p.solution_point();
    if (static_cast<index_t>(pt.size()) != n)
        fail(ErrorCode::TooLarge,
             "projector distances on the device need A of full column rank (the solution set is the point "
             "A^+ b); a rank-deficient A would need the dense projection of every record");
    return pt;
}

std::vector<double> dense_min_norm_lstsq(const CsrMatrix& A, std::span<const double> b) {
    if (static_cast<index_t>(b.size()) != A.rows()) fail(ErrorCode::DimensionMismatch, "lstsq: b has wrong length");
    return pinv_apply(decompose(A, true, 0), b);
}

std::vector<std::vector<double>> to_dense(const CsrMatrix& A) {
    std::vector<std::vector<double>> D(static_cast<std::size_t>(A.rows()),
                                       std::vector<double>(static_cast<std::size_t>(A.cols()), 0.0));
    for (index_t i = 0; i < A.rows(); ++i)
        for (index_t k = A.row_ptr()[static_cast<std::size_t>(i)]; k < A.row_ptr()[static_cast<std::size_t>(i) + 1]; ++k)
            D[static_cast<std::size_t>(i)][static_cast<std::size_t>(A.col_idx()[static_cast<std::size_t>(k)])] =
                A.values()[static_cast<std::size_t>(k)];
    return D;
}

}  // namespace asyrk

extern "C" asyrk_status asyrk_dense_spectrum(const asyrk_csr_view* A, asyrk_spectrum* out) {
    if (!A || !out) return ak::fail(ASYRK_E_InvalidArgument, "null argument");
    const int64_t k = std::min(A->m, A->n);
    if (k < 1) return asyrk_dense_svd(A, 0, nullptr, nullptr, nullptr, nullptr, nullptr);
    std::vector<double> sigma(static_cast<std::size_t>(k));
    int32_t rank = 0;
    const asyrk_status st = asyrk_dense_svd(A, 0, sigma.data(), nullptr, nullptr, &rank, nullptr);
    if (st) return st;
    out->lambda_max = sigma[0] * sigma[0];
    out->sigma_r = rank > 0 ? sigma[static_cast<std::size_t>(rank - 1)] : 0.0;
    out->lambda_min = out->sigma_r * out->sigma_r;
    out->rank = rank;
    return ASYRK_OK;
}

extern "C" asyrk_status asyrk_dense_lstsq(const asyrk_csr_view* A, const double* b, double* x) {
    if (!A || !b || !x || !A->row_ptr || (A->nnz > 0 && (!A->col_idx || !A->values)))
        return ak::fail(ASYRK_E_InvalidArgument, "null argument");
    try {
        const asyrk::CsrMatrix M = asyrk::CsrMatrix::from_csr(
            A->m, A->n, std::vector<int64_t>(A->row_ptr, A->row_ptr + A->m + 1),
            std::vector<int64_t>(A->col_idx, A->col_idx + A->nnz), std::vector<double>(A->values, A->values + A->nnz));
        const std::vector<double> r = asyrk::dense_min_norm_lstsq(M, std::span<const double>(b, (size_t)A->m));
        std::copy(r.begin(), r.end(), x);
        return ASYRK_OK;
    } catch (const asyrk::Error& e) {
        return ak::fail((asyrk_status)(static_cast<int>(e.code()) + 1), e.what());
    } catch (const std::exception& e) {
        return ak::fail(ASYRK_E_TooLarge, e.what());
    }
}
