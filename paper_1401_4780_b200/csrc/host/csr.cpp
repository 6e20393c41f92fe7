// Host side of the drop-in CSR (include/asyrk/csr.hpp): construction and
// normalization semantics of ref/src/csr.cpp:9-63,103-138, with every
// numeric pass (multiply, multiply_transpose, residuals) on the device.
#include <algorithm>
#include <array>
#include <cmath>
#include <cstring>
#include <mutex>
#include <numeric>

#include "asyrk/csr.hpp"
#include "asyrk_cuda.h"
#include "csr_coo.hpp"
#include "par.hpp"

namespace asyrk {

const char* error_code_name(ErrorCode c) {
    static const char* const names[] = {
        "IndexOutOfRange", "DuplicateEntry", "ZeroRow", "ZeroColumn", "NotNormalized",
        "DimensionMismatch", "PowerIterationDiverged", "NonFinite", "ComponentNotInSupport",
        "Inconsistent", "TooLarge", "InvalidRho", "MissingStats", "StepTooLarge", "ZeroLambdaMin",
        "InvalidGamma", "NonPositiveData", "InsufficientData", "NonPositiveSigma", "SigmaUnavailable",
        "InfeasibleSpec", "ThreadSpawnFailure", "IoError", "InvalidArgument"};
    const int k = static_cast<int>(c);
    return (k >= 0 && k < static_cast<int>(sizeof(names) / sizeof(names[0]))) ? names[k] : "Unknown";
}

void throw_status(int status) {
    if (status == ASYRK_OK) return;
    throw Error(static_cast<ErrorCode>(status - 1), asyrk_last_error());
}

// ---- device cache: one asyrk_system per precision, built on first use
struct CsrMatrix::DeviceCache {
    std::mutex mu;
    std::array<asyrk_system*, 3> sys{nullptr, nullptr, nullptr};
    ~DeviceCache() {
        for (auto* s : sys)
            if (s) asyrk_system_destroy(s);
    }
};

CsrMatrix::CsrMatrix(const CsrMatrix& o)
    : m_(o.m_), n_(o.n_), row_ptr_(o.row_ptr_), col_idx_(o.col_idx_), values_(o.values_),
      row_norm_(o.row_norm_), normalized_(o.normalized_) {}

CsrMatrix& CsrMatrix::operator=(const CsrMatrix& o) {
    if (this != &o) {
        m_ = o.m_;
        n_ = o.n_;
        row_ptr_ = o.row_ptr_;
        col_idx_ = o.col_idx_;
        values_ = o.values_;
        row_norm_ = o.row_norm_;
        normalized_ = o.normalized_;
        dev_.reset();
    }
    return *this;
}

CsrMatrix::~CsrMatrix() = default;

asyrk_system* CsrMatrix::device(int precision) const {
    if (precision < 0 || precision > 2) fail(ErrorCode::InvalidArgument, "unknown precision");
    if (!dev_) dev_ = std::make_shared<DeviceCache>();
    std::lock_guard<std::mutex> lk(dev_->mu);
    auto*& s = dev_->sys[static_cast<std::size_t>(precision)];
    if (!s) {
        asyrk_csr_view v{m_, n_, nnz(), row_ptr_.data(), col_idx_.data(), values_.data(), row_norm_.data(),
                         normalized_ ? 1 : 0};
        throw_status(asyrk_system_create(&v, nullptr, precision, nullptr, &s));
    }
    return s;
}

void CsrMatrix::release_device() const { dev_.reset(); }

void CsrMatrix::compute_norms() {
    row_norm_.resize(static_cast<std::size_t>(m_));
    // rows in parallel chunks (each row's sum is serial, so the result is the serial one)
    const int T = par::threads_for(values_.size() + static_cast<std::size_t>(m_));
    std::vector<index_t> first_zero(static_cast<std::size_t>(T), -1);
    par::chunks(static_cast<std::size_t>(m_), T, [&](int t, std::size_t lo, std::size_t hi) {
        for (std::size_t i = lo; i < hi; ++i) {
            const index_t b = row_ptr_[i], e = row_ptr_[i + 1];
            if (e == b) {
                if (first_zero[static_cast<std::size_t>(t)] < 0) first_zero[static_cast<std::size_t>(t)] = static_cast<index_t>(i);
                continue;
            }
            double ss = 0.0;  // storage order, like the reference (csr.cpp:53-61)
            for (index_t k = b; k < e; ++k)
                ss += values_[static_cast<std::size_t>(k)] * values_[static_cast<std::size_t>(k)];
            row_norm_[i] = std::sqrt(ss);
        }
    });
    for (index_t z : first_zero)  // chunks are in row order: the first one found is the first zero row
        if (z >= 0) fail(ErrorCode::ZeroRow, "row " + std::to_string(z) + " has no nonzeros");
}

CsrMatrix CsrMatrix::from_triplets(std::span<const Triplet> entries, index_t m, index_t n) {
    if (m < 1 || n < 1) fail(ErrorCode::InvalidArgument, "matrix dimensions must be positive");
    for (const Triplet& t : entries)
        if (t.row < 0 || t.row >= m || t.col < 0 || t.col >= n)
            fail(ErrorCode::IndexOutOfRange, "triplet (" + std::to_string(t.row) + "," + std::to_string(t.col) +
                                                 ") outside " + std::to_string(m) + "x" + std::to_string(n));
    // already in (row, column) order with no repeats — triplets taken from a
    // CSR, the common case: one pass, same result as the general path below
    bool sorted = true;
    for (std::size_t k = 1; k < entries.size() && sorted; ++k) {
        const Triplet &p = entries[k - 1], &q = entries[k];
        sorted = q.row > p.row || (q.row == p.row && q.col > p.col);
    }
    if (sorted) {
        CsrMatrix A;
        A.m_ = m;
        A.n_ = n;
        A.row_ptr_.assign(static_cast<std::size_t>(m) + 1, 0);
        A.col_idx_.reserve(entries.size());
        A.values_.reserve(entries.size());
        for (const Triplet& t : entries)
            if (t.value != 0.0) {
                A.col_idx_.push_back(t.col);
                A.values_.push_back(t.value);
                ++A.row_ptr_[static_cast<std::size_t>(t.row) + 1];
            }
        for (index_t i = 0; i < m; ++i) A.row_ptr_[static_cast<std::size_t>(i) + 1] += A.row_ptr_[static_cast<std::size_t>(i)];
        A.compute_norms();
        return A;
    }
    // counting sort by row, then sort each row's columns: O(nnz + rows * theta log theta)
    std::vector<index_t> start(static_cast<std::size_t>(m) + 1, 0);
    for (const Triplet& t : entries) ++start[static_cast<std::size_t>(t.row) + 1];
    for (index_t i = 0; i < m; ++i) start[static_cast<std::size_t>(i) + 1] += start[static_cast<std::size_t>(i)];
    std::vector<std::size_t> order(entries.size());
    {
        std::vector<index_t> cur(start.begin(), start.end() - 1);
        for (std::size_t k = 0; k < entries.size(); ++k)
            order[static_cast<std::size_t>(cur[static_cast<std::size_t>(entries[k].row)]++)] = k;
    }
    CsrMatrix A;
    A.m_ = m;
    A.n_ = n;
    A.row_ptr_.assign(static_cast<std::size_t>(m) + 1, 0);
    A.col_idx_.reserve(entries.size());
    A.values_.reserve(entries.size());
    for (index_t i = 0; i < m; ++i) {
        auto b = order.begin() + start[static_cast<std::size_t>(i)];
        auto e = order.begin() + start[static_cast<std::size_t>(i) + 1];
        std::stable_sort(b, e, [&](std::size_t x, std::size_t y) { return entries[x].col < entries[y].col; });
        index_t kept = 0;
        for (auto it = b; it != e; ++it) {
            if (it != b && entries[*it].col == entries[*(it - 1)].col)
                fail(ErrorCode::DuplicateEntry, "duplicate entry at (" + std::to_string(i) + "," +
                                                    std::to_string(entries[*it].col) + ")");
            if (entries[*it].value != 0.0) {
                A.col_idx_.push_back(entries[*it].col);
                A.values_.push_back(entries[*it].value);
                ++kept;
            }
        }
        A.row_ptr_[static_cast<std::size_t>(i) + 1] = A.row_ptr_[static_cast<std::size_t>(i)] + kept;
    }
    A.compute_norms();
    return A;
}

CsrMatrix CsrMatrix::from_csr(index_t m, index_t n, std::vector<index_t> row_ptr, std::vector<index_t> col_idx,
                              std::vector<double> values) {
    if (m < 1 || n < 1) fail(ErrorCode::InvalidArgument, "matrix dimensions must be positive");
    if (row_ptr.size() != static_cast<std::size_t>(m) + 1 || row_ptr.front() != 0 ||
        row_ptr.back() != static_cast<index_t>(col_idx.size()) || col_idx.size() != values.size())
        fail(ErrorCode::DimensionMismatch, "from_csr: inconsistent arrays");
    CsrMatrix A;
    A.m_ = m;
    A.n_ = n;
    A.row_ptr_ = std::move(row_ptr);
    A.col_idx_ = std::move(col_idx);
    A.values_ = std::move(values);
    A.compute_norms();
    return A;
}

double CsrMatrix::row_dot(index_t i, std::span<const double> x) const {
    double s = 0.0;
    for (index_t k = row_ptr_[static_cast<std::size_t>(i)]; k < row_ptr_[static_cast<std::size_t>(i) + 1]; ++k)
        s += values_[static_cast<std::size_t>(k)] * x[static_cast<std::size_t>(col_idx_[static_cast<std::size_t>(k)])];
    return s;
}

void CsrMatrix::multiply(std::span<const double> x, std::vector<double>& y) const {
    if (static_cast<index_t>(x.size()) != n_) fail(ErrorCode::DimensionMismatch, "multiply: x has wrong length");
    y.assign(static_cast<std::size_t>(m_), 0.0);
    throw_status(asyrk_system_multiply(device(0), x.data(), y.data()));
}

void CsrMatrix::multiply_transpose(std::span<const double> x, std::vector<double>& y) const {
    if (static_cast<index_t>(x.size()) != m_)
        fail(ErrorCode::DimensionMismatch, "multiply_transpose: x has wrong length");
    y.assign(static_cast<std::size_t>(n_), 0.0);
    throw_status(asyrk_system_multiply_transpose(device(0), x.data(), y.data()));
}

std::vector<Triplet> CsrMatrix::to_triplets() const {
    std::vector<Triplet> out;
    out.reserve(values_.size());
    for (index_t i = 0; i < m_; ++i)
        for (index_t k = row_ptr_[static_cast<std::size_t>(i)]; k < row_ptr_[static_cast<std::size_t>(i) + 1]; ++k)
            out.push_back({i, col_idx_[static_cast<std::size_t>(k)], values_[static_cast<std::size_t>(k)]});
    return out;
}

void CsrMatrix::flag_normalized() {
    for (index_t i = 0; i < m_; ++i)
        if (std::abs(row_norm_[static_cast<std::size_t>(i)] - 1.0) > kNormTol)
            fail(ErrorCode::NotNormalized, "row " + std::to_string(i) + " norm " +
                                               std::to_string(row_norm_[static_cast<std::size_t>(i)]) +
                                               " not within 1e-12 of 1");
    normalized_ = true;
    dev_.reset();
}

std::pair<CsrMatrix, std::vector<double>> normalize_rows(const CsrMatrix& A, std::span<const double> b) {
    if (!b.empty() && static_cast<index_t>(b.size()) != A.rows())
        fail(ErrorCode::DimensionMismatch, "normalize_rows: b has wrong length");
    for (index_t i = 0; i < A.rows(); ++i)
        if (A.row_norm_[static_cast<std::size_t>(i)] == 0.0)
            fail(ErrorCode::ZeroRow, "row " + std::to_string(i) + " has zero norm");
    CsrMatrix N = A;
    std::vector<double> nb(b.begin(), b.end());
    // rows in parallel chunks: every row is scaled and re-summed on its own
    par::chunks(static_cast<std::size_t>(A.rows()), par::threads_for(N.values_.size()),
                [&](int, std::size_t lo, std::size_t hi) {
                    for (std::size_t si = lo; si < hi; ++si) {
                        const double nrm = A.row_norm_[si];
                        if (std::abs(nrm - 1.0) <= CsrMatrix::kNormTol) continue;  // unit rows stay bit-identical
                        double ss = 0.0;
                        for (index_t k = N.row_ptr_[si]; k < N.row_ptr_[si + 1]; ++k) {
                            double& v = N.values_[static_cast<std::size_t>(k)];
                            v /= nrm;
                        }
                        for (index_t k = N.row_ptr_[si]; k < N.row_ptr_[si + 1]; ++k)
                            ss += N.values_[static_cast<std::size_t>(k)] * N.values_[static_cast<std::size_t>(k)];
                        if (!nb.empty()) nb[si] /= nrm;
                        N.row_norm_[si] = std::sqrt(ss);  // recomputed, not assumed 1
                    }
                });
    N.flag_normalized();
    return {std::move(N), std::move(nb)};
}

namespace {
struct CooArrays {
    std::vector<index_t> rp, ci;
    std::vector<double> v;
};

// CSR arrays from coordinates already in strictly increasing (row, column)
// order (false: another order — the caller takes the reference path); bounds
// are checked first either way, as from_triplets does
bool assemble_sorted_coo(index_t m, index_t n, const index_t* rows, const index_t* cols, const double* vals,
                         std::size_t nnz, CooArrays& out) {
    if (m < 1 || n < 1) fail(ErrorCode::InvalidArgument, "matrix dimensions must be positive");
    const int T = par::threads_for(nnz);
    // per chunk: first out-of-range entry, and whether (row, col) strictly increases
    std::vector<std::size_t> bad(static_cast<std::size_t>(T), SIZE_MAX);
    std::vector<char> sorted(static_cast<std::size_t>(T), 1);
    std::vector<std::size_t> kept(static_cast<std::size_t>(T) + 1, 0);
    par::chunks(nnz, T, [&](int t, std::size_t lo, std::size_t hi) {
        std::size_t nk = 0;
        bool srt = true;
        for (std::size_t k = lo; k < hi; ++k) {
            if (rows[k] < 0 || rows[k] >= m || cols[k] < 0 || cols[k] >= n) {
                bad[static_cast<std::size_t>(t)] = k;
                break;
            }
            if (k > 0 && !(rows[k] > rows[k - 1] || (rows[k] == rows[k - 1] && cols[k] > cols[k - 1]))) srt = false;
            nk += vals[k] != 0.0;
        }
        sorted[static_cast<std::size_t>(t)] = srt;
        kept[static_cast<std::size_t>(t) + 1] = nk;
    });
    for (std::size_t k : bad)
        if (k != SIZE_MAX)
            fail(ErrorCode::IndexOutOfRange, "triplet (" + std::to_string(rows[k]) + "," + std::to_string(cols[k]) +
                                                 ") outside " + std::to_string(m) + "x" + std::to_string(n));
    if (!std::all_of(sorted.begin(), sorted.end(), [](char c) { return c != 0; })) return false;
    // (row, column) order with no repeats — the common case, e.g. triplets taken
    // from a CSR: zero values dropped as from_triplets does, chunks write their
    // kept entries at prefix offsets and the row starts they cross
    for (int t = 0; t < T; ++t) kept[static_cast<std::size_t>(t) + 1] += kept[static_cast<std::size_t>(t)];
    const std::size_t total = kept[static_cast<std::size_t>(T)];
    std::vector<index_t>& rp = out.rp;
    std::vector<index_t>& ci = out.ci;
    std::vector<double>& v = out.v;
    rp.resize(static_cast<std::size_t>(m) + 1);
    ci.resize(total);
    v.resize(total);
    // the row of the last kept entry before each chunk (-1: none)
    std::vector<index_t> last_row(static_cast<std::size_t>(T), -1);
    par::chunks(nnz, T, [&](int t, std::size_t lo, std::size_t hi) {
        index_t lr = -1;
        for (std::size_t k = hi; k > lo; --k)
            if (vals[k - 1] != 0.0) {
                lr = rows[k - 1];
                break;
            }
        last_row[static_cast<std::size_t>(t)] = lr;
    });
    par::chunks(nnz, T, [&](int t, std::size_t lo, std::size_t hi) {
        index_t prev = -1;
        for (int u = t - 1; u >= 0 && prev < 0; --u) prev = last_row[static_cast<std::size_t>(u)];
        std::size_t p = kept[static_cast<std::size_t>(t)];
        for (std::size_t k = lo; k < hi; ++k) {
            if (vals[k] == 0.0) continue;
            for (index_t i = prev + 1; i <= rows[k]; ++i) rp[static_cast<std::size_t>(i)] = static_cast<index_t>(p);
            prev = rows[k];
            ci[p] = cols[k];
            v[p] = vals[k];
            ++p;
        }
    });
    index_t lr = -1;
    for (int t = T - 1; t >= 0 && lr < 0; --t) lr = last_row[static_cast<std::size_t>(t)];
    for (index_t i = lr + 1; i <= m; ++i) rp[static_cast<std::size_t>(i)] = static_cast<index_t>(total);
    return true;
}

CsrMatrix coo_reference_path(index_t m, index_t n, const index_t* rows, const index_t* cols, const double* vals,
                             std::size_t nnz) {
    // general order: counting sort by row, duplicates rejected (from_triplets)
    std::vector<Triplet> t(nnz);
    for (std::size_t k = 0; k < nnz; ++k) t[k] = Triplet{rows[k], cols[k], vals[k]};
    return CsrMatrix::from_triplets(t, m, n);
}
}  // namespace

CsrMatrix csr_from_coo(index_t m, index_t n, const index_t* rows, const index_t* cols, const double* vals,
                       std::size_t nnz) {
    CooArrays c;
    if (!assemble_sorted_coo(m, n, rows, cols, vals, nnz, c)) return coo_reference_path(m, n, rows, cols, vals, nnz);
    return CsrMatrix::from_csr(m, n, std::move(c.rp), std::move(c.ci), std::move(c.v));
}

std::pair<CsrMatrix, std::vector<double>> csr_from_coo_normalized(index_t m, index_t n, const index_t* rows,
                                                                  const index_t* cols, const double* vals,
                                                                  std::size_t nnz, std::span<const double> b) {
    CooArrays c;
    if (!assemble_sorted_coo(m, n, rows, cols, vals, nnz, c))
        return normalize_rows(coo_reference_path(m, n, rows, cols, vals, nnz), b);
    // normalize_rows on the arrays in place (no copy of A): the row norm as
    // compute_norms forms it, unit rows left bit-identical, the others scaled;
    // from_csr then re-forms every norm from the final values, as normalize_rows does
    const bool b_ok = b.empty() || static_cast<index_t>(b.size()) == m;
    std::vector<double> nb;
    if (b_ok) nb.assign(b.begin(), b.end());
    const int T = par::threads_for(c.v.size());
    std::vector<index_t> first_empty(static_cast<std::size_t>(T), -1), first_zero(static_cast<std::size_t>(T), -1);
    par::chunks(static_cast<std::size_t>(m), T, [&](int t, std::size_t lo, std::size_t hi) {
        for (std::size_t i = lo; i < hi; ++i) {
            const index_t kb = c.rp[i], ke = c.rp[i + 1];
            if (kb == ke) {
                if (first_empty[static_cast<std::size_t>(t)] < 0) first_empty[static_cast<std::size_t>(t)] = static_cast<index_t>(i);
                continue;
            }
            double ss = 0.0;
            for (index_t k = kb; k < ke; ++k) ss += c.v[static_cast<std::size_t>(k)] * c.v[static_cast<std::size_t>(k)];
            const double nrm = std::sqrt(ss);
            if (nrm == 0.0) {
                if (first_zero[static_cast<std::size_t>(t)] < 0) first_zero[static_cast<std::size_t>(t)] = static_cast<index_t>(i);
                continue;
            }
            if (std::abs(nrm - 1.0) <= CsrMatrix::kNormTol) continue;
            for (index_t k = kb; k < ke; ++k) c.v[static_cast<std::size_t>(k)] /= nrm;
            if (!nb.empty()) nb[i] /= nrm;
        }
    });
    for (index_t z : first_empty)  // from_triplets' compute_norms error comes first, then normalize_rows' checks
        if (z >= 0) fail(ErrorCode::ZeroRow, "row " + std::to_string(z) + " has no nonzeros");
    if (!b_ok) fail(ErrorCode::DimensionMismatch, "normalize_rows: b has wrong length");
    for (index_t z : first_zero)
        if (z >= 0) fail(ErrorCode::ZeroRow, "row " + std::to_string(z) + " has zero norm");
    CsrMatrix N = CsrMatrix::from_csr(m, n, std::move(c.rp), std::move(c.ci), std::move(c.v));
    N.flag_normalized();
    return {std::move(N), std::move(nb)};
}

Residuals residuals(const CsrMatrix& A, std::span<const double> x, std::span<const double> b) {
    if (static_cast<index_t>(x.size()) != A.cols() || static_cast<index_t>(b.size()) != A.rows())
        fail(ErrorCode::DimensionMismatch, "residuals: dimension mismatch");
    asyrk_system* s = A.device(0);
    throw_status(asyrk_system_set_rhs(s, b.data()));
    Residuals out;
    throw_status(asyrk_system_residuals(s, x.data(), &out.r_sq, &out.grad_sq));
    return out;
}

}  // namespace asyrk
