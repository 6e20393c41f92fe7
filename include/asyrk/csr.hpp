// Drop-in CSR storage (ref/include/asyrk/csr.hpp:12-90, hot-path subset).
// Same public interface as the reference CsrMatrix; additionally owns a
// lazily created device copy (row records + CSC) that every
// GPU entry point reuses while the matrix lives. A is immutable after
// construction, so the cache never goes stale.
#pragma once

#include <cstdint>
#include <memory>
#include <span>
#include <string>
#include <utility>
#include <vector>

#include "asyrk/error.hpp"

struct asyrk_system;

namespace asyrk {

using index_t = std::int64_t;

struct Triplet {
    index_t row;
    index_t col;
    double value;
};

class CsrMatrix {
  public:
    static constexpr double kNormTol = 1e-12;

    CsrMatrix() = default;
    CsrMatrix(const CsrMatrix& o);
    CsrMatrix& operator=(const CsrMatrix& o);
    CsrMatrix(CsrMatrix&&) noexcept = default;
    CsrMatrix& operator=(CsrMatrix&&) noexcept = default;
    ~CsrMatrix();

    /// Rows sorted, columns ascending within rows, explicit zeros dropped,
    /// duplicates and empty rows rejected (ref csr.cpp:9-63).
    static CsrMatrix from_triplets(std::span<const Triplet> entries, index_t m, index_t n);

    /// Adopts ready CSR arrays (sorted, duplicate-free); row norms are
    /// computed as from_triplets does. Used by the config generators.
    static CsrMatrix from_csr(index_t m, index_t n, std::vector<index_t> row_ptr, std::vector<index_t> col_idx,
                              std::vector<double> values);

    index_t rows() const { return m_; }
    index_t cols() const { return n_; }
    index_t nnz() const { return static_cast<index_t>(values_.size()); }
    bool is_normalized() const { return normalized_; }

    const std::vector<index_t>& row_ptr() const { return row_ptr_; }
    const std::vector<index_t>& col_idx() const { return col_idx_; }
    const std::vector<double>& values() const { return values_; }
    const std::vector<double>& row_norm() const { return row_norm_; }
    double row_norm(index_t i) const { return row_norm_[static_cast<std::size_t>(i)]; }
    index_t row_nnz(index_t i) const {
        return row_ptr_[static_cast<std::size_t>(i) + 1] - row_ptr_[static_cast<std::size_t>(i)];
    }

    /// a_i . x in storage order (host, O(theta)).
    double row_dot(index_t i, std::span<const double> x) const;
    /// y = A x and y = A^T x on the device (reference summation order).
    void multiply(std::span<const double> x, std::vector<double>& y) const;
    void multiply_transpose(std::span<const double> x, std::vector<double>& y) const;

    std::vector<Triplet> to_triplets() const;
    void flag_normalized();

    /// Device copy for fp64 (precision 0) or the fp32 layouts (1, 2).
    asyrk_system* device(int precision = 0) const;
    void release_device() const;

  private:
    friend std::pair<CsrMatrix, std::vector<double>> normalize_rows(const CsrMatrix&, std::span<const double>);
    void compute_norms();

    index_t m_ = 0;
    index_t n_ = 0;
    std::vector<index_t> row_ptr_;
    std::vector<index_t> col_idx_;
    std::vector<double> values_;
    std::vector<double> row_norm_;
    bool normalized_ = false;
    struct DeviceCache;
    mutable std::shared_ptr<DeviceCache> dev_;
};

/// Row scaling by 1/||a_i||; rows already within 1e-12 of unit norm are left
/// bit-identical (ref csr.cpp:113-138).
std::pair<CsrMatrix, std::vector<double>> normalize_rows(const CsrMatrix& A, std::span<const double> b);

struct Residuals {
    std::vector<double> r;  // Ax - b (left empty by the device path unless requested)
    double r_sq;            // ||Ax - b||^2
    double grad_sq;         // ||A^T (Ax - b)||^2
};

/// r_sq and grad_sq on the device, in the reference's summation order.
Residuals residuals(const CsrMatrix& A, std::span<const double> x, std::span<const double> b);

}  // namespace asyrk
