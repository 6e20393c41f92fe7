// CSR from coordinate arrays (the pybind drop-in path): from_triplets'
// semantics (ref csr.cpp:9-63: bounds, duplicates, zero values dropped, row
// norms) without the intermediate Triplet vector, with the passes over the
// entries in parallel when the input is already in (row, column) order.
#pragma once
#include <cstddef>
#include <span>
#include <utility>
#include <vector>

#include "asyrk/csr.hpp"

namespace asyrk {
CsrMatrix csr_from_coo(index_t m, index_t n, const index_t* rows, const index_t* cols, const double* vals,
                       std::size_t nnz);
// normalize_rows(csr_from_coo(...), b) without the copy of A (the arrays are
// scaled in place); the same matrix, b and errors
std::pair<CsrMatrix, std::vector<double>> csr_from_coo_normalized(index_t m, index_t n, const index_t* rows,
                                                                  const index_t* cols, const double* vals,
                                                                  std::size_t nnz, std::span<const double> b);
}
