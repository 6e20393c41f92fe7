// Drop-in instance I/O (ref/include/asyrk/io.hpp:12-33): Matrix Market
// coordinate files (1-based, %.17g values), one-value-per-line vectors, and
// instance directories (A.mtx, b.txt, xstar.txt, meta.json). Same file bytes
// as the reference; parsing and formatting are multithreaded. Additionally a
// binary CSR cache (write_csr_cache / read_csr_cache) that reloads a matrix
// without text parsing.
#pragma once

#include <span>
#include <string>
#include <vector>

#include "asyrk/csr.hpp"
#include "asyrk/datagen.hpp"

namespace asyrk {

void write_matrix_market(const std::string& path, const CsrMatrix& A);
CsrMatrix read_matrix_market(const std::string& path);

void write_vector(const std::string& path, std::span<const double> v);
std::vector<double> read_vector(const std::string& path);

void write_text(const std::string& path, const std::string& text);
std::string read_text(const std::string& path);

void write_instance(const std::string& dir, const Instance& inst);
Instance read_instance(const std::string& dir);

/// Binary CSR cache: "ASYRKCSR", version, flags (bit 0: normalized), m, n,
/// nnz, then row_ptr, col_idx (int64), values, row_norm (fp64), little endian.
void write_csr_cache(const std::string& path, const CsrMatrix& A);
CsrMatrix read_csr_cache(const std::string& path);

}  // namespace asyrk
