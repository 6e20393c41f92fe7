// Test infrastructure only (oracle/_ref build). The reference's dense.cpp needs
// Eigen3, which is absent from this image; the hot path never calls it (it
// backs the optional SolutionProjector dist oracle and exact spectra). These
// stand-ins satisfy the linker and fail loudly if reached.
// Declarations: /root/reference/proj/include/asyrk/dense.hpp:21-54.
#include "asyrk/dense.hpp"
#include "asyrk/error.hpp"

namespace asyrk {

namespace {
[[noreturn]] void no_eigen(const char* what) {
    fail(ErrorCode::TooLarge, std::string(what) + ": dense SVD unavailable (Eigen3 absent in this build)");
}
}  // namespace

Spectrum dense_spectrum(const CsrMatrix&) { no_eigen("dense_spectrum"); }

SolutionProjector::SolutionProjector(const CsrMatrix&, std::vector<double>, index_t) {
    no_eigen("SolutionProjector");
}

std::vector<double> SolutionProjector::project(std::span<const double>) const {
    no_eigen("SolutionProjector::project");
}

double SolutionProjector::dist_sq(std::span<const double>) const {
    no_eigen("SolutionProjector::dist_sq");
}

std::vector<double> dense_min_norm_lstsq(const CsrMatrix&, std::span<const double>) {
    no_eigen("dense_min_norm_lstsq");
}

std::vector<std::vector<double>> to_dense(const CsrMatrix&) { no_eigen("to_dense"); }

}  // namespace asyrk
