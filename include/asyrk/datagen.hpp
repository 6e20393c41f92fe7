// Instance types of the reference generator (ref/include/asyrk/datagen.hpp:11-25),
// used by the instance directory I/O (asyrk/io.hpp). The reference's
// gen_sparse_gaussian itself is not part of this build; BASELINE-shaped
// systems come from asyrk_generate_fixed_theta (include/asyrk_datagen.h).
#pragma once

#include <cstdint>
#include <optional>
#include <vector>

#include "asyrk/csr.hpp"

namespace asyrk {

struct GenSpec {
    index_t m = 0;
    index_t n = 0;
    double delta = 0.0;        // target nonzero fraction
    std::uint64_t seed = 0;
    bool consistent = true;
    double noise_level = 0.0;  // residual magnitude when inconsistent
};

struct Instance {
    CsrMatrix A;  // rows normalized
    std::vector<double> b;
    std::optional<std::vector<double>> x_star;  // present only when consistent
    GenSpec spec;
};

}  // namespace asyrk
