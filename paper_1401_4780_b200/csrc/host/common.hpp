// Host-side glue shared by the drop-in entry points: caller-side trace
// buffers for the C ABI and their conversion into asyrk::Trace.
#pragma once

#include <vector>

#include "asyrk/csr.hpp"
#include "asyrk/trace.hpp"
#include "asyrk_cuda.h"

// opaque host CSR handle of the C ABI (include/asyrk_io.h)
struct asyrk_host_csr {
    asyrk::CsrMatrix A;
};

namespace asyrk {

struct TraceBuffers {
    std::vector<int64_t> epoch, updates;
    std::vector<double> r_sq, grad_sq, dist_sq, wall, final_x;
    asyrk_trace_out out{};

    TraceBuffers(index_t n, index_t cap) {
        if (cap < 1) cap = 1;
        const auto c = static_cast<std::size_t>(cap);
        epoch.resize(c);
        updates.resize(c);
        r_sq.resize(c);
        grad_sq.resize(c);
        dist_sq.resize(c);
        wall.resize(c);
        final_x.resize(static_cast<std::size_t>(n));
        out.cap = cap;
        out.epoch_index = epoch.data();
        out.r_sq = r_sq.data();
        out.grad_sq = grad_sq.data();
        out.dist_sq = dist_sq.data();
        out.wall_seconds = wall.data();
        out.updates_applied = updates.data();
        out.final_x = final_x.data();
    }

    Trace to_trace(bool has_dist) {
        Trace t;
        const auto k = static_cast<std::size_t>(out.count < out.cap ? out.count : out.cap);
        t.epochs.resize(k);
        for (std::size_t i = 0; i < k; ++i) {
            EpochRecord& e = t.epochs[i];
            e.epoch_index = epoch[i];
            e.r_sq = r_sq[i];
            e.grad_sq = grad_sq[i];
            if (has_dist) e.dist_sq = dist_sq[i];
            e.wall_seconds = wall[i];
            e.updates_applied = updates[i];
        }
        t.final_x = std::move(final_x);
        return t;
    }
};

}  // namespace asyrk
