// Drop-in rk_solve (ref/src/kaczmarz.cpp:128-227) and AliasTable
// (kaczmarz.cpp:14-61): the solve runs on the device's deterministic worker.
#include "asyrk/kaczmarz.hpp"

#include "asyrk/dense.hpp"
#include "asyrk/error.hpp"
#include "asyrk_cuda.h"
#include "common.hpp"
#include "json.hpp"

namespace asyrk {

AliasTable::AliasTable(std::span<const double> weights) {
    const std::size_t n = weights.size();
    if (n == 0) fail(ErrorCode::InvalidArgument, "alias table needs weights");
    double total = 0.0;
    for (double w : weights) {
        if (!(w >= 0.0)) fail(ErrorCode::InvalidArgument, "alias weights must be >= 0");
        total += w;
    }
    if (total <= 0.0) fail(ErrorCode::InvalidArgument, "alias weights sum to zero");
    prob_.assign(n, 0.0);
    alias_.assign(n, 0);
    std::vector<double> scaled(n);
    std::vector<index_t> lo, hi;  // under-full / over-full columns, used as stacks
    for (std::size_t k = 0; k < n; ++k) {
        scaled[k] = weights[k] * static_cast<double>(n) / total;
        (scaled[k] < 1.0 ? lo : hi).push_back(static_cast<index_t>(k));
    }
    while (!lo.empty() && !hi.empty()) {
        const index_t s = lo.back();
        lo.pop_back();
        const index_t l = hi.back();
        prob_[static_cast<std::size_t>(s)] = scaled[static_cast<std::size_t>(s)];
        alias_[static_cast<std::size_t>(s)] = l;
        scaled[static_cast<std::size_t>(l)] -= 1.0 - scaled[static_cast<std::size_t>(s)];
        if (scaled[static_cast<std::size_t>(l)] < 1.0) {
            hi.pop_back();
            lo.push_back(l);
        }
    }
    for (index_t k : hi) prob_[static_cast<std::size_t>(k)] = 1.0;
    for (index_t k : lo) prob_[static_cast<std::size_t>(k)] = 1.0;
}

index_t AliasTable::sample(std::mt19937_64& gen) const {
    const index_t k = static_cast<index_t>(uniform_below(gen, static_cast<std::uint64_t>(prob_.size())));
    return uniform_unit(gen) < prob_[static_cast<std::size_t>(k)] ? k : alias_[static_cast<std::size_t>(k)];
}

static const char* sampling_label(Sampling s) {
    switch (s) {
        case Sampling::uniform: return "uniform";
        case Sampling::norm_proportional: return "norm_proportional";
        case Sampling::shuffle: return "shuffle";
    }
    return "?";
}

Trace rk_solve(const CsrMatrix& A, std::span<const double> b, std::span<const double> x0, const RkConfig& cfg) {
    const index_t m = A.rows(), n = A.cols();
    if (static_cast<index_t>(b.size()) != m || static_cast<index_t>(x0.size()) != n)
        fail(ErrorCode::DimensionMismatch, "rk_solve: b or x0 size mismatch");
    if (cfg.sampling == Sampling::uniform && !A.is_normalized())
        fail(ErrorCode::NotNormalized,
             "uniform row sampling is only unbiased on normalized rows; use norm_proportional or normalize first");
    if (cfg.max_epochs < 0) fail(ErrorCode::InvalidArgument, "max_epochs must be >= 0");
    const std::vector<double>* xs =
        cfg.x_star ? cfg.x_star : (cfg.projector ? &projector_point(*cfg.projector, n) : nullptr);

    json::Object c;
    c["solver"] = "rk";
    c["m"] = m;
    c["n"] = n;
    c["max_epochs"] = cfg.max_epochs;
    c["target_r_sq"] = cfg.target_r_sq;
    c["seed"] = cfg.seed;
    c["sampling"] = sampling_label(cfg.sampling);
    c["dist_oracle"] = cfg.x_star ? "x_star" : (cfg.projector ? "projector" : "none");
    c["device"] = "sm_100a";

    asyrk_system* sys = A.device(0);
    throw_status(asyrk_system_set_rhs(sys, b.data()));
    asyrk_rk_config rc{};
    rc.max_epochs = cfg.max_epochs;
    rc.target_r_sq = cfg.target_r_sq;
    rc.seed = cfg.seed;
    rc.sampling = cfg.sampling == Sampling::uniform ? ASYRK_RK_UNIFORM
                  : cfg.sampling == Sampling::norm_proportional ? ASYRK_RK_NORM_PROPORTIONAL
                                                                 : ASYRK_RK_SHUFFLE;
    rc.x_star = xs ? xs->data() : nullptr;
    TraceBuffers tb(n, cfg.max_epochs + 1);
    throw_status(asyrk_system_rk_solve(sys, x0.data(), &rc, &tb.out));
    Trace t = tb.to_trace(xs != nullptr);
    t.config_echo = json::dump(json::Value(std::move(c)));
    return t;
}

}  // namespace asyrk
