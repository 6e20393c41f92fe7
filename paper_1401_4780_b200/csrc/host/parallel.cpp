// Drop-in solve_parallel / sweep_threads (ref/src/parallel.cpp:220-506):
// validation and config echo on the host, everything else on the device
// through the C ABI (system.cu).
#include "asyrk/parallel.hpp"

#include <algorithm>

#include "asyrk/dense.hpp"
#include "asyrk/error.hpp"
#include "asyrk_cuda.h"
#include "common.hpp"
#include "json.hpp"

namespace asyrk {

namespace {

std::string run_config_json(const RunConfig& cfg, index_t m, index_t n, const DeviceOptions& dev) {
    json::Object c;
    c["solver"] = "asyrk_parallel";
    c["m"] = m;
    c["n"] = n;
    c["threads"] = cfg.threads;
    c["gamma"] = cfg.gamma;
    c["epochs"] = cfg.epochs;
    c["target_r_sq"] = cfg.target_r_sq;
    c["variant"] = cfg.variant == UpdateVariant::full_row ? "full_row" : "single_component";
    c["sampling"] = dev.norm_proportional ? "norm_proportional"
                    : cfg.sampling == ParSampling::slice_shuffle ? "slice_shuffle"
                                                                 : "with_replacement";
    c["seed"] = cfg.seed;
    c["snapshot_interval"] = cfg.snapshot_interval;
    c["epoch_updates"] = m;
    c["dist_oracle"] = cfg.x_star ? "x_star" : (cfg.projector ? "projector" : "none");
    c["device"] = "sm_100a";
    c["worker"] = cfg.threads == 1 ? "deterministic" : "warp";
    c["precision"] = dev.precision == 0 ? "fp64" : dev.precision == 1 ? "fp32" : "fp32_values_fp64_x";
    return json::dump(json::Value(std::move(c)));
}

asyrk_run_config to_c(const RunConfig& cfg, const DeviceOptions& dev) {
    asyrk_run_config c{};
    c.threads = cfg.threads;
    c.gamma = cfg.gamma;
    c.epochs = cfg.epochs;
    c.target_r_sq = cfg.target_r_sq;
    c.variant = cfg.variant == UpdateVariant::full_row ? ASYRK_FULL_ROW : ASYRK_SINGLE_COMPONENT;
    c.sampling = dev.norm_proportional                          ? ASYRK_NORM_PROPORTIONAL
                 : cfg.sampling == ParSampling::slice_shuffle ? ASYRK_SLICE_SHUFFLE
                                                               : ASYRK_WITH_REPLACEMENT;
    c.seed = cfg.seed;
    c.snapshot_interval = cfg.snapshot_interval;
    c.x_star = cfg.x_star ? cfg.x_star->data() : nullptr;
    c.precision = dev.precision;
    c.allow_unnormalized = dev.norm_proportional ? 1 : 0;
    c.record_every_boundary = dev.record_every_boundary ? 1 : 0;
    c.det_reassociate = dev.det_reassociate ? 1 : 0;
    return c;
}

}  // namespace

Trace solve_parallel(const CsrMatrix& A, std::span<const double> b, std::span<const double> x0,
                     const RunConfig& cfg, InstrumentReport* instrument) {
    return solve_parallel(A, b, x0, cfg, instrument, DeviceOptions{});
}

Trace solve_parallel(const CsrMatrix& A, std::span<const double> b, std::span<const double> x0,
                     const RunConfig& cfg, InstrumentReport* instrument, const DeviceOptions& dev) {
    if (static_cast<index_t>(b.size()) != A.rows() || static_cast<index_t>(x0.size()) != A.cols())
        fail(ErrorCode::DimensionMismatch, "solve_parallel: b or x0 size mismatch");
    // a projector's distance is ||x - A^+ b||^2 on the device (full column rank)
    RunConfig dc = cfg;
    if (!dc.x_star && dc.projector) dc.x_star = &projector_point(*cfg.projector, A.cols());
    const int prec = cfg.threads == 1 ? 0 : dev.precision;
    asyrk_system* sys = A.device(prec);
    throw_status(asyrk_system_set_rhs(sys, b.data()));
    const asyrk_run_config c = to_c(dc, dev);
    const index_t interval = std::max<index_t>(cfg.snapshot_interval, 1);
    TraceBuffers tb(A.cols(), std::max<index_t>(cfg.epochs, 0) / interval + 2);
    asyrk_instrument_out rep{};
    throw_status(asyrk_system_solve(sys, x0.data(), &c, &tb.out, instrument ? &rep : nullptr));
    Trace t = tb.to_trace(dc.x_star != nullptr);
    t.config_echo = run_config_json(cfg, A.rows(), A.cols(), dev);
    if (instrument) {
        instrument->row_updates = rep.row_updates;
        instrument->increments = rep.increments;
        instrument->max_abs_error = rep.max_abs_error;
        instrument->tolerance = rep.tolerance;
        instrument->consistent = rep.consistent != 0;
    }
    return t;
}

SpeedupReport sweep_threads(const CsrMatrix& A, std::span<const double> b, std::span<const double> x0,
                            const RunConfig& cfg, std::span<const index_t> thread_list) {
    if (thread_list.empty()) fail(ErrorCode::InvalidArgument, "thread list is empty");
    if (std::find(thread_list.begin(), thread_list.end(), 1) == thread_list.end())
        fail(ErrorCode::InvalidArgument, "thread list must contain 1 (the speedup reference)");
    SpeedupReport rep;
    for (index_t t : thread_list) {
        RunConfig c = cfg;
        c.threads = t;
        const Trace tr = solve_parallel(A, b, x0, c);
        SpeedupEntry e;
        e.threads = t;
        e.wall_seconds = tr.epochs.back().wall_seconds;
        e.epochs = tr.epochs.back().epoch_index;
        e.final_r_sq = tr.epochs.back().r_sq;
        rep.entries.push_back(e);
    }
    double wall1 = 0.0;
    for (const SpeedupEntry& e : rep.entries)
        if (e.threads == 1) {
            wall1 = e.wall_seconds;
            break;
        }
    for (SpeedupEntry& e : rep.entries) e.speedup = e.wall_seconds > 0.0 ? wall1 / e.wall_seconds : 0.0;
    return rep;
}

std::string SpeedupReport::to_json() const {
    json::Array a;
    for (const SpeedupEntry& e : entries) {
        json::Object o;
        o["threads"] = e.threads;
        o["wall_seconds"] = e.wall_seconds;
        o["epochs"] = e.epochs;
        o["final_r_sq"] = e.final_r_sq;
        o["speedup"] = e.speedup;
        a.emplace_back(std::move(o));
    }
    return json::dump(json::Value(std::move(a)));
}

std::string SpeedupReport::to_csv() const {
    std::string out = "threads,wall_seconds,epochs,final_r_sq,speedup\n";
    for (const SpeedupEntry& e : entries)
        out += std::to_string(e.threads) + ',' + std::to_string(e.wall_seconds) + ',' + std::to_string(e.epochs) + ',' +
               std::to_string(e.final_r_sq) + ',' + std::to_string(e.speedup) + '\n';
    return out;
}

}  // namespace asyrk
