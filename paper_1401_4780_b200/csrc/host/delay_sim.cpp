// simulate / monte_carlo_ratios / rate_fit (ref/src/delay_sim.cpp:71-338)
// over the C ABI: the recursion runs on the device (csrc/delay.cu).
#include "asyrk/delay_sim.hpp"
#include "asyrk/dense.hpp"

#include "asyrk/error.hpp"
#include "asyrk_cuda.h"
#include "asyrk/csr.hpp"
#include "common.hpp"
#include "json.hpp"

namespace asyrk {

namespace {

const char* delay_name(DelayModel::Kind k) {
    switch (k) {
        case DelayModel::Kind::fixed: return "fixed";
        case DelayModel::Kind::uniform_random: return "uniform_random";
        case DelayModel::Kind::max_staleness: return "max_staleness";
    }
    return "?";
}

asyrk_sim_config sim_config(const StepParams& params, const DelayModel& delay, index_t iterations,
                            std::uint64_t seed, SimVariant variant) {
    asyrk_sim_config c{};
    c.gamma = params.gamma;
    c.tau = delay.tau;
    c.delay = static_cast<int32_t>(delay.kind);
    c.variant = variant == SimVariant::full_row ? 1 : 0;
    c.iterations = iterations;
    c.seed = seed;
    return c;
}

void check_dims(const CsrMatrix& A, std::span<const double> b, std::span<const double> x0) {
    if (static_cast<index_t>(b.size()) != A.rows() || static_cast<index_t>(x0.size()) != A.cols())
        fail(ErrorCode::DimensionMismatch, "simulate: b or x0 size mismatch");
}

}  // namespace

SimRun simulate(const CsrMatrix& A, std::span<const double> b, std::span<const double> x0, const StepParams& params,
                const DelayModel& delay, index_t iterations, std::uint64_t seed, SimVariant variant,
                const SimOptions& opts) {
    check_dims(A, b, x0);
    asyrk_sim_config c = sim_config(params, delay, iterations, seed, variant);
    // the projector's distance runs on the device as ||x - A^+ b||^2 (full column rank)
    if (opts.projector) c.dist_point = projector_point(*opts.projector, A.cols()).data();
    c.probe_every = opts.probe_every;
    c.probe_r_sq = opts.probe_r_sq ? 1 : 0;
    c.probe_dist_sq = opts.probe_dist_sq ? 1 : 0;
    c.max_events = opts.max_events;
    const index_t m = A.rows(), n = A.cols();
    const index_t rec_cap = iterations > 0 ? iterations / m + 2 : 1;
    const index_t ev_cap = std::max<index_t>(0, std::min<index_t>(opts.max_events, std::max<index_t>(iterations, 0)));
    const index_t hist_cap = delay.tau >= 0 ? std::min<index_t>(delay.tau + 1, std::max<index_t>(iterations, 0) + 1) : 0;
    const bool probing = opts.probe_every > 0 && (opts.probe_r_sq || opts.probe_dist_sq);
    const index_t probe_cap = probing && iterations > 0 ? iterations / opts.probe_every + 1 : 0;

    std::vector<int64_t> ep(rec_cap), upd(rec_cap), ej(ev_cap), ei(ev_cap), et(ev_cap), ek(ev_cap), pit(probe_cap);
    std::vector<double> rs(rec_cap), gs(rec_cap), ds(rec_cap), wall(rec_cap), es(ev_cap), hist(hist_cap * n),
        prs(probe_cap), pds(probe_cap);
    SimRun run;
    run.params = params;
    run.trace.final_x.resize(static_cast<std::size_t>(n));
    asyrk_sim_out o{};
    o.trace = asyrk_trace_out{rec_cap, 0, ep.data(), rs.data(), gs.data(), ds.data(), wall.data(), upd.data(),
                              run.trace.final_x.data()};
    o.ev_cap = ev_cap;
    o.ev_j = ej.data();
    o.ev_i = ei.data();
    o.ev_t = et.data();
    o.ev_k = ek.data();
    o.ev_step = es.data();
    o.history_cap = hist_cap;
    o.history = hist.data();
    o.probe_cap = probe_cap;
    o.probe_iteration = pit.data();
    o.probe_r_sq = prs.data();
    o.probe_dist_sq = pds.data();
    asyrk_system* sys = A.device(0);  // cached fp64 device matrix, b replaced in place
    throw_status(asyrk_system_set_rhs(sys, b.data()));
    throw_status(asyrk_system_simulate(sys, x0.data(), &c, &o));

    json::Object cj;
    cj["solver"] = json::Value("simulate");
    cj["m"] = json::Value(m);
    cj["n"] = json::Value(n);
    cj["variant"] = json::Value(variant == SimVariant::full_row ? "full_row" : "single_component");
    cj["delay"] = json::Value(delay_name(delay.kind));
    cj["tau"] = json::Value(delay.tau);
    cj["gamma"] = json::Value(params.gamma);
    cj["iterations"] = json::Value(iterations);
    cj["seed"] = json::Value(static_cast<uint64_t>(seed));
    run.trace.config_echo = json::dump(json::Value(std::move(cj)));
    const index_t k = std::min<index_t>(o.trace.count, rec_cap);
    for (index_t r = 0; r < k; ++r) {
        EpochRecord e;
        e.epoch_index = ep[r];
        e.r_sq = rs[r];
        e.grad_sq = gs[r];
        if (opts.projector) e.dist_sq = ds[r];
        e.wall_seconds = wall[r];
        e.updates_applied = upd[r];
        run.trace.epochs.push_back(e);
    }
    for (index_t e = 0; e < std::min<index_t>(o.ev_count, ev_cap); ++e)
        run.events.push_back(UpdateEvent{ej[e], ei[e], et[e], ek[e], es[e]});
    for (index_t h = 0; h < std::min<index_t>(o.history_rows, hist_cap); ++h)
        run.history.emplace_back(hist.begin() + h * n, hist.begin() + (h + 1) * n);
    for (index_t p = 0; p < std::min<index_t>(o.probe_count, probe_cap); ++p) {
        run.probe_iteration.push_back(pit[p]);
        if (opts.probe_r_sq) run.probe_r_sq.push_back(prs[p]);
        if (opts.probe_dist_sq) run.probe_dist_sq.push_back(pds[p]);
    }
    return run;
}

MonteCarloRatios monte_carlo_ratios(const CsrMatrix& A, std::span<const double> b, std::span<const double> x0,
                                    const StepParams& params, const DelayModel& delay, index_t iterations,
                                    index_t runs, std::uint64_t base_seed, SimVariant variant) {
    if (runs < 100) fail(ErrorCode::InsufficientData, "need >= 100 runs for stable ratio estimates");
    check_dims(A, b, x0);
    asyrk_sim_config c = sim_config(params, delay, iterations, base_seed, variant);
    MonteCarloRatios out;
    out.mean_r_sq.resize(static_cast<std::size_t>(std::max<index_t>(iterations, 0)) + 1);
    out.ratios.resize(static_cast<std::size_t>(std::max<index_t>(iterations, 0)));
    asyrk_system* sys = A.device(0);
    throw_status(asyrk_system_set_rhs(sys, b.data()));
    throw_status(asyrk_system_monte_carlo_ratios(sys, x0.data(), &c, runs, out.mean_r_sq.data(), out.ratios.data()));
    return out;
}

RateFit rate_fit(std::span<const double> y, double stride) {
    RateFit f;
    throw_status(asyrk_rate_fit(y.data(), static_cast<int64_t>(y.size()), stride, &f.slope, &f.r2));
    return f;
}

}  // namespace asyrk
