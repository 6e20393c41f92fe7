// compute_stats / power_iteration_lambda_max on the device (ref/src/stats.cpp:
// 15-130), SystemStats JSON, and the step-size corollary (ref/src/stepsize.cpp:
// 26-82), scalar host math.
#include <algorithm>
#include <cmath>
#include <numbers>

#include "asyrk/dense.hpp"
#include "asyrk/error.hpp"
#include "asyrk/stepsize.hpp"
#include "asyrk_cuda.h"
#include "json.hpp"

namespace asyrk {

double power_iteration_lambda_max(const CsrMatrix& A, double tol, index_t max_iters) {
    double lam = 0.0;
    int64_t iters = 0;
    throw_status(asyrk_system_power_iteration(A.device(0), tol, max_iters, &lam, &iters));
    return lam;
}

SystemStats compute_stats(const CsrMatrix& A, const StatsOptions& opts) {
    if (!A.is_normalized())
        fail(ErrorCode::NotNormalized, "stats are defined for row-normalized matrices; call normalize_rows first");
    SystemStats s;
    s.theta.resize(static_cast<std::size_t>(A.rows()));
    asyrk_stats_out o{};
    o.theta = s.theta.data();
    throw_status(asyrk_system_compute_stats(A.device(0), opts.tol, opts.exact_spectral ? -1 : opts.max_power_iters, &o));
    s.m = o.m;
    s.n = o.n;
    s.delta = o.delta;
    s.mu = o.mu;
    s.nu = o.nu;
    s.alpha = o.alpha;
    s.frob_sq = o.frob_sq;
    s.l_max = o.l_max;
    s.l_res = o.l_res;
    if (opts.exact_spectral) {  // stats.cpp:136-140, dense spectrum from the device Jacobi SVD
        const Spectrum sp = dense_spectrum(A);
        s.lambda_max = sp.lambda_max;
        s.lambda_min = sp.lambda_min;
        s.sigma_r = sp.sigma_r;
    } else {
        s.lambda_max = o.lambda_max;
    }
    return s;
}

// ref stats.cpp:132-178 (field names and presence rules of the JSON object)
std::string SystemStats::to_json() const {
    json::Object j;
    j["m"] = json::Value(m);
    j["n"] = json::Value(n);
    j["delta"] = json::Value(delta);
    json::Array th;
    th.reserve(theta.size());
    for (index_t t : theta) th.emplace_back(t);
    j["theta"] = json::Value(std::move(th));
    j["mu"] = json::Value(mu);
    j["nu"] = json::Value(nu);
    j["alpha"] = json::Value(alpha);
    if (lambda_min) j["lambda_min"] = json::Value(*lambda_min);
    j["lambda_max"] = json::Value(lambda_max);
    j["frob_sq"] = json::Value(frob_sq);
    j["l_max"] = json::Value(l_max);
    j["l_res"] = json::Value(l_res);
    if (sigma_r) j["sigma_r"] = json::Value(*sigma_r);
    return json::dump(json::Value(std::move(j)));
}

SystemStats SystemStats::from_json(const std::string& text) {
    json::Value v;
    try {
        v = json::parse(text);
    } catch (const std::exception& e) {
        fail(ErrorCode::IoError, std::string("bad stats JSON: ") + e.what());
    }
    SystemStats s;
    try {
        if (!v.is_object()) throw std::runtime_error("not an object");
        const json::Object& o = v.object();
        s.m = o.at("m").integer();
        s.n = o.at("n").integer();
        s.delta = o.at("delta").number();
        for (const auto& t : o.at("theta").array()) s.theta.push_back(t.integer());
        s.mu = o.at("mu").integer();
        s.nu = o.at("nu").integer();
        s.alpha = o.at("alpha").number();
        if (o.count("lambda_min")) s.lambda_min = o.at("lambda_min").number();
        s.lambda_max = o.at("lambda_max").number();
        s.frob_sq = o.at("frob_sq").number();
        s.l_max = o.at("l_max").number();
        s.l_res = o.at("l_res").number();
        if (o.count("sigma_r")) s.sigma_r = o.at("sigma_r").number();
    } catch (const Error&) {
        throw;
    } catch (const std::exception& e) {
        fail(ErrorCode::IoError, std::string("bad stats JSON: ") + e.what());
    }
    return s;
}

double psi(double mu, double lambda_max, index_t tau, double rho, index_t m) {
    if (m < 1) fail(ErrorCode::InvalidArgument, "m must be >= 1");
    if (tau < 0) fail(ErrorCode::InvalidArgument, "tau must be >= 0");
    if (tau == 0) return mu;
    if (!(rho > 1.0)) fail(ErrorCode::InvalidRho, "rho must exceed 1 when tau > 0");
    const double t = static_cast<double>(tau);
    return mu + 2.0 * lambda_max * t * std::pow(rho, t) / static_cast<double>(m);
}

static void need_core(const SystemStats& s) {
    if (s.m <= 0 || s.mu <= 0 || s.alpha <= 0.0 || s.lambda_max <= 0.0)
        fail(ErrorCode::MissingStats, "need m, mu, alpha and lambda_max to evaluate step bounds");
}

GammaBounds gamma_bounds(const SystemStats& s, index_t tau, double rho) {
    need_core(s);
    if (!(rho > 1.0)) fail(ErrorCode::InvalidRho, "rho must exceed 1");
    const double m = static_cast<double>(s.m), t = static_cast<double>(tau), L = s.lambda_max;
    const double rt = std::pow(rho, t);
    GammaBounds g;
    g.b1 = 1.0 / psi(static_cast<double>(s.mu), L, tau, rho, s.m);
    g.b2 = m * (rho - 1.0) / (2.0 * L * rt * rho);
    g.b3 = m * std::sqrt((rho - 1.0) / (rt * (m * s.alpha * s.alpha + L * L * t * rt)));
    g.gamma = std::min({g.b1, g.b2, g.b3});
    return g;
}

StepParams corollary_params(const SystemStats& s, index_t tau) {
    need_core(s);
    if (tau < 0) fail(ErrorCode::InvalidArgument, "tau must be >= 0");
    const double m = static_cast<double>(s.m);
    const double lhs = 2.0 * std::numbers::e * s.lambda_max * static_cast<double>(tau + 1) / m;
    StepParams p;
    p.tau = tau;
    p.feasible = lhs <= 1.0;
    p.rho = 1.0 + lhs;
    p.psi = psi(static_cast<double>(s.mu), s.lambda_max, tau, p.rho, s.m);
    if (p.feasible) {
        p.gamma_bounds = gamma_bounds(s, tau, p.rho);
        p.gamma = 1.0 / p.psi;
        if (s.lambda_min) {
            p.rate_iter = rate_iteration(s, p.gamma, p.psi).per_iteration;
            p.rate_simplified = 1.0 - *s.lambda_min / (m * (static_cast<double>(s.mu) + 1.0));
        }
    }
    return p;
}

RateIteration rate_iteration(const SystemStats& s, double gamma, double psi_value) {
    if (!(gamma > 0.0)) fail(ErrorCode::InvalidGamma, "gamma must be positive");
    if (!(gamma < 2.0 / psi_value)) fail(ErrorCode::StepTooLarge, "gamma must stay below 2/psi for guaranteed progress");
    if (!s.lambda_min) fail(ErrorCode::MissingStats, "lambda_min required for rate");
    const double m = static_cast<double>(s.m);
    RateIteration r;
    r.per_iteration = 1.0 - *s.lambda_min * gamma * (2.0 - gamma * psi_value) / m;
    r.per_epoch = std::pow(r.per_iteration, m);
    return r;
}

ProbBound iteration_bound(const SystemStats& s, double x0_dist_sq, double epsilon, double eta) {
    if (!s.lambda_min || !(*s.lambda_min > 0.0)) fail(ErrorCode::ZeroLambdaMin, "the bound requires lambda_min > 0");
    if (!(epsilon > 0.0) || !(x0_dist_sq > 0.0)) fail(ErrorCode::InvalidArgument, "epsilon and x0_dist_sq must be > 0");
    if (!(eta > 0.0 && eta < 1.0)) fail(ErrorCode::InvalidArgument, "eta must lie in (0,1)");
    const double m = static_cast<double>(s.m), mu = static_cast<double>(s.mu);
    const double j = m * (mu + 1.0) / *s.lambda_min * std::abs(std::log(x0_dist_sq / (eta * epsilon)));
    ProbBound b;
    b.epsilon = epsilon;
    b.eta = eta;
    b.j_min = static_cast<index_t>(std::ceil(j));
    return b;
}

index_t max_feasible_tau(index_t m, double lambda_max) {
    return static_cast<index_t>(std::floor(static_cast<double>(m) / (2.0 * std::numbers::e * lambda_max))) - 1;
}

}  // namespace asyrk
