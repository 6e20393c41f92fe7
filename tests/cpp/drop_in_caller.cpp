// A reference-style C++ caller of the drop-in API (include/asyrk/*.hpp), the
// way code written against the reference's headers uses it: triplets ->
// CsrMatrix -> normalize_rows, then rk_solve, solve_parallel (deterministic
// and warp workers), compute_stats (exact spectrum), the projector, lsq_solve
// and the trace JSON. Built and run by tests/test_host.py / test_gpu_parity.py;
// prints one "key value..." line per result for the Python side to check.
#include <cmath>
#include <cstdio>
#include <vector>

#include "asyrk/csr.hpp"
#include "asyrk/dense.hpp"
#include "asyrk/error.hpp"
#include "asyrk/kaczmarz.hpp"
#include "asyrk/lsq.hpp"
#include "asyrk/parallel.hpp"
#include "asyrk/stats.hpp"
#include "asyrk/stepsize.hpp"

using namespace asyrk;

int main() {
    std::setvbuf(stdout, nullptr, _IONBF, 0);
    // a small consistent system with unnormalized rows: 60 x 24, 6 entries per row
    const index_t m = 60, n = 24;
    std::vector<Triplet> t;
    std::vector<double> xs(n);
    for (index_t j = 0; j < n; ++j) xs[j] = std::sin(0.7 * j + 0.3);
    for (index_t i = 0; i < m; ++i)
        for (index_t q = 0; q < 6; ++q) {
            const index_t j = (i * 7 + q * 5 + (i * q) % 3) % n;
            bool dup = false;
            for (const Triplet& e : t)
                if (e.row == i && e.col == j) dup = true;
            if (!dup) t.push_back({i, j, std::cos(1.3 * i + 0.9 * q) + 0.1 * (q + 1)});
        }
    CsrMatrix A0 = CsrMatrix::from_triplets(t, m, n);
    std::vector<double> b0(m, 0.0);
    for (index_t i = 0; i < m; ++i) b0[i] = A0.row_dot(i, xs);
    auto [A, b] = normalize_rows(A0, b0);
    std::vector<double> x0(n, 0.0);

    RkConfig rk;
    rk.max_epochs = 30;
    rk.seed = 5;
    rk.x_star = &xs;
    Trace tr = rk_solve(A, b, x0, rk);
    std::printf("rk_final_x");
    for (double v : tr.final_x) std::printf(" %.17g", v);
    std::printf("\nrk_records %zu %.17g\n", tr.epochs.size(), tr.epochs.back().r_sq);

    RunConfig rc;
    rc.threads = 1;
    rc.epochs = 12;
    rc.seed = 9;
    Trace t1 = solve_parallel(A, b, x0, rc);
    std::printf("single_final_x");
    for (double v : t1.final_x) std::printf(" %.17g", v);
    std::printf("\n");

    RunConfig ra;
    ra.threads = 2;  // (a 60-row system: more concurrent rows than that diverge at gamma = 1)
    ra.epochs = 2000;
    ra.target_r_sq = 1e-24;
    ra.sampling = ParSampling::with_replacement;
    ra.seed = 3;
    InstrumentReport rep;
    Trace ta = solve_parallel(A, b, x0, ra, &rep);
    std::printf("async_r_sq %.17g consistent %d\n", ta.epochs.back().r_sq, rep.consistent ? 1 : 0);

    SystemStats st = compute_stats(A);
    std::printf("stats %lld %lld %.17g %.17g %.17g\n", (long long)st.mu, (long long)st.nu, st.alpha, st.lambda_max,
                st.lambda_min ? *st.lambda_min : -1.0);
    StepParams p = corollary_params(st, 1);
    std::printf("step %d %.17g\n", p.feasible ? 1 : 0, p.rho);

    SolutionProjector proj(A, b);
    RkConfig rp;
    rp.max_epochs = 10;
    rp.projector = &proj;
    Trace tp = rk_solve(A, b, x0, rp);
    double d = 0.0;
    for (index_t j = 0; j < n; ++j) d += (tp.final_x[j] - xs[j]) * (tp.final_x[j] - xs[j]);
    std::printf("projector %.17g %.17g %.17g\n", tp.epochs.back().dist_sq.value_or(-1.0), d, proj.dist_sq(tp.final_x));

    std::vector<double> bn(b);
    for (index_t i = 0; i < m; ++i) bn[i] += 0.05 * std::cos(3.1 * i);
    LsqConfig lc;
    lc.max_epochs = 20000;
    lc.target_r_sq = 1e-22;
    LsqResult lr = lsq_solve(A, bn, lc);
    const std::vector<double> xl = dense_min_norm_lstsq(A, bn);
    double e = 0.0;
    for (index_t j = 0; j < n; ++j) e += (lr.x_ls[j] - xl[j]) * (lr.x_ls[j] - xl[j]);
    std::printf("lsq %.17g %.17g\n", lr.grad_norm, std::sqrt(e));
    std::printf("trace_jsonl %zu\n", ta.to_jsonl().size());

    try {
        RunConfig bad;
        bad.threads = 0;
        (void)solve_parallel(A, b, x0, bad);
        std::printf("error none\n");
    } catch (const Error& err) {
        std::printf("error %s\n", error_code_name(err.code()));
    }
    return 0;
}
