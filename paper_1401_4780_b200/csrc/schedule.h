// Host-driven monitor schedule of the asynchronous solves (single-RHS K2 and
// multi-RHS K2b).
//
// The reference's coordinator records "the latest boundary crossed" — it takes
// a snapshot whenever its previous residual evaluation is done, so boundaries
// go unrecorded while the workers run on (ref/src/parallel.cpp:388-408). A
// residual pass costs as much L2 traffic as most of a worker epoch on the GPU
// (two SpMVs over A), so here the coordinator decides WHICH boundaries to
// evaluate from the records it already has: with the residual decaying
// geometrically, the last two records give a rate and the number of snapshot
// intervals left until r_sq <= target; the next evaluation is placed at the
// first boundary at or after the predicted crossing (never more than max_gap
// intervals ahead; the next boundary when the crossing is at most 1 away,
// while fewer than two records exist, or when the residual did not drop).
// The residual decays faster early on, so a two-record rate predicts the
// crossing early, and the first boundary after an early prediction is still
// at or before the actual crossing (an integer boundary). (Round 2 first
// placed it at the last boundary BEFORE the prediction — one evaluation more
// per solve on every replayed trace, profiles/r02_schedule_replay.txt.)
// Near the stop every boundary is evaluated, so the stop is taken at the first
// evaluated boundary that meets the target, and no epoch runs past it. With
// target <= 0 (a fixed epoch budget) or record_every_boundary, every boundary
// is evaluated, the reference's snapshot_interval semantics.
//
// The decision inputs are the records' r_sq — for a sharded multi-RHS solve
// the all-reduced one — so every rank computes the same schedule.
#pragma once
#include <cmath>
#include "env.h"
#include <cstdlib>

namespace ak {

struct MonitorSchedule {
    double target = 0.0;
    bool every = false;
    long long max_gap = 24;
    long long b_prev = -1, b_last = -1;  // boundaries (in snapshot intervals) of the last two records
    double r_prev = 0.0, r_last = 0.0;

    void reset(double tgt, bool every_boundary) {
        target = tgt;
        static const long long env_gap = getenv("ASYRK_MONITOR_MAX_GAP") ? atoll(getenv("ASYRK_MONITOR_MAX_GAP")) : 24;
        static const bool env_every = env_flag("ASYRK_MONITOR_EVERY");
        max_gap = env_gap > 0 ? env_gap : 1;
        every = every_boundary || env_every || !(tgt > 0.0);
        b_prev = b_last = -1;
        r_prev = r_last = 0.0;
    }

    // a record at boundary b; returns the next boundary to evaluate (> b)
    long long push(long long b, double r_sq) {
        b_prev = b_last;
        r_prev = r_last;
        b_last = b;
        r_last = r_sq;
        return b + gap();
    }

    long long gap() const {
        if (every || b_prev < 0 || b_last <= b_prev) return 1;
        if (!(r_last > target) || !(r_last < r_prev) || !(r_prev > 0.0) || !std::isfinite(r_last)) return 1;
        const double rate = (std::log(r_last) - std::log(r_prev)) / (double)(b_last - b_prev);  // < 0
        const double left = (std::log(target) - std::log(r_last)) / rate;                        // > 0
        if (!(left > 1.0) || !std::isfinite(left)) return 1;
        long long g = (long long)std::ceil(left);  // the first boundary at or after the predicted crossing
        if (g < 1) g = 1;
        if (g > max_gap) g = max_gap;
        return g;
    }
};

}  // namespace ak
