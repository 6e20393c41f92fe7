// K6 — batched bounded-delay simulator (replaces simulate / monte_carlo_ratios,
// ref/src/delay_sim.cpp:71-270).
//
// One warp replays one run (Monte-Carlo: `runs` warps side by side, run r
// seeded base_seed + r as in delay_sim.cpp:249-251); a single `simulate` uses
// a whole CTA for its run. The recursion is a serial chain; warp 0 of a run
// replays it: lane 0 draws from the reference's own generator
// (std::mt19937_64 restated on the device, state in shared memory), lanes
// load the row / column entries and form products in parallel, and the
// serial sums (stale residual, the LiveResidual running r_sq) are replayed in
// the reference's order from shuffles, with explicitly rounded intrinsics —
// so every trace record, probe, event, history row and final_x is
// bit-identical to the reference. The run's iterate, ring of tau + 1
// iterates (delay_sim.cpp:100-104) and LiveResidual r live in shared memory
// when they fit. The epoch-boundary residual passes (rows, then columns in
// make_csc order) use every thread of the run. A is read from the fp64 row
// records and the plain CSC (serial walks) and the SELL-32 copies (passes).
#include "kernels.h"

namespace ak {

namespace {

constexpr int kMtN = 312, kMtM = 156;

// std::mt19937_64 (C++ [rand.eng.mers] / [rand.predef]), seeded through
// splitmix64(seed ^ stream) as make_stream does (ref rng.hpp:14-25)
__device__ __forceinline__ unsigned long long splitmix64(unsigned long long x) {
    x += 0x9e3779b97f4a7c15ULL;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
}

struct DevMt {
    unsigned long long* s;  // kMtN words (shared memory)
    int idx;

    __device__ void seed(unsigned long long v) {
        s[0] = v;
        for (int i = 1; i < kMtN; ++i) s[i] = 6364136223846793005ULL * (s[i - 1] ^ (s[i - 1] >> 62)) + (unsigned)i;
        idx = kMtN;
    }
    __device__ void refill() {
        const unsigned long long up = 0xFFFFFFFF80000000ULL, lo = 0x7FFFFFFFULL, a = 0xB5026F5AA96619E9ULL;
        for (int i = 0; i < kMtN; ++i) {
            const unsigned long long y = (s[i] & up) | (s[i + 1 < kMtN ? i + 1 : 0] & lo);
            unsigned long long v = s[i + kMtM < kMtN ? i + kMtM : i + kMtM - kMtN] ^ (y >> 1);
            if (y & 1ULL) v ^= a;
            s[i] = v;
        }
        idx = 0;
    }
    __device__ unsigned long long next() {
        if (idx >= kMtN) refill();
        unsigned long long x = s[idx++];
        x ^= (x >> 29) & 0x5555555555555555ULL;
        x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
        x ^= (x << 37) & 0xFFF7EEE000000000ULL;
        x ^= x >> 43;
        return x;
    }
    // uniform_below: rejection, then modulo (rng.hpp:26-33)
    __device__ unsigned long long below(unsigned long long n) {
        const unsigned long long lim = ~0ULL - ~0ULL % n;
        for (;;) {
            const unsigned long long v = next();
            if (v < lim) return v % n;
        }
    }
};

struct Rows {  // SELL-32 rows: entry t of row i at grp_off[i/32] + i%32 + 32 t (CSR order)
    const CscDev& R;
    __device__ long long base(long long i) const { return __ldg(R.grp_off + (i >> 5)) + (i & 31); }
    __device__ int len(long long i) const { return __ldg(R.col_len + i); }
    __device__ int col(long long e) const { return __ldg(R.row + e); }
    __device__ double val(long long e) const { return __ldg(static_cast<const double*>(R.val) + e); }
};

// a_i^T x in storage order (csr.cpp:65-70)
__device__ __forceinline__ double row_dot(const Rows& rw, long long i, const double* x) {
    const long long b0 = rw.base(i);
    const int l = rw.len(i);
    double s = 0.0;
    for (int t = 0; t < l; ++t) {
        const long long e = b0 + 32ll * t;
        s = __dadd_rn(s, __dmul_rn(rw.val(e), x[rw.col(e)]));
    }
    return s;
}

// LiveResidual::bump (delay_sim.cpp:35-44) of column t over the plain CSC
// (make_csc order, rows ascending), by the whole warp: lane u holds entry u
// of a 32-entry chunk (the rows of a column are distinct, so the loads and
// the r updates run in parallel) and every lane replays the serial r_sq
// chain -old^2 +new^2 in entry order from shuffles. Returns the new r_sq
// (warp-uniform).
__device__ __forceinline__ double warp_bump(const SimArgs& a, int t, double delta, double* rl, double rsq, int lane) {
    const long long q1 = __ldg(a.col_ptr + t + 1);
    for (long long q0 = __ldg(a.col_ptr + t); q0 < q1; q0 += 32) {
        const long long q = q0 + lane;
        const bool act = q < q1;
        double o2 = 0.0, n2 = 0.0;
        if (act) {
            const int r = __ldg(a.csc_row + q);
            const double old = rl[r];
            const double nv = __dadd_rn(old, __dmul_rn(__ldg(a.csc_val + q), delta));
            rl[r] = nv;
            o2 = __dmul_rn(old, old);
            n2 = __dmul_rn(nv, nv);
        }
        const int lim = (int)min(32ll, q1 - q0);
        for (int u = 0; u < lim; ++u) {
            rsq = __dsub_rn(rsq, __shfl_sync(FULL, o2, u));
            rsq = __dadd_rn(rsq, __shfl_sync(FULL, n2, u));
        }
    }
    __syncwarp();  // the next column may touch the same rows
    return rsq;
}

// a_i^T x - b_i (stale_residual, kaczmarz.hpp:48-60) from the contiguous fp64
// row record, by the whole warp: products in parallel, the storage-order sum
// replayed from shuffles. The record's b_i is a bit copy of b[i].
__device__ __forceinline__ double warp_residual(const double* v, const int32_t* c, int len, const double* x, double bi,
                                                int lane) {
    double s = 0.0;
    for (int c0 = 0; c0 < len; c0 += 32) {
        const int u = c0 + lane;
        const double p = u < len ? __dmul_rn(__ldg(v + u), x[__ldg(c + u)]) : 0.0;
        const int lim = min(32, len - c0);
        for (int q = 0; q < lim; ++q) s = __dadd_rn(s, __shfl_sync(FULL, p, q));
    }
    return __dsub_rn(s, bi);
}

template <bool CTA>
__device__ __forceinline__ void run_sync() {
    if (CTA)
        __syncthreads();
    else
        __syncwarp();
}

// ||x - xd||^2 by the run's threads (strided partial sums, fixed-order tree):
// the SolutionProjector distance for a full-column-rank A (dense.hpp), equal
// to the reference's SVD-based dist_sq up to rounding; returned to every thread
template <bool CTA>
__device__ double run_dist(const double* x, const double* xd, long long n, int tid, int nthr) {
    double s = 0.0;
    for (long long q = tid; q < n; q += nthr) {
        const double d = x[q] - xd[q];
        s = fma(d, d, s);
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(FULL, s, o);
    if (!CTA) return s;
    __shared__ double red[8];
    __syncthreads();
    if ((tid & 31) == 0) red[tid >> 5] = s;
    __syncthreads();
    double t = 0.0;
    for (int w = 0; w < (nthr >> 5); ++w) t += red[w];
    __syncthreads();
    return t;
}

// residuals (csr.cpp:140-160) of x by every thread of the run: rt = Ax - b,
// gt = A^T rt; returns {r_sq, grad_sq} on thread 0 (serial sums)
template <bool CTA>
__device__ void run_residuals(const SimArgs& a, const Rows& rw, const double* x, double* rt, double* gt, int tid,
                              int nthr, double& r_sq, double& g_sq) {
    for (long long i = tid; i < a.m; i += nthr) rt[i] = __dsub_rn(row_dot(rw, i, x), a.b[i]);
    run_sync<CTA>();
    for (long long q = tid; q < a.n; q += nthr) {  // positions of the sigma-sorted column copy
        const long long j = a.C.col(q);
        const long long c0 = __ldg(a.C.grp_off + (q >> 5)) + (q & 31);
        const int cl = __ldg(a.C.col_len + q);
        const double* cv = static_cast<const double*>(a.C.val);
        double g = 0.0;
        for (int q = 0; q < cl; ++q) {
            const long long e = c0 + 32ll * q;
            g = __dadd_rn(g, __dmul_rn(__ldg(cv + e), rt[__ldg(a.C.row + e)]));
        }
        gt[j] = g;
    }
    run_sync<CTA>();
    if (tid == 0) {
        double s = 0.0, q = 0.0;
        for (long long i = 0; i < a.m; ++i) s = __dadd_rn(s, __dmul_rn(rt[i], rt[i]));
        for (long long j = 0; j < a.n; ++j) q = __dadd_rn(q, __dmul_rn(gt[j], gt[j]));
        r_sq = s;
        g_sq = q;
    }
}

}  // namespace

template <bool CTA>
__global__ void __launch_bounds__(256) sim_kernel(SimArgs a) {
    extern __shared__ __align__(16) unsigned char sm_raw[];
    __shared__ int stop_flag[8];
    const int wib = threadIdx.x >> 5;
    const int tid = CTA ? (int)threadIdx.x : (int)(threadIdx.x & 31);
    const int nthr = CTA ? (int)blockDim.x : 32;
    const long long run = CTA ? (long long)blockIdx.x : (long long)blockIdx.x * (blockDim.x >> 5) + wib;
    if (run >= a.runs) return;  // warp- (or block-) uniform
    const int slot = CTA ? 0 : wib;
    const int lane = threadIdx.x & 31;
    const long long m = a.m, n = a.n;
    const long long ring_len = a.tau + 1;
    // per run: mt state, then (smem_state) the hot doubles x | ring | LiveResidual r
    unsigned char* mine = sm_raw + (size_t)slot * (kMtN * 8 + (a.smem_state ? (size_t)a.hot * 8 : 0));
    DevMt g{reinterpret_cast<unsigned long long*>(mine), kMtN};
    double* gw = a.work + run * a.work_stride;  // global: [hot | rt m | gt n]
    double* x = a.smem_state ? reinterpret_cast<double*>(mine + kMtN * 8) : gw;
    double* ring = a.tau == 0 ? x : x + n;  // tau = 0: the ring's only slot is always the current iterate
    double* rl = x + n + (a.tau == 0 ? 0 : ring_len * n);  // LiveResidual r
    double* rt = gw + a.hot;
    double* gt = rt + m;
    const Rows rw{a.R};
    const bool probing = a.probe_every > 0 && a.probe_r_sq;  // LiveResidual maintained
    const bool probe_any = a.probe_every > 0 && (a.probe_r_sq || a.probe_d != nullptr);
    const bool rec_out = run == 0 && a.rec != nullptr;
    double* probe = a.probe ? a.probe + run * a.probe_stride : nullptr;
    double* probe_d = a.probe_d ? a.probe_d + run * a.probe_stride : nullptr;
    const unsigned long long t0 = globaltimer_ns();

    for (long long q = tid; q < n; q += nthr) {
        x[q] = a.x0[q];
        if (a.tau != 0) ring[q] = a.x0[q];
    }
    if (tid == 0) {
        g.seed(splitmix64(a.seed0 + (unsigned long long)run));
        stop_flag[slot] = 0;
    }
    run_sync<CTA>();

    long long nrec = 0, nprobe = 0, nev = 0;
    double live_rsq = 0.0;
    // record(epoch, updates) + LiveResidual recompute, delay_sim.cpp:144-166, :218-221
    auto boundary = [&](long long epoch, long long updates, bool recompute) {
        double r_sq = 0.0, g_sq = 0.0;
        run_residuals<CTA>(a, rw, x, rt, gt, tid, nthr, r_sq, g_sq);
        const double dist = (rec_out && a.xdist) ? run_dist<CTA>(x, a.xdist, n, tid, nthr) : -1.0;
        if (tid == 0) {
            if (!isfinite(r_sq) || !isfinite(g_sq)) {
                a.status[run] = 8;  // ASYRK_E_NonFinite
                a.fail_updates[run] = updates;
                stop_flag[slot] = 1;
            } else if (rec_out) {
                if (nrec < a.rec_cap) {
                    DevRecord rc;
                    rc.epoch = epoch;
                    rc.updates = updates;
                    rc.r_sq = r_sq;
                    rc.grad_sq = g_sq;
                    rc.dist_sq = dist;
                    rc.t_ns = globaltimer_ns() - t0;
                    a.rec[nrec] = rc;
                }
                ++nrec;
            }
        }
        if (recompute) {  // LiveResidual::recompute == the rows pass above, summed the same way
            for (long long i = tid; i < m; i += nthr) rl[i] = rt[i];
            if (tid < 32) live_rsq = __shfl_sync(FULL, r_sq, 0);
        }
        run_sync<CTA>();
    };
    auto do_probe = [&](long long jj) {
        if (tid == 0 && probe) probe[nprobe] = live_rsq;
        if (probe_d) {
            const double d = run_dist<CTA>(x, a.xdist, n, tid, nthr);
            if (tid == 0) probe_d[nprobe] = d;
        }
        ++nprobe;
    };

    boundary(0, 0, probing);  // LiveResidual ctor recompute(A, x0) + record(0, 0)
    if (!stop_flag[slot] && probe_any) do_probe(0);

    for (long long j = 0; j < a.iterations && !stop_flag[slot]; ++j) {
        if (tid < 32) {  // warp 0 of the run replays iteration j; lane 0 owns the generator
            long long i = 0, k = 0, pick = 0;
            if (lane == 0) {  // draw order: row, delay (uniform_random), component (single)
                i = (long long)g.below((unsigned long long)m);
                if (a.delay_kind == 1) {
                    const long long d = (long long)g.below((unsigned long long)(a.tau + 1));
                    k = j - d > 0 ? j - d : 0;
                } else {
                    k = j - a.tau > 0 ? j - a.tau : 0;
                }
                if (a.variant == 0) pick = (long long)g.below((unsigned long long)row_ref(a.L, i).len);
            }
            i = __shfl_sync(FULL, i, 0);
            k = __shfl_sync(FULL, k, 0);
            pick = __shfl_sync(FULL, pick, 0);
            const RowRef rr = row_ref(a.L, i);
            const double* rv = rec_vals<double>(rr);
            const int32_t* rc = rec_cols<double>(rr);
            const int theta = rr.len;
            const double* xr = ring + (a.tau == 0 ? 0 : (k % ring_len) * n);
            const double res = warp_residual(rv, rc, theta, xr, rec_b(rr), lane);  // stale_residual
            long long ev_t;
            double ev_step;
            if (a.variant == 0) {  // single_component
                const int t = __ldg(rc + pick);
                const double delta = __dmul_rn(__dmul_rn(__dmul_rn(-a.gamma, (double)theta), __ldg(rv + pick)), res);
                if (lane == 0) x[t] = __dadd_rn(x[t], delta);
                if (probing) live_rsq = warp_bump(a, t, delta, rl, live_rsq, lane);
                ev_t = t;
                ev_step = delta;
            } else {  // full_row: row_coef + apply_row, kaczmarz.hpp:63-80 (distinct columns)
                const double nrm = a.row_norm[i];
                const double c = __ddiv_rn(__dmul_rn(a.gamma, res), __dmul_rn(nrm, nrm));
                for (int u = lane; u < theta; u += 32) {
                    const int t = __ldg(rc + u);
                    x[t] = __dsub_rn(x[t], __dmul_rn(c, __ldg(rv + u)));
                }
                if (probing)
                    for (int u = 0; u < theta; ++u)
                        live_rsq = warp_bump(a, __ldg(rc + u), __dmul_rn(-c, __ldg(rv + u)), rl, live_rsq, lane);
                ev_t = -1;  // kAllComponents
                ev_step = c;
            }
            if (lane == 0 && run == 0 && a.ev && nev < a.max_events) {
                a.ev[nev] = SimEventDev{j, i, ev_t, k, ev_step};
                ++nev;
            }
        }
        run_sync<CTA>();
        if (a.tau != 0) {  // ring[(j + 1) % (tau + 1)] = x
            double* dst = ring + ((j + 1) % ring_len) * n;
            for (long long q = tid; q < n; q += nthr) dst[q] = x[q];
            run_sync<CTA>();
        }
        const long long done = j + 1;
        if (done % m == 0) boundary(done / m, done, probing);
        if (stop_flag[slot]) break;
        if (probe_any && done % a.probe_every == 0) do_probe(done);
    }
    if (!stop_flag[slot] && a.iterations % m != 0) boundary(a.iterations / m + 1, a.iterations, false);
    if (a.smem_state && run == 0) {  // final x and the ring back to global memory for the host
        run_sync<CTA>();
        for (long long q = tid; q < a.hot; q += nthr) gw[q] = x[q];
    }
    if (tid == 0) {
        if (run == 0 && a.nrec) *a.nrec = nrec;
        if (run == 0 && a.nev) *a.nev = nev;
        if (run == 0 && a.nprobe) *a.nprobe = nprobe;
    }
}

// mean_r_sq[j] = (sum over runs, in run order) * (1 / runs), delay_sim.cpp:247-258,
// then ratios[j] = mean[j+1] / mean[j] with the reference's zero rules (:260-268)
__global__ void sim_mean_kernel(const double* probe, long long probe_stride, long long runs, long long K, double* mean) {
    const long long j = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (j > K) return;
    double s = 0.0;
    for (long long r = 0; r < runs; ++r) s = __dadd_rn(s, probe[r * probe_stride + j]);
    mean[j] = __dmul_rn(s, __ddiv_rn(1.0, (double)runs));
}

__global__ void sim_ratio_kernel(const double* mean, long long K, double* ratios) {
    const long long j = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= K) return;
    const double a = mean[j], c = mean[j + 1];
    ratios[j] = a == 0.0 ? (c == 0.0 ? 1.0 : __longlong_as_double(0x7ff0000000000000LL)) : __ddiv_rn(c, a);
}

static long long sim_hot_doubles(long long m, long long n, long long tau) {
    return n * (tau == 0 ? 1 : tau + 2) + m;  // x | ring | LiveResidual r
}

size_t sim_work_doubles(long long m, long long n, long long tau) {
    return (size_t)sim_hot_doubles(m, n, tau) + (size_t)m + (size_t)n;  // + residual scratch rt, gt
}

// The recursion is a serial latency chain per run (the LiveResidual r_sq
// chain, store -> load through r): its state lives in shared memory when it
// fits (up to 4 runs per block in warp mode).
void launch_sim(const SimArgs& a0, bool cta_per_run, cudaStream_t s) {
    SimArgs a = a0;
    a.hot = sim_hot_doubles(a.m, a.n, a.tau);
    constexpr size_t kBudget = 200u << 10;
    const size_t per_run = kMtN * 8 + (size_t)a.hot * 8;
    if (cta_per_run) {
        a.smem_state = per_run <= kBudget;
        const size_t smem = a.smem_state ? per_run : kMtN * 8;
        cudaFuncSetAttribute(sim_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        sim_kernel<true><<<(unsigned)a.runs, 256, smem, s>>>(a);
    } else {
        int wpb = 4;
        while (wpb > 1 && per_run * wpb > kBudget) wpb >>= 1;
        a.smem_state = per_run * wpb <= kBudget;
        const size_t smem = (size_t)wpb * (a.smem_state ? per_run : kMtN * 8);
        cudaFuncSetAttribute(sim_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        sim_kernel<false><<<(unsigned)((a.runs + wpb - 1) / wpb), 32 * wpb, smem, s>>>(a);
    }
}

void launch_sim_mean(const double* probe, long long probe_stride, long long runs, long long K, double* mean,
                     double* ratios, cudaStream_t s) {
    sim_mean_kernel<<<(unsigned)((K + 1 + 127) / 128), 128, 0, s>>>(probe, probe_stride, runs, K, mean);
    if (K > 0) sim_ratio_kernel<<<(unsigned)((K + 127) / 128), 128, 0, s>>>(mean, K, ratios);
}

}  // namespace ak
