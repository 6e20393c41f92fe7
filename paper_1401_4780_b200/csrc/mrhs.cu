// K2b / K3b — multi-right-hand-side AsyRK (BASELINE config 5; the reference
// is single-RHS, its oracle is k independent single-RHS solves sharing the
// row sequence).
//
// X (n x KL) and B (m x KL) are row-major fp32 with KL = the RHS columns this
// GPU owns (64/G for G GPUs). One warp projects one row for all KL columns:
// lanes own column pairs (float2) and, when KL < 64, several nonzeros are
// processed side by side ("slots"), so every gather of an X row and every
// red.global.add.v2.f32 back into it is a contiguous, coalesced 8*KL-byte
// access — the multi-RHS row turns the single-RHS random 8-byte gather into
// full-sector traffic.
//
//   res_c = a_i^T X[:, c] - B[i, c]          (per column c, fp32)
//   X[t, c] -= res_c / ||a_i||^2 * a_it      (t in supp a_i)
//
// Monitor: R = A X - B (warp per row, lanes over columns), G = A^T R (warp
// per column over a plain CSC, lanes over columns), block partials of
// ||R||_F^2, ||G||_F^2, ||X - X*||_F^2 in fp64. The partials are what a
// multi-GPU caller all-reduces (NCCL) before the stop decision.
#include "kernels.h"

namespace ak {

constexpr int kMrThreads = 256;

template <int KL>
struct MrGeom {
    static constexpr int GL = KL / 2;      // lanes per nonzero slot (float2 each)
    static constexpr int S = 32 / GL;      // nonzeros processed side by side
    static_assert(KL >= 2 && KL <= 64 && (KL & (KL - 1)) == 0, "KL must be a power of two in [2, 64]");
};

__device__ __forceinline__ float2 ld_x2(const float* p) { return __ldcg(reinterpret_cast<const float2*>(p)); }

template <int KL>
__global__ void __launch_bounds__(256) mrhs_worker_kernel(MrhsArgs a) {
    using G = MrGeom<KL>;
    const DevState* st = a.st;
    if (st->stop) return;
    const long long epoch = st->epoch;
    const long long span = chunk_span(st);
    if (span <= 0) return;
    const long long warp = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (warp >= a.W) return;
    const int lane = threadIdx.x & 31;
    const int slot = lane / G::GL, cl = lane % G::GL;
    const long long m = a.L.m;
    const long long total = span * m;
    const long long count = total / a.W + (warp < total % a.W ? 1 : 0);
    float* __restrict__ X = a.X;

    for (long long j0 = 0; j0 < count; j0 += 32) {
        // 32 rows per lane-parallel Philox draw (with replacement)
        const long long j = j0 + lane;
        const U4 rr = philox4x32(U4{(uint32_t)j, (uint32_t)(j >> 32), (uint32_t)warp, (uint32_t)epoch}, a.key0,
                                 a.key1);
        const long long myrow = (long long)bounded64(((uint64_t)rr.x << 32) | rr.y, (uint64_t)m);
        const int nq = (int)min(32ll, count - j0);
        for (int q = 0; q < nq; ++q) {
            const long long i = __shfl_sync(FULL, myrow, q);
            const RowRef r = row_ref(a.L, i);
            const float* vals = rec_vals<float>(r);
            const int32_t* cols = rec_cols<float>(r);
            const int len = r.len;
            float2 acc = make_float2(0.f, 0.f);
            for (int t0 = 0; t0 < len; t0 += G::S) {
                const int t = t0 + slot;
                if (t < len) {
                    const float v = __ldg(vals + t);
                    const float2 xv = ld_x2(X + (size_t)__ldg(cols + t) * KL + 2 * cl);
                    acc.x = fmaf(v, xv.x, acc.x);
                    acc.y = fmaf(v, xv.y, acc.y);
                }
            }
#pragma unroll
            for (int o = G::GL; o < 32; o <<= 1) {
                acc.x += __shfl_xor_sync(FULL, acc.x, o);
                acc.y += __shfl_xor_sync(FULL, acc.y, o);
            }
            const float2 bv = __ldg(reinterpret_cast<const float2*>(a.B + (size_t)i * KL) + cl);
            const float inv = (float)rec_inv(r);
            const float g = (float)a.gamma;
            const float cx = g * (acc.x - bv.x) * inv, cy = g * (acc.y - bv.y) * inv;
            for (int t0 = 0; t0 < len; t0 += G::S) {
                const int t = t0 + slot;
                if (t < len) {
                    const float v = __ldg(vals + t);
                    float2* dst = reinterpret_cast<float2*>(X + (size_t)__ldg(cols + t) * KL + 2 * cl);
                    atomicAdd(dst, make_float2(-cx * v, -cy * v));
                }
            }
        }
    }
}

// R = A X - B (fp32 storage, fp64 r^2 block partials)
template <int KL>
__global__ void __launch_bounds__(kMrThreads) mrhs_rows_kernel(MrhsArgs a) {
    using G = MrGeom<KL>;
    if (a.st->stop) return;
    __shared__ double red[kMrThreads / 32];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int slot = lane / G::GL, cl = lane % G::GL;
    const long long gw = (long long)blockIdx.x * (kMrThreads / 32) + wib;
    const long long nw = (long long)gridDim.x * (kMrThreads / 32);
    double mine = 0.0;
    for (long long i = gw; i < a.L.m; i += nw) {
        const RowRef r = row_ref(a.L, i);
        const float* vals = rec_vals<float>(r);
        const int32_t* cols = rec_cols<float>(r);
        float2 acc = make_float2(0.f, 0.f);
        for (int t0 = 0; t0 < r.len; t0 += G::S) {
            const int t = t0 + slot;
            if (t < r.len) {
                const float v = __ldg(vals + t);
                const float2 xv = __ldg(reinterpret_cast<const float2*>(a.X + (size_t)__ldg(cols + t) * KL) + cl);
                acc.x = fmaf(v, xv.x, acc.x);
                acc.y = fmaf(v, xv.y, acc.y);
            }
        }
#pragma unroll
        for (int o = G::GL; o < 32; o <<= 1) {
            acc.x += __shfl_xor_sync(FULL, acc.x, o);
            acc.y += __shfl_xor_sync(FULL, acc.y, o);
        }
        if (slot == 0) {
            const float2 bv = __ldg(reinterpret_cast<const float2*>(a.B + (size_t)i * KL) + cl);
            const float2 rv = make_float2(acc.x - bv.x, acc.y - bv.y);
            reinterpret_cast<float2*>(a.R + (size_t)i * KL)[cl] = rv;
            mine += (double)rv.x * rv.x + (double)rv.y * rv.y;
        }
    }
    mine = warp_sum(mine);
    if (lane == 0) red[wib] = mine;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < kMrThreads / 32; ++w) t += red[w];
        a.part[blockIdx.x] = t;
    }
}

// G = A^T R over the plain CSC (rows ascending), ||G||^2 and ||X - X*||^2 partials
template <int KL>
__global__ void __launch_bounds__(kMrThreads) mrhs_cols_kernel(MrhsArgs a, int nb_rows) {
    using G = MrGeom<KL>;
    if (a.st->stop) return;
    __shared__ double red_g[kMrThreads / 32], red_d[kMrThreads / 32];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int slot = lane / G::GL, cl = lane % G::GL;
    const long long gw = (long long)blockIdx.x * (kMrThreads / 32) + wib;
    const long long nw = (long long)gridDim.x * (kMrThreads / 32);
    double g2 = 0.0, d2 = 0.0;
    for (long long j = gw; j < a.L.n; j += nw) {
        const long long e0 = __ldg(a.col_ptr + j), e1 = __ldg(a.col_ptr + j + 1);
        double gx = 0.0, gy = 0.0;
        for (long long e = e0 + slot; e < e1; e += G::S) {
            const double v = (double)__ldg(a.csc_val + e);
            const float2 rv = __ldg(reinterpret_cast<const float2*>(a.R + (size_t)__ldg(a.csc_row + e) * KL) + cl);
            gx += v * rv.x;
            gy += v * rv.y;
        }
#pragma unroll
        for (int o = G::GL; o < 32; o <<= 1) {
            gx += __shfl_xor_sync(FULL, gx, o);
            gy += __shfl_xor_sync(FULL, gy, o);
        }
        if (slot == 0) {
            g2 += gx * gx + gy * gy;
            if (a.Xstar) {
                const float2 xv = __ldg(reinterpret_cast<const float2*>(a.X + (size_t)j * KL) + cl);
                const double dx = (double)xv.x - a.Xstar[(size_t)j * KL + 2 * cl];
                const double dy = (double)xv.y - a.Xstar[(size_t)j * KL + 2 * cl + 1];
                d2 += dx * dx + dy * dy;
            }
        }
    }
    g2 = warp_sum(g2);
    d2 = warp_sum(d2);
    if (lane == 0) {
        red_g[wib] = g2;
        red_d[wib] = d2;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double s0 = 0.0, s1 = 0.0;
        for (int w = 0; w < kMrThreads / 32; ++w) {
            s0 += red_g[w];
            s1 += red_d[w];
        }
        a.part[nb_rows + blockIdx.x] = s0;
        a.part[nb_rows + gridDim.x + blockIdx.x] = s1;
    }
}

// partials -> norms[0..2] = {r_sq, g_sq, d_sq} of this shard (fixed order)
__global__ void __launch_bounds__(kMrThreads) mrhs_reduce_kernel(MrhsArgs a, int nb_rows, int nb_cols) {
    if (a.st->stop) return;
    __shared__ double red[3][kMrThreads];
    double s[3] = {0.0, 0.0, 0.0};
    for (int k = threadIdx.x; k < nb_rows; k += kMrThreads) s[0] += a.part[k];
    for (int k = threadIdx.x; k < nb_cols; k += kMrThreads) {
        s[1] += a.part[nb_rows + k];
        s[2] += a.part[nb_rows + nb_cols + k];
    }
    for (int c = 0; c < 3; ++c) red[c][threadIdx.x] = s[c];
    __syncthreads();
    for (int o = kMrThreads / 2; o > 0; o >>= 1) {
        if (threadIdx.x < o)
            for (int c = 0; c < 3; ++c) red[c][threadIdx.x] += red[c][threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x == 0)
        for (int c = 0; c < 3; ++c) a.norms[c] = red[c][0];
}

// norms (possibly all-reduced over ranks) -> record + stop (one thread)
__global__ void mrhs_commit_kernel(MrhsArgs a, int advance) {
    DevState* st = a.st;
    if (st->stop) return;
    if (advance) {
        const long long sp = chunk_span(st);
        st->epoch += sp;
        st->updates += sp * a.L.m;
    }
    const double rs = a.norms[0], gs = a.norms[1], ds = a.norms[2];
    if (!isfinite(rs) || !isfinite(gs)) {
        st->status = 8;
        st->stop = 1;
    } else {
        const long long k = st->nrec;
        if (k < a.rec_cap) {
            DevRecord rc;
            rc.epoch = st->epoch;
            rc.updates = st->updates;
            rc.r_sq = rs;
            rc.grad_sq = gs;
            rc.dist_sq = a.Xstar ? ds : -1.0;
            rc.t_ns = globaltimer_ns() - st->t0_ns;
            a.rec[k] = rc;
        }
        st->nrec = k + 1;
        if (rs <= st->target || st->epoch >= st->epochs_cap) st->stop = 1;
    }
    if (st->stop && a.host_flag) {
        *reinterpret_cast<volatile int*>(a.host_flag) = 1;
        __threadfence_system();
    }
}

static int mr_sms() { return current_sm_count(); }

int mrhs_row_blocks(long long m) {
    const long long want = (m + 7) / 8;
    return (int)(want < mr_sms() * 8 ? want : mr_sms() * 8);
}
int mrhs_col_blocks(long long n) {
    const long long want = (n + 7) / 8;
    return (int)(want < mr_sms() * 8 ? want : mr_sms() * 8);
}

template <int KL>
static void mrhs_worker_launch(const MrhsArgs& a, cudaStream_t s) {
    const int blocks = (int)((a.W * 32 + 255) / 256);
    mrhs_worker_kernel<KL><<<blocks, 256, 0, s>>>(a);
}
template <int KL>
static void mrhs_monitor_launch(const MrhsArgs& a, cudaStream_t s) {
    const int nbr = mrhs_row_blocks(a.L.m), nbc = mrhs_col_blocks(a.L.n);
    mrhs_rows_kernel<KL><<<nbr, kMrThreads, 0, s>>>(a);
    mrhs_cols_kernel<KL><<<nbc, kMrThreads, 0, s>>>(a, nbr);
    mrhs_reduce_kernel<<<1, kMrThreads, 0, s>>>(a, nbr, nbc);
}

#define MR_DISPATCH(KL_, FN, ...)                 \
    switch (KL_) {                                \
        case 2: FN<2>(__VA_ARGS__); break;        \
        case 4: FN<4>(__VA_ARGS__); break;        \
        case 8: FN<8>(__VA_ARGS__); break;        \
        case 16: FN<16>(__VA_ARGS__); break;      \
        case 32: FN<32>(__VA_ARGS__); break;      \
        default: FN<64>(__VA_ARGS__); break;      \
    }

bool mrhs_supported_kl(long long kl) { return kl >= 2 && kl <= 64 && (kl & (kl - 1)) == 0; }
void launch_mrhs_worker(const MrhsArgs& a, cudaStream_t s) { MR_DISPATCH(a.KL, mrhs_worker_launch, a, s) }
void launch_mrhs_monitor(const MrhsArgs& a, cudaStream_t s) { MR_DISPATCH(a.KL, mrhs_monitor_launch, a, s) }
void launch_mrhs_commit(const MrhsArgs& a, int advance, cudaStream_t s) { mrhs_commit_kernel<<<1, 1, 0, s>>>(a, advance); }

}  // namespace ak
