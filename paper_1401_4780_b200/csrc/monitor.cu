// K3 — the residual / convergence monitor (replaces residuals,
// ref/src/csr.cpp:140-160, as called by the snapshot/record lambdas of
// ref/src/parallel.cpp:244-270 and ref/src/kaczmarz.cpp:178-199) and the
// coordinator's stop logic (parallel.cpp:388-408).
//
// Pass 1 (rows):    r_i = a_i^T x - b_i
// Pass 2 (columns): g_j = sum_i a_ij r_i, rows ascending (multiply_transpose
//                   order, csr.cpp:80-92), plus (x_j - x*_j)^2 with an x* oracle
// Finalize:         r_sq, grad_sq, dist_sq -> trace record, stop / NonFinite
//
// r_i and g_j are formed in the reference's floating-point order (serial
// storage-order sums of rounded products) and are bit-identical to
// ref residuals(). exact = 1 (deterministic path) also sums r^2, g^2 and
// (x - x*)^2 serially in index order, making every trace record
// bit-identical; exact = 0 (async path) sums them as fixed-order block
// partials: deterministic run to run, within a few ulps of the reference.
//
// One lane per row / column keeps the serial order without any shuffle
// chain; coalescing comes from the layouts: both passes read SELL-32 copies
// of A (entry t of the 32 rows / columns of a group stored contiguously,
// kernels.h CscDev), so every load of a warp is contiguous, and each lane
// keeps 8 independent gathers in flight. x and r are read through the
// read-only path: the kernels run quiesced (L1 is invalidated at every
// launch), unlike the workers.
#include "kernels.h"

namespace ak {

constexpr int kMonThreads = 256;

static int sm_count() { return current_sm_count(); }


template <class X>
__device__ __forceinline__ double ldro(const X* p) {
    return (double)__ldg(p);
}

// One SELL-32 lane: sum_t v_t * y[idx_t] in storage order from 0.0 (a serial
// row_dot, csr.cpp:65-70, or a multiply_transpose column, csr.cpp:80-92).
// Software-pipelined: the index/value loads of block t+1 are in flight while
// block t's gathers resolve, and the ragged tail is a predicated block, so a
// lane's latency chain is ceil(len/U)+1 load rounds instead of one per entry.
template <int U, class V, class Y>
__device__ __forceinline__ double sell_dot(const int32_t* __restrict__ idx, const V* __restrict__ val, long long e,
                                           int len, const Y* __restrict__ y) {
    int ci[U];
    double av[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
        const bool ok = u < len;
        ci[u] = ok ? __ldg(idx + e + 32 * u) : 0;
        av[u] = ok ? (double)__ldg(val + e + 32 * u) : 0.0;
    }
    double s = 0.0;
    for (int t = 0; t < len; t += U) {
        double yv[U];
#pragma unroll
        for (int u = 0; u < U; ++u) yv[u] = (t + u < len) ? ldro(y + ci[u]) : 0.0;
        const long long en = e + 32ll * (t + U);
        int cn[U];
        double an[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const bool ok = t + U + u < len;
            cn[u] = ok ? __ldg(idx + en + 32 * u) : 0;
            an[u] = ok ? (double)__ldg(val + en + 32 * u) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
            if (t + u < len) s = __dadd_rn(s, __dmul_rn(av[u], yv[u]));
#pragma unroll
        for (int u = 0; u < U; ++u) {
            ci[u] = cn[u];
            av[u] = an[u];
        }
    }
    return s;
}

// Pass 1 / SpMV rows over the SELL-32 row copy: lane l of group g owns row
// 32g + l and adds v_k * x[c_k] in storage order starting from 0.0 — the
// reference's serial row_dot (csr.cpp:65-70) — with every load of a warp
// contiguous (sell_dot).
// out[i] = a_i^T x (- b_i when b); part: r^2 block partials or null.
template <class V, class X>
__global__ void __launch_bounds__(kMonThreads) rows_kernel(CscDev R, long long m, const X* __restrict__ x,
                                                          const double* __restrict__ b, double* out, double* part,
                                                          const DevState* st, const X* __restrict__ x_alt = nullptr,
                                                          const int* sel = nullptr) {
    if (st && st->stop) return;
    if (sel) {  // decoupled snapshots: the slot the monitor stream claimed, or none
        const int q = *sel;
        if (q < 0) return;
        if (q == 1) x = x_alt;
    }
    __shared__ double red[kMonThreads / 32];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const long long i = (long long)blockIdx.x * kMonThreads + threadIdx.x;
    double r2 = 0.0;
    if (i < m) {
        const int len = __ldg(R.col_len + i);
        const long long base = __ldg(R.grp_off + (i >> 5)) + lane;
        double s = sell_dot<8>(R.row, static_cast<const V*>(R.val), base, len, x);
        if (b) s = __dsub_rn(s, b[i]);
        out[i] = s;
        r2 = s * s;
    }
    if (!part) return;
    r2 = warp_sum(r2);
    if (lane == 0) red[wib] = r2;
    __syncthreads();
    if (threadIdx.x == 0) {
        double tot = 0.0;
        for (int w = 0; w < kMonThreads / 32; ++w) tot += red[w];
        part[blockIdx.x] = tot;
    }
}

// Pass 2 / SpMV columns over SELL-32: lane l of group g owns position 32g + l
// (column C.col(p) of the sigma-sorted copy; results land at the column).
// out: g (or null), part: {g^2, dist^2} block partials (or null).
template <class V, class X>
__device__ __forceinline__ void cols_block(const CscDev& C, long long n, const double* __restrict__ r, double* out,
                                           double* part_g, double* part_d, const X* __restrict__ x,
                                           const double* __restrict__ x_star) {
    __shared__ double red_g[kMonThreads / 32], red_d[kMonThreads / 32];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const long long p = (long long)blockIdx.x * kMonThreads + threadIdx.x;  // position (sigma-sorted)
    double g2 = 0.0, d2 = 0.0;
    if (p < n) {
        const long long j = C.col(p);
        const int len = __ldg(C.col_len + p);
        const long long base = __ldg(C.grp_off + (p >> 5)) + lane;
        const double g = sell_dot<8>(C.row, static_cast<const V*>(C.val), base, len, r);
        if (out) out[j] = g;
        g2 = g * g;
        if (x_star) {
            const double d = ldro(x + j) - x_star[j];
            d2 = d * d;
        }
    }
    if (!part_g) return;
    g2 = warp_sum(g2);
    d2 = warp_sum(d2);
    if (lane == 0) {
        red_g[wib] = g2;
        red_d[wib] = d2;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double a = 0.0, b = 0.0;
        for (int w = 0; w < kMonThreads / 32; ++w) {
            a += red_g[w];
            b += red_d[w];
        }
        part_g[blockIdx.x] = a;
        part_d[blockIdx.x] = b;
    }
}

template <class V, class X>
__global__ void __launch_bounds__(kMonThreads) cols_kernel(CscDev C, long long n, const double* __restrict__ r,
                                                          double* out, double* part_g, double* part_d,
                                                          const X* __restrict__ x, const double* __restrict__ x_star,
                                                          const DevState* st) {
    if (st && st->stop) return;
    cols_block<V, X>(C, n, r, out, part_g, part_d, x, x_star);
}

// Record + stop decision. Three modes:
//  * in-stream (slot < 0, !force): advance the epoch by this chunk's span
//    (advance = 1) or record the initial state (advance = 0);
//  * overlapped (slot >= 0): record the epoch-boundary snapshot of that slot,
//    taken on the worker stream while the workers went on (the reference's
//    coordinator snapshot, parallel.cpp:388-408, but quiesced);
//  * final (force = 1): the exact record after the workers stopped; like the
//    reference (parallel.cpp:415-426) it replaces a snapshot record of the
//    same epoch.
__device__ void commit_record(const MonitorArgs& a, double r_sq, double g_sq, double d_sq) {
    DevState* st = a.st;
    long long epoch, updates;
    const int slot = a.slot == kDynSlot ? st->mon_slot : a.slot;
    if (a.slot == kDynSlot && slot < 0) return;  // nothing claimed: no record
    if (slot >= 0) {
        if (!st->snap_valid[slot]) return;
        epoch = st->snap_epoch[slot];
        updates = st->snap_updates[slot];
    } else {
        if (a.set_epoch >= 0) {
            st->epoch = a.set_epoch;
            st->updates = a.set_epoch * a.m_rows;
        } else if (a.advance) {
            const long long sp = chunk_span(st);
            st->epoch += sp;
            st->updates += sp * a.m_rows;
        }
        epoch = st->epoch;
        updates = st->updates;
    }
    if (!isfinite(r_sq) || !isfinite(g_sq)) {
        st->status = 8;  // ASYRK_E_NonFinite
        st->stop = 1;
    } else {
        long long k = st->nrec;
        if (a.force && k > 0 && k <= a.rec_cap && a.rec[k - 1].epoch >= epoch) --k;
        if (k < a.rec_cap) {
            DevRecord rc;
            rc.epoch = epoch;
            rc.updates = updates;
            rc.r_sq = r_sq;
            rc.grad_sq = g_sq;
            rc.dist_sq = a.x_star ? d_sq : -1.0;
            rc.t_ns = globaltimer_ns() - st->t0_ns;
            a.rec[k] = rc;
        }
        st->nrec = k + 1;
        if (!st->stop && (r_sq <= st->target || epoch >= st->epochs_cap)) {
            st->stop = 1;
            if (slot >= 0) {
                st->stop_slot = slot;
                st->stop_epoch = epoch;
                st->stop_updates = updates;
            }
        }
    }
    // a decoupled slot goes back to the snapshot kernel unless it decided the stop
    if (a.slot == kDynSlot && !(st->stop && st->stop_slot == slot)) {
        __threadfence();
        atomicExch(&st->slot_state[slot], 0);
    }
    if (a.slot < 0) st->go = (!st->stop && st->epoch < st->epochs_cap) ? 1 : 0;
    if (a.mirror) {
        volatile HostMirror* hm = a.mirror;
        hm->epoch = epoch;
        hm->nrec = st->nrec;
        hm->r_sq = r_sq;
        hm->status = st->status;
        hm->stop = st->stop;
        hm->seq = hm->seq + 1;
    }
    if (st->stop && a.host_flag) *reinterpret_cast<volatile int*>(a.host_flag) = 1;
    if (a.mirror || (st->stop && a.host_flag)) __threadfence_system();
}

// ---- finalize, exact: serial sums in the reference's order (residuals
// csr.cpp:147-158, dist oracle parallel.cpp:82-92). The three sums are
// independent chains, one warp each; lane 0 of the warp streams its series
// through a kFinStages-deep shared-memory ring filled by 1D bulk copies
// (cp.async.bulk, completion on an mbarrier), so its loop runs at the
// latency of the dependent adds instead of a memory round trip per element.
constexpr int kFinChunk = 256;  // doubles per stage (2 KB)
constexpr int kFinStages = 4;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
    uint32_t done = 0;
    while (!done)
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                     : "=r"(done)
                     : "r"(smem_u32(bar)), "r"(phase)
                     : "memory");
}

// serial sum_k (v_k - w_k)^2 (w may be null) by one thread, streamed through
// bv / bw (kFinStages x kFinChunk doubles each)
__device__ double streamed_sumsq(const double* v, const double* w, long long n, double* bv, double* bw,
                                 uint64_t* bar) {
    const long long chunks = (n + kFinChunk - 1) / kFinChunk;
    auto issue = [&](long long c) {
        const int st = (int)(c % kFinStages);
        const long long e0 = c * kFinChunk;
        const int cnt = (int)min((long long)kFinChunk, n - e0) & ~1;  // bulk copies move multiples of 16 B
        const uint32_t bytes = (uint32_t)cnt * 8u * (w ? 2u : 1u);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar + st)), "r"(bytes)
                     : "memory");
        if (cnt) {
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                    smem_u32(bv + st * kFinChunk)),
                "l"(v + e0), "r"((uint32_t)cnt * 8u), "r"(smem_u32(bar + st))
                : "memory");
            if (w)
                asm volatile(
                    "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                        smem_u32(bw + st * kFinChunk)),
                    "l"(w + e0), "r"((uint32_t)cnt * 8u), "r"(smem_u32(bar + st))
                    : "memory");
        }
    };
    for (long long c = 0; c < chunks && c < kFinStages; ++c) issue(c);
    double s = 0.0;
    for (long long c = 0; c < chunks; ++c) {
        const int st = (int)(c % kFinStages);
        mbar_wait(bar + st, (uint32_t)((c / kFinStages) & 1));
        const long long e0 = c * kFinChunk;
        const int cnt = (int)min((long long)kFinChunk, n - e0);
        const int even = cnt & ~1;
        const double* pv = bv + st * kFinChunk;
        const double* pw = bw + st * kFinChunk;
        int k = 0;
        for (; k + 8 <= even; k += 8) {
            double q[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const double d = w ? __dsub_rn(pv[k + u], pw[k + u]) : pv[k + u];
                q[u] = __dmul_rn(d, d);
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) s = __dadd_rn(s, q[u]);
        }
        for (; k < even; ++k) {
            const double d = w ? __dsub_rn(pv[k], pw[k]) : pv[k];
            s = __dadd_rn(s, __dmul_rn(d, d));
        }
        if (cnt & 1) {  // the odd last element straight from global memory
            const double d = w ? __dsub_rn(__ldcg(v + e0 + cnt - 1), __ldcg(w + e0 + cnt - 1)) : __ldcg(v + e0 + cnt - 1);
            s = __dadd_rn(s, __dmul_rn(d, d));
        }
        if (c + kFinStages < chunks) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic reads before the async refill
            issue(c + kFinStages);
        }
    }
    return s;
}

__global__ void __launch_bounds__(96) finalize_exact_kernel(MonitorArgs a) {
    if (!a.force && a.st->stop) return;
    __shared__ __align__(128) double bufv[3][kFinStages * kFinChunk];
    __shared__ __align__(128) double bufw[kFinStages * kFinChunk];
    __shared__ __align__(8) uint64_t bar[3][kFinStages];
    __shared__ double res[3];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0) {
        for (int k = 0; k < kFinStages; ++k) mbar_init(&bar[w][k]);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        double r = 0.0;
        if (w == 0)
            r = streamed_sumsq(a.r, nullptr, a.L.m, bufv[0], nullptr, bar[0]);
        else if (w == 1)
            r = streamed_sumsq(a.g, nullptr, a.L.n, bufv[1], nullptr, bar[1]);
        else if (a.x_star)  // exact mode is fp64
            r = streamed_sumsq(static_cast<const double*>(a.x), a.x_star, a.L.n, bufv[2], bufw, bar[2]);
        res[w] = r;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        if (a.col_out) {
            a.col_out[0] = res[0];
            a.col_out[1] = res[1];
            a.col_out[2] = res[2];
        } else {
            commit_record(a, res[0], res[1], res[2]);
        }
    }
}

__global__ void multi_commit_kernel(MonitorArgs a, const double* colres, int ncols) {
    if (!a.force && a.st->stop) return;
    double r = 0.0, g = 0.0, d = 0.0;
    for (int c = 0; c < ncols; ++c) {
        r = __dadd_rn(r, colres[3 * c]);
        g = __dadd_rn(g, colres[3 * c + 1]);
        d = __dadd_rn(d, colres[3 * c + 2]);
    }
    commit_record(a, r, g, d);
}
void launch_multi_commit(const MonitorArgs& a, const double* colres, int ncols, cudaStream_t s) {
    multi_commit_kernel<<<1, 1, 0, s>>>(a, colres, ncols);
}

// ---- finalize, fast: fixed-order sum of the block partials (one block)
__device__ __forceinline__ void finalize_fast_block(const MonitorArgs& a, int nb_rows, int nb_cols) {
    if (!a.force && a.st->stop) return;
    __shared__ double red[3][kMonThreads];
    double s[3] = {0.0, 0.0, 0.0};
    for (int k = threadIdx.x; k < nb_rows; k += kMonThreads) s[0] += __ldcg(a.part + k);
    for (int k = threadIdx.x; k < nb_cols; k += kMonThreads) {
        s[1] += __ldcg(a.part + nb_rows + k);
        s[2] += __ldcg(a.part + nb_rows + nb_cols + k);
    }
    for (int c = 0; c < 3; ++c) red[c][threadIdx.x] = s[c];
    __syncthreads();
    for (int o = kMonThreads / 2; o > 0; o >>= 1) {
        if (threadIdx.x < o)
            for (int c = 0; c < 3; ++c) red[c][threadIdx.x] += red[c][threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x == 0) commit_record(a, red[0][0], red[1][0], red[2][0]);
}

// columns pass + finalize_fast in the last block to finish (async path):
// blocks always take their ticket, so the counter resets even when a stop
// makes them skip the work (the finalize then skips too)
template <class V, class X>
__global__ void __launch_bounds__(kMonThreads) cols_final_kernel(MonitorArgs a, int nb_rows, int nb_cols) {
    const DevState* gate = a.force ? nullptr : a.st;
    const int q = a.slot == kDynSlot ? a.st->mon_slot : 0;
    if (!(gate && gate->stop) && q >= 0)
        cols_block<V, X>(a.csc, a.L.n, a.r, nullptr, a.part + nb_rows, a.part + nb_rows + nb_cols,
                         static_cast<const X*>(q == 1 ? a.x_alt : a.x), a.x_star);
    __shared__ bool last;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) last = atomicAdd(&a.st->mon_ticket, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!last) return;
    if (threadIdx.x == 0) a.st->mon_ticket = 0;
    finalize_fast_block(a, nb_rows, nb_cols);
}

// ---- launch geometry
int monitor_row_blocks(long long m) { return (int)((m + kMonThreads - 1) / kMonThreads); }
int monitor_col_blocks(long long n) { return (int)((n + kMonThreads - 1) / kMonThreads); }

template <class V, class X>
static void monitor_impl(const MonitorArgs& a, cudaStream_t s) {
    const int nbr = monitor_row_blocks(a.L.m);
    const int nbc = monitor_col_blocks(a.L.n);
    const X* x = static_cast<const X*>(a.x);
    const DevState* gate = a.force ? nullptr : a.st;  // the final record runs after stop
    const bool dyn = a.slot == kDynSlot;
    rows_kernel<V, X><<<nbr, kMonThreads, 0, s>>>(a.rows, a.L.m, x, a.b, a.r, a.exact ? nullptr : a.part, gate,
                                                  dyn ? static_cast<const X*>(a.x_alt) : nullptr,
                                                  dyn ? &a.st->mon_slot : nullptr);
    if (a.exact) {
        cols_kernel<V, X><<<nbc, kMonThreads, 0, s>>>(a.csc, a.L.n, a.r, a.g, nullptr, nullptr, x, a.x_star, gate);
        finalize_exact_kernel<<<1, 96, 0, s>>>(a);
    } else {
        cols_final_kernel<V, X><<<nbc, kMonThreads, 0, s>>>(a, nbr, nbc);
    }
}

void launch_monitor(const MonitorArgs& a, int precision, cudaStream_t s) {
    switch (precision) {
        case P_F32: monitor_impl<float, float>(a, s); break;
        case P_F32X64: monitor_impl<float, double>(a, s); break;
        default: monitor_impl<double, double>(a, s); break;
    }
}

// ---- power iteration pieces (ref/src/stats.cpp:15-50): y = A v and
// w = A^T y in the reference's order (CsrMatrix::multiply / multiply_transpose).
void launch_spmv_rows(const CscDev& R, int precision, long long m, const double* v, double* out, cudaStream_t s) {
    const int nb = monitor_row_blocks(m);
    if (precision == P_F64)
        rows_kernel<double, double><<<nb, kMonThreads, 0, s>>>(R, m, v, nullptr, out, nullptr, nullptr);
    else
        rows_kernel<float, double><<<nb, kMonThreads, 0, s>>>(R, m, v, nullptr, out, nullptr, nullptr);
}
void launch_spmv_cols(const CscDev& C, int precision, long long n, const double* r, double* out, cudaStream_t s) {
    const unsigned nb = (unsigned)((n + kMonThreads - 1) / kMonThreads);
    if (precision == P_F64)
        cols_kernel<double, double><<<nb, kMonThreads, 0, s>>>(C, n, r, out, nullptr, nullptr, nullptr, nullptr,
                                                               nullptr);
    else
        cols_kernel<float, double><<<nb, kMonThreads, 0, s>>>(C, n, r, out, nullptr, nullptr, nullptr, nullptr,
                                                              nullptr);
}

__global__ void __launch_bounds__(kMonThreads) dot_part_kernel(const double* a, const double* b, long long n,
                                                              double* part) {
    __shared__ double red[kMonThreads];
    double s = 0.0;
    for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (long long)gridDim.x * blockDim.x)
        s += a[k] * b[k];
    red[threadIdx.x] = s;
    __syncthreads();
    for (int o = kMonThreads / 2; o > 0; o >>= 1) {
        if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x == 0) part[blockIdx.x] = red[0];
}
__global__ void __launch_bounds__(kMonThreads) sum_part_kernel(const double* part, int np, double* out) {
    __shared__ double red[kMonThreads];
    double s = 0.0;
    for (int k = threadIdx.x; k < np; k += kMonThreads) s += part[k];
    red[threadIdx.x] = s;
    __syncthreads();
    for (int o = kMonThreads / 2; o > 0; o >>= 1) {
        if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x == 0) *out = red[0];
}
void launch_dot(const double* a, const double* b, long long n, double* scratch, double* out, cudaStream_t s) {
    long long want = (n + kMonThreads - 1) / kMonThreads;
    const int nb = (int)(want < 4 * sm_count() ? (want > 0 ? want : 1) : 4 * sm_count());
    dot_part_kernel<<<nb, kMonThreads, 0, s>>>(a, b, n, scratch);
    sum_part_kernel<<<1, kMonThreads, 0, s>>>(scratch, nb, out);
}
// v = w / sqrt(ww)  (stats.cpp:37,41)
__global__ void power_update_kernel(double* v, const double* w, const double* ww, long long n) {
    const double wn = sqrt(*ww);
    for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (long long)gridDim.x * blockDim.x)
        v[k] = w[k] / wn;
}
void launch_power_update(double* v, const double* w, const double* ww, long long n, cudaStream_t s) {
    power_update_kernel<<<4 * sm_count(), kMonThreads, 0, s>>>(v, w, ww, n);
}

}  // namespace ak
