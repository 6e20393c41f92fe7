// K2 — the asynchronous AsyRK worker (replaces the worker lambda of
// ref/src/parallel.cpp:306-373 and its do_update :309-347).
//
// One warp is one lock-free worker. Per row event it
//   1. draws the row (counter-based Philox: no shared RNG state; slice mode
//      walks a keyed Feistel permutation of the warp's slice per pass),
//   2. fetches the row record with coalesced per-lane loads (one dependent
//      L2/HBM round trip: header + values + columns are contiguous),
//   3. gathers x at the row's columns with L1-bypassing loads and reduces
//      a_i^T x with warp shuffles,
//   4. scatters -c * a_i into x with fire-and-forget red.global.add
//      (exactly-once, like the reference's CAS loop parallel.cpp:21-26).
// The next row's record is prefetched into registers while the current
// row's gather/reduce/scatter runs, and row indices are drawn 32 at a time
// (one per lane) one batch ahead, so the only serialized latency per row is
// the x gather -> reduce -> red window — which is also what bounds the
// staleness tau (PAPER §4) for a given throughput.
//
// Differences from the CPU reference, by design:
//  * no global fetch_add per row (parallel.cpp:349): each launch processes an
//    exact number of row events (span * m, split evenly over the warps), so
//    epochs are exact and the per-launch records are quiesced snapshots;
//  * no CAS retry loop: the L2 atomic unit performs the add.
#include <cstdlib>

#include "kernels.h"

namespace ak {

// 3 blocks x 8 warps per SM (<= 85 registers, no spills with two rows in
// flight per warp): 24 worker warps x 2 rows resident per SM.
#ifndef ASYRK_WORKER_MIN_BLOCKS
#define ASYRK_WORKER_MIN_BLOCKS 3
#endif
constexpr int kWorkerBlocksPerSM = ASYRK_WORKER_MIN_BLOCKS;

template <class V, int E>
struct Frag {
    V v[E];
    int c[E];
    double b, inv;
    int len;
};

template <class V, int E>
__device__ __forceinline__ void load_frag(const Layout& L, long long row, int lane, Frag<V, E>& f) {
    const RowRef r = row_ref(L, row);
    const V* vals = rec_vals<V>(r);
    const int32_t* cols = rec_cols<V>(r);
    f.len = r.len;
#pragma unroll
    for (int e = 0; e < E; ++e) {
        const int k = lane + 32 * e;
        if (k < r.len) {
            f.v[e] = __ldg(vals + k);
            f.c[e] = __ldg(cols + k);
        } else {
            f.v[e] = V(0);
            f.c[e] = -1;
        }
    }
    f.b = rec_b(r);
    f.inv = rec_inv(r);
}

// a warp's audit checksums and increment count into its own slots (warp w
// owns audit[w][0..K) and increments[w]; launches are stream-ordered, so a
// plain read-add-write is race-free and no address is contended)
__device__ __forceinline__ void audit_flush(const WorkerArgs& a, long long warp, double (&cs)[kAuditK], int lane,
                                            unsigned long long incr) {
#pragma unroll
    for (int k = 0; k < kAuditK; ++k) {
        const double v = warp_sum(cs[k]);
        if (lane == 0) a.audit[warp * kAuditK + k] += v;
    }
    if (lane == 0) a.increments[warp] += incr;
}

// Lane-parallel draw of the rows for positions [j0, j0+32) of this warp's
// launch. Also returns 32 random bits per position for single_component picks.
struct Draw {
    long long row;
    uint32_t pick;
};

__device__ __forceinline__ Draw draw_row(const WorkerArgs& a, long long warp, long long epoch, long long j,
                                         long long slice_lo, long long slice_len) {
    Draw d;
    const U4 r = philox4x32(U4{(uint32_t)j, (uint32_t)(j >> 32), (uint32_t)warp, (uint32_t)epoch}, a.key0,
                            a.key1);
    d.pick = r.z;
    const long long m = a.L.m;
    if (a.sampling == S_SLICE) {
        const long long s = j / slice_len;
        const uint32_t jj = (uint32_t)(j - s * slice_len);
        const uint32_t pass = (uint32_t)(epoch + s);
        const uint32_t k0 = a.key0 ^ (uint32_t)(warp * 0x85EBCA6Bull) ^ 0x68E31DA4u;
        const uint32_t k1 = a.key1 ^ (pass * 0xC2B2AE35u) ^ 0xB5297A4Du;
        d.row = slice_lo + permute_index(jj, (uint32_t)slice_len, feistel_half_bits((uint32_t)slice_len), k0, k1);
    } else {
        const uint64_t bits = ((uint64_t)r.x << 32) | r.y;
        long long k = (long long)bounded64(bits, (uint64_t)m);
        if (a.sampling == S_ALIAS) {
            // Walker alias lookup (ref kaczmarz.cpp:63-69 semantics, fp32 prob)
            const int2 e = __ldg(reinterpret_cast<const int2*>(a.alias) + k);  // {prob bits, alias}
            const float u = (float)(r.w >> 8) * (1.0f / 16777216.0f);
            k = (u < __int_as_float(e.x)) ? k : (long long)e.y;
        }
        d.row = k;
    }
    return d;
}

// R rows are in flight per warp: their gathers are issued back to back, then
// their reductions interleave, then their reds — R-fold memory-level
// parallelism per warp without more resident warps (R workers per warp).
template <class V, class X, int E, int R, bool FULL_ROW>
__global__ void __launch_bounds__(256, kWorkerBlocksPerSM) worker_kernel(WorkerArgs a) {
    using T = X;  // arithmetic type of the projection (x's precision)
    const DevState* st = a.st;
    if (!st->go) return;  // decided on the worker stream before this launch
    const long long epoch = a.span0 > 0 ? a.epoch0 : st->epoch;
    const long long span = a.span0 > 0 ? a.span0 : chunk_span(st);
    if (span <= 0) return;
    const long long warp = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (warp >= a.W) return;
    const int lane = threadIdx.x & 31;
    const long long m = a.L.m;

    long long count, slice_lo = 0, slice_len = 1;
    if (a.sampling == S_SLICE) {
        slice_lo = warp * m / a.W;
        slice_len = (warp + 1) * m / a.W - slice_lo;
        count = span * slice_len;
    } else {
        const long long total = span * m;
        count = total / a.W + (warp < total % a.W ? 1 : 0);
    }
    if (count <= 0) return;

    X* __restrict__ x = static_cast<X*>(a.x);
    const bool audit = a.audit != nullptr;
    double cs[kAuditK] = {};
    const T gamma = (T)a.gamma;
    unsigned long long incr = 0;

    const long long nb = (count + 31) >> 5;
    Draw B0 = draw_row(a, warp, epoch, lane, slice_lo, slice_len);
    Draw B1 = nb > 1 ? draw_row(a, warp, epoch, 32 + lane, slice_lo, slice_len) : B0;

    Frag<V, E> cur[R];
    uint32_t pick_cur[R];
    bool ok_cur[R];
    {
        const int nq0 = (int)min(32ll, count);
#pragma unroll
        for (int r = 0; r < R; ++r) {
            ok_cur[r] = r < nq0;
            const long long row = __shfl_sync(FULL, B0.row, r);
            pick_cur[r] = __shfl_sync(FULL, B0.pick, r);
            if (ok_cur[r]) load_frag<V, E>(a.L, row, lane, cur[r]);
        }
    }

    for (long long bi = 0; bi < nb; ++bi) {
        const int nq = (int)min(32ll, count - bi * 32);
        const int nq_next = bi + 1 < nb ? (int)min(32ll, count - (bi + 1) * 32) : 0;
        for (int q0 = 0; q0 < nq; q0 += R) {
            // ---- prefetch the next R rows' records (independent of x)
            Frag<V, E> nxt[R];
            uint32_t pick_nxt[R];
            bool ok_nxt[R];
            const bool in_batch = q0 + R < nq;
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const int qn = in_batch ? q0 + R + r : r;
                ok_nxt[r] = in_batch ? (q0 + R + r < nq) : (r < nq_next);
                const long long nrow = __shfl_sync(FULL, in_batch ? B0.row : B1.row, qn & 31);
                pick_nxt[r] = __shfl_sync(FULL, in_batch ? B0.pick : B1.pick, qn & 31);
                if (ok_nxt[r]) load_frag<V, E>(a.L, nrow, lane, nxt[r]);
            }

            // ---- stale residuals a_i^T x - b_i (relaxed, L1-bypassing reads)
            T acc[R];
#pragma unroll
            for (int r = 0; r < R; ++r) {
                acc[r] = T(0);
#pragma unroll
                for (int e = 0; e < E; ++e)
                    if (ok_cur[r] && cur[r].c[e] >= 0) acc[r] += (T)cur[r].v[e] * (T)ld_x(x + cur[r].c[e]);
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1)
#pragma unroll
                for (int r = 0; r < R; ++r) acc[r] += __shfl_xor_sync(FULL, acc[r], o);

#pragma unroll
            for (int r = 0; r < R; ++r) {
                if (!ok_cur[r]) continue;
                const T res = acc[r] - (T)cur[r].b;
                if (FULL_ROW) {
                    // x -= gamma * res / ||a_i||^2 * a_i   (parallel.cpp:318-331)
                    const T c = gamma * res * (T)cur[r].inv;
#pragma unroll
                    for (int e = 0; e < E; ++e) {
                        if (cur[r].c[e] >= 0) {
                            const T d = -c * (T)cur[r].v[e];
                            atomicAdd(x + cur[r].c[e], d);
                            if (audit) audit_add(cs, cur[r].c[e], (double)d);
                        }
                    }
                    incr += (unsigned long long)cur[r].len;
                } else {
                    // one component t ~ U(supp a_i): x_t += -gamma*theta*a_it*res  (parallel.cpp:332-346)
                    const int t = (int)__umulhi(pick_cur[r], (uint32_t)cur[r].len);
#pragma unroll
                    for (int e = 0; e < E; ++e) {
                        if (lane + 32 * e == t) {
                            const T d = -gamma * (T)cur[r].len * (T)cur[r].v[e] * res;
                            atomicAdd(x + cur[r].c[e], d);
                            if (audit) audit_add(cs, cur[r].c[e], (double)d);
                        }
                    }
                    incr += 1;
                }
            }
#pragma unroll
            for (int r = 0; r < R; ++r) {
                cur[r] = nxt[r];
                pick_cur[r] = pick_nxt[r];
                ok_cur[r] = ok_nxt[r];
            }
        }
        B0 = B1;
        if (bi + 2 < nb) B1 = draw_row(a, warp, epoch, (bi + 2) * 32 + lane, slice_lo, slice_len);
    }
    if (audit) audit_flush(a, warp, cs, lane, incr);
}

// Rows longer than 128 nonzeros: chunked loop, no record prefetch.
template <class V, class X, bool FULL_ROW>
__global__ void __launch_bounds__(256) worker_kernel_long(WorkerArgs a) {
    using T = X;
    const DevState* st = a.st;
    if (!st->go) return;
    const long long epoch = a.span0 > 0 ? a.epoch0 : st->epoch;
    const long long span = a.span0 > 0 ? a.span0 : chunk_span(st);
    if (span <= 0) return;
    const long long warp = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (warp >= a.W) return;
    const int lane = threadIdx.x & 31;
    const long long m = a.L.m;
    long long count, slice_lo = 0, slice_len = 1;
    if (a.sampling == S_SLICE) {
        slice_lo = warp * m / a.W;
        slice_len = (warp + 1) * m / a.W - slice_lo;
        count = span * slice_len;
    } else {
        const long long total = span * m;
        count = total / a.W + (warp < total % a.W ? 1 : 0);
    }
    X* __restrict__ x = static_cast<X*>(a.x);
    const bool audit = a.audit != nullptr;
    double cs[kAuditK] = {};
    const T gamma = (T)a.gamma;
    unsigned long long incr = 0;
    for (long long j0 = 0; j0 < count; j0 += 32) {
        const Draw D = draw_row(a, warp, epoch, j0 + lane, slice_lo, slice_len);
        const int nq = (int)min(32ll, count - j0);
        for (int q = 0; q < nq; ++q) {
            const long long row = __shfl_sync(FULL, D.row, q);
            const uint32_t pick = __shfl_sync(FULL, D.pick, q);
            const RowRef r = row_ref(a.L, row);
            const V* vals = rec_vals<V>(r);
            const int32_t* cols = rec_cols<V>(r);
            T acc = T(0);
            for (int k = lane; k < r.len; k += 32) acc += (T)__ldg(vals + k) * (T)ld_x(x + __ldg(cols + k));
            acc = warp_sum(acc);
            const T res = acc - (T)rec_b(r);
            if (FULL_ROW) {
                const T c = gamma * res * (T)rec_inv(r);
                for (int k = lane; k < r.len; k += 32) {
                    const T d = -c * (T)__ldg(vals + k);
                    const int col = __ldg(cols + k);
                    atomicAdd(x + col, d);
                    if (audit) audit_add(cs, col, (double)d);
                }
                incr += (unsigned long long)r.len;
            } else {
                const int t = (int)__umulhi(pick, (uint32_t)r.len);
                if (lane == (t & 31)) {
                    const T d = -gamma * (T)r.len * (T)__ldg(vals + t) * res;
                    const int col = __ldg(cols + t);
                    atomicAdd(x + col, d);
                    if (audit) audit_add(cs, col, (double)d);
                }
                incr += 1;
            }
        }
    }
    if (audit) audit_flush(a, warp, cs, lane, incr);
}

// The workers' own row draws, written out (tests: alias frequencies, slice
// permutations): warp w's positions [0, per_warp) of epoch `epoch`.
__global__ void sample_rows_kernel(WorkerArgs a, long long epoch, long long per_warp, int32_t* out) {
    const long long warp = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (warp >= a.W) return;
    const int lane = threadIdx.x & 31;
    const long long m = a.L.m;
    long long slice_lo = 0, slice_len = 1;
    if (a.sampling == S_SLICE) {
        slice_lo = warp * m / a.W;
        slice_len = (warp + 1) * m / a.W - slice_lo;
    }
    for (long long j = lane; j < per_warp; j += 32)
        out[warp * per_warp + j] = (int32_t)draw_row(a, warp, epoch, j, slice_lo, slice_len).row;
}

void launch_sample_rows(const WorkerArgs& a, long long epoch, long long per_warp, int32_t* out, cudaStream_t s) {
    const long long threads = a.W * 32;
    sample_rows_kernel<<<(unsigned)((threads + 255) / 256), 256, 0, s>>>(a, epoch, per_warp, out);
}

int worker_elems_per_lane(uint32_t max_len) {
    if (max_len <= 32) return 1;
    if (max_len <= 64) return 2;
    if (max_len <= 128) return 4;
    return 0;
}

template <class V, class X, bool F>
static const void* pick_kernel_r(int E, int R) {
    switch (E) {
        case 1: return R == 2 ? (const void*)worker_kernel<V, X, 1, 2, F> : (const void*)worker_kernel<V, X, 1, 1, F>;
        case 2: return R == 2 ? (const void*)worker_kernel<V, X, 2, 2, F> : (const void*)worker_kernel<V, X, 2, 1, F>;
        case 4: return (const void*)worker_kernel<V, X, 4, 1, F>;
        default: return (const void*)worker_kernel_long<V, X, F>;
    }
}
template <class V, class X>
static const void* pick_kernel(int E, int full_row, int R) {
    return full_row ? pick_kernel_r<V, X, true>(E, R) : pick_kernel_r<V, X, false>(E, R);
}

static int rows_per_warp() {
    static int r = -1;
    if (r < 0) {
        const char* e = getenv("ASYRK_ROWS_PER_WARP");
        r = (e && atoi(e) == 1) ? 1 : 2;
    }
    return r;
}

static const void* kernel_for(int precision, int E, int full_row) {
    const int R = rows_per_warp();
    switch (precision) {
        case P_F32: return pick_kernel<float, float>(E, full_row, R);
        case P_F32X64: return pick_kernel<float, double>(E, full_row, R);
        default: return pick_kernel<double, double>(E, full_row, R);
    }
}

static int num_sms() { return current_sm_count(); }

// Spread W warps over all SMs: up to 8 warps per block, as few warps per
// block as it takes to give every SM work when W is small.
static void grid_for(long long W, int& blocks, int& threads) {
    const long long sms = num_sms();
    long long wpb = (W + sms - 1) / sms;
    if (wpb < 1) wpb = 1;
    if (wpb > 8) wpb = 8;
    threads = (int)(32 * wpb);
    blocks = (int)((W + wpb - 1) / wpb);
}

void launch_worker(const WorkerArgs& a, int precision, int E, cudaStream_t s) {
    int blocks, threads;
    grid_for(a.W, blocks, threads);
    const void* k = kernel_for(precision, E, a.full_row);
    void* args[] = {const_cast<WorkerArgs*>(&a)};
    cudaLaunchKernel(k, dim3(blocks), dim3(threads), args, 0, s);
}

int worker_max_resident_warps(int precision, int E, int full_row) {
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel_for(precision, E, full_row), 256, 0);
    return per_sm * 8 * num_sms();
}

}  // namespace ak
