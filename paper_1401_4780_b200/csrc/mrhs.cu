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
#include <cstdlib>
#include "env.h"

#include "kernels.h"

namespace ak {

constexpr int kMrThreads = 256;

// Lane geometry of a KL-column row of X: VW consecutive floats per lane
// (float4 for KL >= 4, one red.global.add.v4.f32 per lane per nonzero), GL
// lanes cover one nonzero's KL columns, S nonzeros are processed side by side.
template <int KL>
struct MrGeom {
    static constexpr int VW = KL >= 4 ? 4 : 2;
    static constexpr int GL = KL / VW;
    static constexpr int S = 32 / GL;
    static_assert(KL >= 2 && KL <= 64 && (KL & (KL - 1)) == 0, "KL must be a power of two in [2, 64]");
};

template <int VW>
struct MrVec {
    float v[VW];
};

// rows of a multiple of 4 nonzeros: records read as int4 / float4 (row_gather,
// the one-row worker); ASYRK_MRHS_VEC=0 at build time keeps per-entry loads
#ifndef ASYRK_MRHS_VEC
#define ASYRK_MRHS_VEC 1
#endif
constexpr bool kVec = ASYRK_MRHS_VEC != 0;
// element k (0..3, lane-varying) of a 4-vector without a local-memory array
__device__ __forceinline__ int pick4(const int4& q, int k) { return k == 0 ? q.x : k == 1 ? q.y : k == 2 ? q.z : q.w; }
__device__ __forceinline__ float pick4(const float4& q, int k) {
    return k == 0 ? q.x : k == 1 ? q.y : k == 2 ? q.z : q.w;
}

template <int VW>
__device__ __forceinline__ MrVec<VW> ld_xv(const float* p) {  // L1-bypassing: X takes other SMs' reds
    MrVec<VW> r;
    if constexpr (VW == 4) {
        const float4 t = __ldcg(reinterpret_cast<const float4*>(p));
        r.v[0] = t.x, r.v[1] = t.y, r.v[2] = t.z, r.v[3] = t.w;
    } else {
        const float2 t = __ldcg(reinterpret_cast<const float2*>(p));
        r.v[0] = t.x, r.v[1] = t.y;
    }
    return r;
}

template <int VW>
__device__ __forceinline__ MrVec<VW> ld_bv(const float* p) {  // B is immutable
    MrVec<VW> r;
    if constexpr (VW == 4) {
        const float4 t = __ldg(reinterpret_cast<const float4*>(p));
        r.v[0] = t.x, r.v[1] = t.y, r.v[2] = t.z, r.v[3] = t.w;
    } else {
        const float2 t = __ldg(reinterpret_cast<const float2*>(p));
        r.v[0] = t.x, r.v[1] = t.y;
    }
    return r;
}

template <int VW>
__device__ __forceinline__ void red_xv(float* p, const MrVec<VW>& d) {
    if constexpr (VW == 4)
        asm volatile("red.relaxed.gpu.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(d.v[0]), "f"(d.v[1]),
                     "f"(d.v[2]), "f"(d.v[3])
                     : "memory");
    else
        asm volatile("red.relaxed.gpu.global.add.v2.f32 [%0], {%1, %2};" ::"l"(p), "f"(d.v[0]), "f"(d.v[1])
                     : "memory");
}

// Row draw of position j of this warp's launch: with-replacement Philox, or
// slice_shuffle — warp w owns rows [w m / W, (w+1) m / W) and walks a keyed
// Feistel permutation of them per pass (ref parallel.cpp:355-363).
__device__ __forceinline__ long long mr_draw(const MrhsArgs& a, long long warp, long long epoch, long long j,
                                             long long slice_lo, long long slice_len) {
    const long long m = a.L.m;
    if (a.sampling == S_SLICE) {
        const long long s = j / slice_len;
        const uint32_t jj = (uint32_t)(j - s * slice_len);
        const uint32_t pass = (uint32_t)(epoch + s);
        const uint32_t k0 = a.key0 ^ (uint32_t)(warp * 0x85EBCA6Bull) ^ 0x68E31DA4u;
        const uint32_t k1 = a.key1 ^ (pass * 0xC2B2AE35u) ^ 0xB5297A4Du;
        return slice_lo + permute_index(jj, (uint32_t)slice_len, feistel_half_bits((uint32_t)slice_len), k0, k1);
    }
    const U4 rr = philox4x32(U4{(uint32_t)j, (uint32_t)(j >> 32), (uint32_t)warp, (uint32_t)epoch}, a.key0, a.key1);
    return (long long)bounded64(((uint64_t)rr.x << 32) | rr.y, (uint64_t)m);
}

// The row data one projection needs, held across the warp: lane k < len keeps
// (value, column) of nonzero k (rows of at most 32 nonzeros), every lane the
// B row slice of its columns and 1/||a_i||^2.
template <int VW>
struct MrRow {
    float v;
    int c;
    MrVec<VW> b;
    float inv;
    int len;
};

template <int KL>
__device__ __forceinline__ void mr_load(const MrhsArgs& a, long long i, int lane, MrRow<MrGeom<KL>::VW>& r) {
    using G = MrGeom<KL>;
    const RowRef rf = row_ref(a.L, i);
    r.len = rf.len;
    r.v = lane < rf.len ? __ldg(rec_vals<float>(rf) + lane) : 0.f;
    r.c = lane < rf.len ? __ldg(rec_cols<float>(rf) + lane) : 0;
    r.b = ld_bv<G::VW>(a.B + (size_t)i * KL + G::VW * (lane % G::GL));
    r.inv = (float)rec_inv(rf);
}

// K2b, pipelined: one warp = one lock-free worker projecting R rows at a time
// for all KL columns (the next R rows' records and B slices are prefetched
// while the current ones gather / reduce / scatter; K2's structure). Pays off
// on narrow shards (KL <= 16: the multi-GPU widths), where a row's X traffic
// is small and the per-row latency chain bounds the one-row worker.
template <int KL, int R>
__global__ void __launch_bounds__(256, R >= 4 ? 2 : 3) mrhs_worker_kernel(MrhsArgs a) {
    using G = MrGeom<KL>;
    const DevState* st = a.st;
    if (!st->go) return;
    const long long epoch = a.span0 > 0 ? a.epoch0 : st->epoch;
    const long long span = a.span0 > 0 ? a.span0 : chunk_span(st);
    if (span <= 0) return;
    const long long warp = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (warp >= a.W) return;
    const int lane = threadIdx.x & 31;
    const int slot = lane / G::GL, cl = lane % G::GL;
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
    float* __restrict__ X = a.X;
    const float gamma = (float)a.gamma;

    const long long nb = (count + 31) >> 5;
    long long D0 = mr_draw(a, warp, epoch, lane, slice_lo, slice_len);
    long long D1 = nb > 1 ? mr_draw(a, warp, epoch, 32 + lane, slice_lo, slice_len) : D0;

    MrRow<G::VW> cur[R];
    bool ok_cur[R];
    {
        const int nq0 = (int)min(32ll, count);
#pragma unroll
        for (int r = 0; r < R; ++r) {
            ok_cur[r] = r < nq0;
            const long long row = __shfl_sync(FULL, D0, r);
            if (ok_cur[r]) mr_load<KL>(a, row, lane, cur[r]);
        }
    }
    for (long long bi = 0; bi < nb; ++bi) {
        const int nq = (int)min(32ll, count - bi * 32);
        const int nq_next = bi + 1 < nb ? (int)min(32ll, count - (bi + 1) * 32) : 0;
        for (int q0 = 0; q0 < nq; q0 += R) {
            // ---- prefetch the next R rows (independent of X)
            MrRow<G::VW> nxt[R];
            bool ok_nxt[R];
            const bool in_batch = q0 + R < nq;
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const int qn = in_batch ? q0 + R + r : r;
                ok_nxt[r] = in_batch ? (q0 + R + r < nq) : (r < nq_next);
                const long long nrow = __shfl_sync(FULL, in_batch ? D0 : D1, qn & 31);
                if (ok_nxt[r]) mr_load<KL>(a, nrow, lane, nxt[r]);
            }
            // ---- stale residuals: the R rows' X gathers issue back to back
            float acc[R][G::VW];
#pragma unroll
            for (int r = 0; r < R; ++r) {
#pragma unroll
                for (int u = 0; u < G::VW; ++u) acc[r][u] = 0.f;
                const int len = ok_cur[r] ? cur[r].len : 0;
                for (int t0 = 0; t0 < len; t0 += G::S) {
                    const int t = t0 + slot;
                    const float v = __shfl_sync(FULL, cur[r].v, t & 31);
                    const int c = __shfl_sync(FULL, cur[r].c, t & 31);
                    if (t < len) {
                        const MrVec<G::VW> xv = ld_xv<G::VW>(X + (size_t)c * KL + G::VW * cl);
#pragma unroll
                        for (int u = 0; u < G::VW; ++u) acc[r][u] = fmaf(v, xv.v[u], acc[r][u]);
                    }
                }
            }
#pragma unroll
            for (int o = G::GL; o < 32; o <<= 1)
#pragma unroll
                for (int r = 0; r < R; ++r)
#pragma unroll
                    for (int u = 0; u < G::VW; ++u) acc[r][u] += __shfl_xor_sync(FULL, acc[r][u], o);
            // ---- X[t, :] -= gamma (a_i^T X - B_i) / ||a_i||^2 * a_it
#pragma unroll
            for (int r = 0; r < R; ++r) {
                if (!ok_cur[r]) continue;
                float cf[G::VW];
#pragma unroll
                for (int u = 0; u < G::VW; ++u) cf[u] = -gamma * (acc[r][u] - cur[r].b.v[u]) * cur[r].inv;
                const int len = cur[r].len;
                for (int t0 = 0; t0 < len; t0 += G::S) {
                    const int t = t0 + slot;
                    const float v = __shfl_sync(FULL, cur[r].v, t & 31);
                    const int c = __shfl_sync(FULL, cur[r].c, t & 31);
                    if (t < len) {
                        MrVec<G::VW> d;
#pragma unroll
                        for (int u = 0; u < G::VW; ++u) d.v[u] = cf[u] * v;
                        red_xv<G::VW>(X + (size_t)c * KL + G::VW * cl, d);
                    }
                }
            }
#pragma unroll
            for (int r = 0; r < R; ++r) {
                cur[r] = nxt[r];
                ok_cur[r] = ok_nxt[r];
            }
        }
        D0 = D1;
        if (bi + 2 < nb) D1 = mr_draw(a, warp, epoch, (bi + 2) * 32 + lane, slice_lo, slice_len);
    }
}

// One row at a time, the record read in the loop (the default worker; any row
// length). STREAM: A's records and B's rows are read with the evict-first
// (streaming) cache policy so the X rows the projections gather and reduce
// into keep their L2 residency (X is 64 MB at config 5, A + B stream 216 MB
// per epoch through the 126 MB L2).
template <class T>
__device__ __forceinline__ T ld_a(const T* p, bool stream) {
    return stream ? __ldcs(p) : __ldg(p);
}
template <int VW>
__device__ __forceinline__ MrVec<VW> ld_b_stream(const float* p) {
    MrVec<VW> r;
    if constexpr (VW == 4) {
        const float4 t = __ldcs(reinterpret_cast<const float4*>(p));
        r.v[0] = t.x, r.v[1] = t.y, r.v[2] = t.z, r.v[3] = t.w;
    } else {
        const float2 t = __ldcs(reinterpret_cast<const float2*>(p));
        r.v[0] = t.x, r.v[1] = t.y;
    }
    return r;
}

template <int KL, bool STREAM, int MINB>
__global__ void __launch_bounds__(256, MINB) mrhs_worker_long_kernel(MrhsArgs a) {
    using G = MrGeom<KL>;
    const DevState* st = a.st;
    if (!st->go) return;
    const long long epoch = a.span0 > 0 ? a.epoch0 : st->epoch;
    const long long span = a.span0 > 0 ? a.span0 : chunk_span(st);
    if (span <= 0) return;
    const long long warp = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (warp >= a.W) return;
    const int lane = threadIdx.x & 31;
    const int slot = lane / G::GL, cl = lane % G::GL;
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
    float* __restrict__ X = a.X;
    const float gamma = (float)a.gamma;
    for (long long j0 = 0; j0 < count; j0 += 32) {
        const long long myrow = mr_draw(a, warp, epoch, j0 + lane, slice_lo, slice_len);
        const int nq = (int)min(32ll, count - j0);
        for (int q = 0; q < nq; ++q) {
            const long long i = __shfl_sync(FULL, myrow, q);
            const RowRef r = row_ref(a.L, i);
            const float* vals = rec_vals<float>(r);
            const int32_t* cols = rec_cols<float>(r);
            const int len = r.len;
            float acc[G::VW];
#pragma unroll
            for (int u = 0; u < G::VW; ++u) acc[u] = 0.f;
            // rows of a multiple of 4 nonzeros (S <= 4): the record as int4 / float4, one
            // broadcast load per 4 nonzeros (slot s takes entries s, s + S, ...) instead
            // of one per nonzero — a quarter of the record's L1TEX wavefronts
            constexpr int PER = G::S <= 4 ? 4 / G::S : 1;  // entries of a chunk per slot
            const bool vec = kVec && G::S <= 4 && (len & 3) == 0;
            if (vec) {
                for (int t0 = 0; t0 < len; t0 += 4) {
                    const int4 c4 = STREAM ? __ldcs(reinterpret_cast<const int4*>(cols + t0))
                                           : __ldg(reinterpret_cast<const int4*>(cols + t0));
                    const float4 v4 = STREAM ? __ldcs(reinterpret_cast<const float4*>(vals + t0))
                                             : __ldg(reinterpret_cast<const float4*>(vals + t0));
                    MrVec<G::VW> xv[PER];
#pragma unroll
                    for (int j = 0; j < PER; ++j) xv[j] = ld_xv<G::VW>(X + (size_t)pick4(c4, slot + G::S * j) * KL + G::VW * cl);
#pragma unroll
                    for (int j = 0; j < PER; ++j) {
                        const float v = pick4(v4, slot + G::S * j);
#pragma unroll
                        for (int u = 0; u < G::VW; ++u) acc[u] = fmaf(v, xv[j].v[u], acc[u]);
                    }
                }
            } else {
                for (int t0 = 0; t0 < len; t0 += G::S) {
                    const int t = t0 + slot;
                    if (t < len) {
                        const float v = ld_a(vals + t, STREAM);
                        const MrVec<G::VW> xv = ld_xv<G::VW>(X + (size_t)ld_a(cols + t, STREAM) * KL + G::VW * cl);
#pragma unroll
                        for (int u = 0; u < G::VW; ++u) acc[u] = fmaf(v, xv.v[u], acc[u]);
                    }
                }
            }
#pragma unroll
            for (int o = G::GL; o < 32; o <<= 1)
#pragma unroll
                for (int u = 0; u < G::VW; ++u) acc[u] += __shfl_xor_sync(FULL, acc[u], o);
            const MrVec<G::VW> bv = STREAM ? ld_b_stream<G::VW>(a.B + (size_t)i * KL + G::VW * cl)
                                           : ld_bv<G::VW>(a.B + (size_t)i * KL + G::VW * cl);
            const float inv = (float)rec_inv(r);
            float cf[G::VW];
#pragma unroll
            for (int u = 0; u < G::VW; ++u) cf[u] = -gamma * (acc[u] - bv.v[u]) * inv;
            if (vec) {
                for (int t0 = 0; t0 < len; t0 += 4) {
                    const int4 c4 = STREAM ? __ldcs(reinterpret_cast<const int4*>(cols + t0))
                                           : __ldg(reinterpret_cast<const int4*>(cols + t0));
                    const float4 v4 = STREAM ? __ldcs(reinterpret_cast<const float4*>(vals + t0))
                                             : __ldg(reinterpret_cast<const float4*>(vals + t0));
#pragma unroll
                    for (int j = 0; j < PER; ++j) {
                        const float v = pick4(v4, slot + G::S * j);
                        MrVec<G::VW> d;
#pragma unroll
                        for (int u = 0; u < G::VW; ++u) d.v[u] = cf[u] * v;
                        red_xv<G::VW>(X + (size_t)pick4(c4, slot + G::S * j) * KL + G::VW * cl, d);
                    }
                }
            } else {
                for (int t0 = 0; t0 < len; t0 += G::S) {
                    const int t = t0 + slot;
                    if (t < len) {
                        const float v = ld_a(vals + t, STREAM);
                        MrVec<G::VW> d;
#pragma unroll
                        for (int u = 0; u < G::VW; ++u) d.v[u] = cf[u] * v;
                        red_xv<G::VW>(X + (size_t)ld_a(cols + t, STREAM) * KL + G::VW * cl, d);
                    }
                }
            }
        }
    }
}

// K2b, batched (rows of at most 32 nonzeros): one row per warp at a time, its
// record (value, column per lane) loaded in one round trip and the next row's
// prefetched, then the row's X gathers issued in batches of U with no
// dependent load in between — so a row costs ~2 L2 round trips instead of one
// (column load -> X load) chain per batch of the looped worker.
template <int KL, int U>
__global__ void __launch_bounds__(256, 3) mrhs_worker_batched_kernel(MrhsArgs a) {
    using G = MrGeom<KL>;
    constexpr int T = (32 + G::S - 1) / G::S;  // slot iterations covering 32 nonzeros
    const DevState* st = a.st;
    if (!st->go) return;
    const long long epoch = a.span0 > 0 ? a.epoch0 : st->epoch;
    const long long span = a.span0 > 0 ? a.span0 : chunk_span(st);
    if (span <= 0) return;
    const long long warp = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (warp >= a.W) return;
    const int lane = threadIdx.x & 31;
    const int slot = lane / G::GL, cl = lane % G::GL;
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
    float* __restrict__ X = a.X;
    const float gamma = (float)a.gamma;
    const long long nb = (count + 31) >> 5;
    long long D0 = mr_draw(a, warp, epoch, lane, slice_lo, slice_len);
    long long D1 = nb > 1 ? mr_draw(a, warp, epoch, 32 + lane, slice_lo, slice_len) : D0;
    MrRow<G::VW> cur;
    mr_load<KL>(a, __shfl_sync(FULL, D0, 0), lane, cur);
    for (long long bi = 0; bi < nb; ++bi) {
        const int nq = (int)min(32ll, count - bi * 32);
        const int nq_next = bi + 1 < nb ? (int)min(32ll, count - (bi + 1) * 32) : 0;
        for (int q = 0; q < nq; ++q) {
            // ---- prefetch the next row (independent of X)
            MrRow<G::VW> nxt;
            const bool in_batch = q + 1 < nq;
            const bool ok_nxt = in_batch || nq_next > 0;
            if (ok_nxt) mr_load<KL>(a, __shfl_sync(FULL, in_batch ? D0 : D1, in_batch ? q + 1 : 0), lane, nxt);
            // ---- a_i^T X: batches of U independent gathers
            const int len = cur.len;
            float acc[G::VW];
#pragma unroll
            for (int u = 0; u < G::VW; ++u) acc[u] = 0.f;
#pragma unroll
            for (int jb = 0; jb < T; jb += U) {
                if (jb * G::S < len) {
                    MrVec<G::VW> xv[U];
                    float vv[U];
#pragma unroll
                    for (int j = 0; j < U; ++j) {
                        const int t = (jb + j) * G::S + slot;
                        vv[j] = __shfl_sync(FULL, cur.v, t & 31);
                        const int c = __shfl_sync(FULL, cur.c, t & 31);
                        if (t < len) {
                            xv[j] = ld_xv<G::VW>(X + (size_t)c * KL + G::VW * cl);
                        } else {
                            vv[j] = 0.f;
#pragma unroll
                            for (int u = 0; u < G::VW; ++u) xv[j].v[u] = 0.f;
                        }
                    }
#pragma unroll
                    for (int j = 0; j < U; ++j)
#pragma unroll
                        for (int u = 0; u < G::VW; ++u) acc[u] = fmaf(vv[j], xv[j].v[u], acc[u]);
                }
            }
#pragma unroll
            for (int o = G::GL; o < 32; o <<= 1)
#pragma unroll
                for (int u = 0; u < G::VW; ++u) acc[u] += __shfl_xor_sync(FULL, acc[u], o);
            // ---- X[t, :] -= gamma (a_i^T X - B_i) / ||a_i||^2 * a_it
            float cf[G::VW];
#pragma unroll
            for (int u = 0; u < G::VW; ++u) cf[u] = -gamma * (acc[u] - cur.b.v[u]) * cur.inv;
#pragma unroll
            for (int jt = 0; jt < T; ++jt) {
                const int t = jt * G::S + slot;
                if (jt * G::S < len) {
                    const float v = __shfl_sync(FULL, cur.v, t & 31);
                    const int c = __shfl_sync(FULL, cur.c, t & 31);
                    if (t < len) {
                        MrVec<G::VW> d;
#pragma unroll
                        for (int u = 0; u < G::VW; ++u) d.v[u] = cf[u] * v;
                        red_xv<G::VW>(X + (size_t)c * KL + G::VW * cl, d);
                    }
                }
            }
            if (ok_nxt) cur = nxt;
        }
        D0 = D1;
        if (bi + 2 < nb) D1 = mr_draw(a, warp, epoch, (bi + 2) * 32 + lane, slice_lo, slice_len);
    }
}

// K2b, row-parallel: a warp projects RPW = 32 / GL rows at once, each by its
// own group of GL = KL / VW lanes (float4 / float2 per lane) that walks the
// row's nonzeros serially — no cross-lane reduction, one shuffle per row (its
// index), the nonzeros' value / column loads broadcast within the group, and
// RPW rows of loads in flight per warp. On narrow shards (the multi-GPU
// widths) this cuts the instructions per row several-fold against the
// lane-per-nonzero layout, which spends most of them on the per-row reduction
// and shuffles (profiles/r02_ncu_mrhs8.txt).

// One lane group's walk over a row record (row-parallel kernels): rows of a
// multiple of 4 nonzeros (the columns then 16-byte aligned in the record) are
// read as int4 / float4 — each load instruction of the warp touches one line
// per row, so the record takes a quarter of the L1TEX wavefronts of
// per-nonzero loads (the unit these kernels saturate at 8 columns:
// profiles/r02_ncu_mrhs8.txt) — with four X accesses in flight per lane.
// acc += sum_t v_t X[c_t, lanes]   (CG: L1-bypassing X loads, the worker's)
template <int KL, bool CG>
__device__ __forceinline__ void row_gather(const float* vals, const int32_t* cols, int len, const float* X, int cl,
                                           float* acc) {
    using G = MrGeom<KL>;
    auto ld = [&](int c) {
        const float* p = X + (size_t)c * KL + G::VW * cl;
        return CG ? ld_xv<G::VW>(p) : ld_bv<G::VW>(p);
    };
    if (kVec && (len & 3) == 0) {
        for (int t = 0; t < len; t += 4) {
            const int4 c4 = __ldg(reinterpret_cast<const int4*>(cols + t));
            const float4 v4 = __ldg(reinterpret_cast<const float4*>(vals + t));
            const MrVec<G::VW> x0 = ld(c4.x), x1 = ld(c4.y), x2 = ld(c4.z), x3 = ld(c4.w);
#pragma unroll
            for (int u = 0; u < G::VW; ++u) {
                acc[u] = fmaf(v4.x, x0.v[u], acc[u]);
                acc[u] = fmaf(v4.y, x1.v[u], acc[u]);
                acc[u] = fmaf(v4.z, x2.v[u], acc[u]);
                acc[u] = fmaf(v4.w, x3.v[u], acc[u]);
            }
        }
        return;
    }
#pragma unroll 4
    for (int t = 0; t < len; ++t) {
        const float v = __ldg(vals + t);
        const MrVec<G::VW> xv = ld(__ldg(cols + t));
#pragma unroll
        for (int u = 0; u < G::VW; ++u) acc[u] = fmaf(v, xv.v[u], acc[u]);
    }
}

// Y[c_t, lanes] += v_t * f[lanes] for every nonzero t of the row (v4 / v2 reds)
template <int KL>
__device__ __forceinline__ void row_scatter(const float* vals, const int32_t* cols, int len, float* Y, int cl,
                                            const float* f) {
    using G = MrGeom<KL>;
    auto red = [&](int c, float v) {
        MrVec<G::VW> d;
#pragma unroll
        for (int u = 0; u < G::VW; ++u) d.v[u] = f[u] * v;
        red_xv<G::VW>(Y + (size_t)c * KL + G::VW * cl, d);
    };
    if (kVec && (len & 3) == 0) {
        for (int t = 0; t < len; t += 4) {
            const int4 c4 = __ldg(reinterpret_cast<const int4*>(cols + t));
            const float4 v4 = __ldg(reinterpret_cast<const float4*>(vals + t));
            red(c4.x, v4.x);
            red(c4.y, v4.y);
            red(c4.z, v4.z);
            red(c4.w, v4.w);
        }
        return;
    }
#pragma unroll 4
    for (int t = 0; t < len; ++t) red(__ldg(cols + t), __ldg(vals + t));
}

template <int KL>
__global__ void __launch_bounds__(256, 4) mrhs_worker_rows_kernel(MrhsArgs a) {
    using G = MrGeom<KL>;
    constexpr int RPW = 32 / G::GL;
    const DevState* st = a.st;
    if (!st->go) return;
    const long long epoch = a.span0 > 0 ? a.epoch0 : st->epoch;
    const long long span = a.span0 > 0 ? a.span0 : chunk_span(st);
    if (span <= 0) return;
    const long long warp = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (warp >= a.W) return;
    const int lane = threadIdx.x & 31;
    const int grp = lane / G::GL, cl = lane % G::GL;
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
    float* __restrict__ X = a.X;
    const float gamma = (float)a.gamma;
    for (long long j0 = 0; j0 < count; j0 += 32) {
        const long long D = mr_draw(a, warp, epoch, j0 + lane, slice_lo, slice_len);
        const int nq = (int)min(32ll, count - j0);
        for (int q0 = 0; q0 < nq; q0 += RPW) {
            const long long i = __shfl_sync(FULL, D, q0 + grp);
            if (q0 + grp >= nq) continue;
            const RowRef r = row_ref(a.L, i);
            const float* vals = rec_vals<float>(r);
            const int32_t* cols = rec_cols<float>(r);
            const int len = r.len;
            float acc[G::VW];
#pragma unroll
            for (int u = 0; u < G::VW; ++u) acc[u] = 0.f;
            row_gather<KL, true>(vals, cols, len, X, cl, acc);
            const MrVec<G::VW> bv = ld_bv<G::VW>(a.B + (size_t)i * KL + G::VW * cl);
            const float inv = (float)rec_inv(r);
            float cf[G::VW];
#pragma unroll
            for (int u = 0; u < G::VW; ++u) cf[u] = -gamma * (acc[u] - bv.v[u]) * inv;
            row_scatter<KL>(vals, cols, len, X, cl, cf);
        }
    }
}

// R = A X - B (fp32 storage, fp64 r^2 block partials): warp per row, lanes
// over the row's KL columns (VW floats each), S nonzeros side by side
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
        float acc[G::VW];
#pragma unroll
        for (int u = 0; u < G::VW; ++u) acc[u] = 0.f;
        for (int t0 = 0; t0 < r.len; t0 += G::S) {
            const int t = t0 + slot;
            if (t < r.len) {
                const float v = __ldg(vals + t);
                const MrVec<G::VW> xv = ld_bv<G::VW>(a.X + (size_t)__ldg(cols + t) * KL + G::VW * cl);
#pragma unroll
                for (int u = 0; u < G::VW; ++u) acc[u] = fmaf(v, xv.v[u], acc[u]);
            }
        }
#pragma unroll
        for (int o = G::GL; o < 32; o <<= 1)
#pragma unroll
            for (int u = 0; u < G::VW; ++u) acc[u] += __shfl_xor_sync(FULL, acc[u], o);
        const MrVec<G::VW> bv = ld_bv<G::VW>(a.B + (size_t)i * KL + G::VW * cl);
        float rv[G::VW];
#pragma unroll
        for (int u = 0; u < G::VW; ++u) rv[u] = acc[u] - bv.v[u];
        if (slot == 0) {
#pragma unroll
            for (int u = 0; u < G::VW; ++u) mine += (double)rv[u] * rv[u];
            if (!a.G) {
                float* rp = a.R + (size_t)i * KL + G::VW * cl;
#pragma unroll
                for (int u = 0; u < G::VW; ++u) rp[u] = rv[u];
            }
        }
        if (a.G) {  // G += a_i r_i^T (every slot lane holds r_i's columns after the butterfly)
            for (int t0 = 0; t0 < r.len; t0 += G::S) {
                const int t = t0 + slot;
                if (t < r.len) {
                    const float v = __ldg(vals + t);
                    MrVec<G::VW> d;
#pragma unroll
                    for (int u = 0; u < G::VW; ++u) d.v[u] = v * rv[u];
                    red_xv<G::VW>(a.G + (size_t)__ldg(cols + t) * KL + G::VW * cl, d);
                }
            }
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
        double g[G::VW];
#pragma unroll
        for (int u = 0; u < G::VW; ++u) g[u] = 0.0;
        for (long long e = e0 + slot; e < e1; e += G::S) {
            const double v = (double)__ldg(a.csc_val + e);
            const MrVec<G::VW> rv = ld_bv<G::VW>(a.R + (size_t)__ldg(a.csc_row + e) * KL + G::VW * cl);
#pragma unroll
            for (int u = 0; u < G::VW; ++u) g[u] += v * rv.v[u];
        }
#pragma unroll
        for (int o = G::GL; o < 32; o <<= 1)
#pragma unroll
            for (int u = 0; u < G::VW; ++u) g[u] += __shfl_xor_sync(FULL, g[u], o);
        if (slot == 0) {
#pragma unroll
            for (int u = 0; u < G::VW; ++u) g2 += g[u] * g[u];
            if (a.Xstar) {
                const MrVec<G::VW> xv = ld_bv<G::VW>(a.X + (size_t)j * KL + G::VW * cl);
#pragma unroll
                for (int u = 0; u < G::VW; ++u) {
                    const double d = (double)xv.v[u] - a.Xstar[(size_t)j * KL + G::VW * cl + u];
                    d2 += d * d;
                }
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

// Row-parallel monitor passes for narrow shards (KL <= 16): a group of GL
// lanes owns a row (pass 1) or a column (pass 2) and walks its entries
// serially, as the row-parallel worker does; no cross-lane reduction per row.
template <int KL>
__global__ void __launch_bounds__(kMrThreads) mrhs_rows_par_kernel(MrhsArgs a) {
    using G = MrGeom<KL>;
    constexpr int RPW = 32 / G::GL;
    if (a.st->stop) return;
    __shared__ double red[kMrThreads / 32];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int grp = lane / G::GL, cl = lane % G::GL;
    const long long gw = (long long)blockIdx.x * (kMrThreads / 32) + wib;
    const long long nw = (long long)gridDim.x * (kMrThreads / 32);
    double mine = 0.0;
    for (long long i = gw * RPW + grp; i < a.L.m; i += nw * RPW) {
        const RowRef r = row_ref(a.L, i);
        const float* vals = rec_vals<float>(r);
        const int32_t* cols = rec_cols<float>(r);
        float acc[G::VW];
#pragma unroll
        for (int u = 0; u < G::VW; ++u) acc[u] = 0.f;
        row_gather<KL, false>(vals, cols, r.len, a.X, cl, acc);
        const MrVec<G::VW> bv = ld_bv<G::VW>(a.B + (size_t)i * KL + G::VW * cl);
        float rv[G::VW];
#pragma unroll
        for (int u = 0; u < G::VW; ++u) {
            rv[u] = acc[u] - bv.v[u];
            mine += (double)rv[u] * rv[u];
        }
        if (a.G) {  // G += a_i r_i^T
            row_scatter<KL>(vals, cols, r.len, a.G, cl, rv);
        } else {
            float* rp = a.R + (size_t)i * KL + G::VW * cl;
#pragma unroll
            for (int u = 0; u < G::VW; ++u) rp[u] = rv[u];
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

template <int KL>
__global__ void __launch_bounds__(kMrThreads) mrhs_cols_par_kernel(MrhsArgs a, int nb_rows) {
    using G = MrGeom<KL>;
    constexpr int RPW = 32 / G::GL;
    if (a.st->stop) return;
    __shared__ double red_g[kMrThreads / 32], red_d[kMrThreads / 32];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int grp = lane / G::GL, cl = lane % G::GL;
    const long long gw = (long long)blockIdx.x * (kMrThreads / 32) + wib;
    const long long nw = (long long)gridDim.x * (kMrThreads / 32);
    double g2 = 0.0, d2 = 0.0;
    for (long long j = gw * RPW + grp; j < a.L.n; j += nw * RPW) {
        const long long e0 = __ldg(a.col_ptr + j), e1 = __ldg(a.col_ptr + j + 1);
        double g[G::VW];
#pragma unroll
        for (int u = 0; u < G::VW; ++u) g[u] = 0.0;
#pragma unroll 4
        for (long long e = e0; e < e1; ++e) {
            const double v = (double)__ldg(a.csc_val + e);
            const MrVec<G::VW> rv = ld_bv<G::VW>(a.R + (size_t)__ldg(a.csc_row + e) * KL + G::VW * cl);
#pragma unroll
            for (int u = 0; u < G::VW; ++u) g[u] += v * rv.v[u];
        }
#pragma unroll
        for (int u = 0; u < G::VW; ++u) g2 += g[u] * g[u];
        if (a.Xstar) {
            const MrVec<G::VW> xv = ld_bv<G::VW>(a.X + (size_t)j * KL + G::VW * cl);
#pragma unroll
            for (int u = 0; u < G::VW; ++u) {
                const double d = (double)xv.v[u] - a.Xstar[(size_t)j * KL + G::VW * cl + u];
                d2 += d * d;
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

// Scatter monitor, pass 2: ||G||_F^2 of the G the rows pass accumulated
// (G = A^T R by fp32 red.add, no CSC gather of R) and ||X - X*||_F^2, fp64
// block partials in the columns slots of part
__global__ void __launch_bounds__(kMrThreads) mrhs_gnorm_kernel(MrhsArgs a, int nb_rows) {
    if (a.st->stop) return;
    __shared__ double red_g[kMrThreads / 32], red_d[kMrThreads / 32];
    const long long total = a.L.n * (long long)a.KL;
    double g2 = 0.0, d2 = 0.0;
    for (long long e = (long long)blockIdx.x * kMrThreads + threadIdx.x; e < total;
         e += (long long)gridDim.x * kMrThreads) {
        const double g = (double)__ldcg(a.G + e);
        g2 += g * g;
        if (a.Xstar) {
            const double d = (double)__ldcg(a.X + e) - a.Xstar[e];
            d2 += d * d;
        }
    }
    g2 = warp_sum(g2);
    d2 = warp_sum(d2);
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
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

// norms (possibly all-reduced over ranks) -> record + stop (one thread), at
// boundary set_epoch (epochs are exact per launch: updates = epoch * m); the
// decision inputs also go to the host mirror for the host-driven schedule
__global__ void mrhs_commit_kernel(MrhsArgs a, long long set_epoch) {
    DevState* st = a.st;
    if (st->stop) return;
    if (set_epoch >= 0) {
        st->epoch = set_epoch;
        st->updates = set_epoch * a.L.m;
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
    st->go = st->stop ? 0 : 1;
    if (a.mirror) {
        volatile HostMirror* hm = a.mirror;
        hm->epoch = st->epoch;
        hm->nrec = st->nrec;
        hm->r_sq = rs;
        hm->status = st->status;
        hm->stop = st->stop;
        hm->seq = hm->seq + 1;
    }
    if (st->stop && a.host_flag) *reinterpret_cast<volatile int*>(a.host_flag) = 1;
    __threadfence_system();
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

// rows in flight per warp of the lane-per-nonzero workers (A/B; the defaults
// below are the measured best: the one-row worker at 32 and 64 columns, the
// row-parallel one at 16 and fewer, profiles/r02_cfg5_probe.txt)
static int mrhs_default_rows(int kl) { return kl >= 32 ? 1 : 2; }

// The worker kernel for a shard width: rows in flight per warp from
// ASYRK_MRHS_ROWS (1, 2 or 4) or the default above; rows of more than 32
// nonzeros always take the one-row worker. ASYRK_MRHS_NOSTREAM=1: plain
// read-only loads for A / B; ASYRK_MRHS_MINB=5: the one-row worker at 5 blocks
// (40 warps) per SM instead of 4 (A/B runs).
// The row-parallel worker (a lane group per row, RPW rows per warp) on 8-, 16-
// and 32-column shards (at 32: 0.300 vs 0.316 ms per epoch, its monitor 0.31 vs
// 0.38 ms; at 64 the one-row worker stays ahead, 0.57 vs 0.60 — A/B in
// scripts/probe_cfg5.py); ASYRK_MRHS_ROWPAR=1 / =0 forces it on / off (any width),
// ASYRK_MRHS_ROWS / ASYRK_MRHS_BATCH select the lane-per-nonzero variants.
template <int KL>
static bool mrhs_use_rowpar() {
    static const int rowpar = getenv("ASYRK_MRHS_ROWPAR") ? atoi(getenv("ASYRK_MRHS_ROWPAR")) : -1;
    static const bool other = getenv("ASYRK_MRHS_ROWS") || getenv("ASYRK_MRHS_BATCH");
    return rowpar == 1 || (rowpar < 0 && !other && (KL == 8 || KL == 16 || KL == 32));
}

bool mrhs_rowpar(int kl) {
    switch (kl) {
        case 8: return mrhs_use_rowpar<8>();
        case 16: return mrhs_use_rowpar<16>();
        case 32: return mrhs_use_rowpar<32>();
        default: return false;
    }
}

template <int KL>
static const void* mrhs_worker_fn(uint32_t max_len) {
    static const int rows_env = getenv("ASYRK_MRHS_ROWS") ? atoi(getenv("ASYRK_MRHS_ROWS")) : 0;
    static const bool nostream = env_flag("ASYRK_MRHS_NOSTREAM");
    static const int minb = getenv("ASYRK_MRHS_MINB") ? atoi(getenv("ASYRK_MRHS_MINB")) : 4;
    const int rows = rows_env > 0 ? rows_env : mrhs_default_rows(KL);
    static const int batched = getenv("ASYRK_MRHS_BATCH") ? atoi(getenv("ASYRK_MRHS_BATCH")) : 0;
    constexpr int T = (32 + MrGeom<KL>::S - 1) / MrGeom<KL>::S;
    if (mrhs_use_rowpar<KL>()) return (const void*)mrhs_worker_rows_kernel<KL>;
    if (max_len <= 32 && batched > 0)
        return batched >= 8 ? (const void*)mrhs_worker_batched_kernel<KL, (T < 8 ? T : 8)>
                            : (const void*)mrhs_worker_batched_kernel<KL, (T < 4 ? T : 4)>;
    if (max_len <= 32 && rows == 2) return (const void*)mrhs_worker_kernel<KL, 2>;
    if (max_len <= 32 && rows >= 4) return (const void*)mrhs_worker_kernel<KL, 4>;
    if (minb >= 5)
        return nostream ? (const void*)mrhs_worker_long_kernel<KL, false, 5>
                        : (const void*)mrhs_worker_long_kernel<KL, true, 5>;
    return nostream ? (const void*)mrhs_worker_long_kernel<KL, false, 4>
                    : (const void*)mrhs_worker_long_kernel<KL, true, 4>;
}

// a.W = concurrent workers (rows in flight), the reference's `threads`: one
// per warp for the lane-per-nonzero workers, one per lane group (RPW per
// warp) for the row-parallel worker, which then launches W / RPW warps
template <int KL>
static void mrhs_worker_launch(const MrhsArgs& a0, cudaStream_t s) {
    MrhsArgs a = a0;
    if (mrhs_use_rowpar<KL>()) a.W = (a.W + (32 / MrGeom<KL>::GL) - 1) / (32 / MrGeom<KL>::GL);
    const int blocks = (int)((a.W * 32 + 255) / 256);
    void* args[] = {&a};
    cudaLaunchKernel(mrhs_worker_fn<KL>(a.max_len), dim3(blocks), dim3(256), args, 0, s);
}
template <int KL>
static void mrhs_monitor_launch(const MrhsArgs& a, cudaStream_t s) {
    const int nbr = mrhs_row_blocks(a.L.m), nbc = mrhs_col_blocks(a.L.n);
    // narrow shards: the row-parallel passes (ASYRK_MRHS_ROWPAR=0 keeps the lane-per-entry ones)
    if (a.G) cudaMemsetAsync(a.G, 0, (size_t)a.L.n * KL * sizeof(float), s);
    if (mrhs_use_rowpar<KL>())
        mrhs_rows_par_kernel<KL><<<nbr, kMrThreads, 0, s>>>(a);
    else
        mrhs_rows_kernel<KL><<<nbr, kMrThreads, 0, s>>>(a);
    if (a.G)
        mrhs_gnorm_kernel<<<nbc, kMrThreads, 0, s>>>(a, nbr);
    else if (mrhs_use_rowpar<KL>())
        mrhs_cols_par_kernel<KL><<<nbc, kMrThreads, 0, s>>>(a, nbr);
    else
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

template <int KL>
static void mrhs_occupancy(int& per_sm, uint32_t max_len) {
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, mrhs_worker_fn<KL>(max_len), 256, 0);
    if (mrhs_use_rowpar<KL>()) per_sm *= 32 / MrGeom<KL>::GL;  // workers, not warps
}
int mrhs_max_resident_warps(int kl, uint32_t max_len) {
    int per_sm = 0;
    MR_DISPATCH(kl, mrhs_occupancy, per_sm, max_len)
    return per_sm * 8 * mr_sms();
}
void launch_mrhs_worker(const MrhsArgs& a, cudaStream_t s) { MR_DISPATCH(a.KL, mrhs_worker_launch, a, s) }
void launch_mrhs_monitor(const MrhsArgs& a, cudaStream_t s) { MR_DISPATCH(a.KL, mrhs_monitor_launch, a, s) }
void launch_mrhs_commit(const MrhsArgs& a, long long set_epoch, cudaStream_t s) {
    mrhs_commit_kernel<<<1, 1, 0, s>>>(a, set_epoch);
}

}  // namespace ak
