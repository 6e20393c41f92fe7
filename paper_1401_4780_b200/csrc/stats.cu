// K5 — structural statistics of a row-normalized A on the device
// (replaces compute_stats, ref/src/stats.cpp:52-130, exact_spectral = false;
// lambda_max comes from the device power iteration, K4).
//
// Every scalar is bit-identical to the reference:
//  * column pass (lane per column over the SELL-32 column copy, rows
//    ascending = make_csc order, csr.cpp:162-185): c_t = serial sum of v^2,
//    col_norm_t = sqrt(c_t), nu = max count, l_max = max c_t, the first empty
//    column (ZeroColumn), and W_t = sum of the row lengths of column t (the
//    l_res hash capacity);
//  * frob_sq = serial sum of c_t in column order (one warp);
//  * alpha = max theta_i * |a_ik| * col_norm[c_k] (lane per row, SELL rows);
//  * l_res = max_t ||A^T (A e_t)||: one warp per column t walks the rows of
//    column t in ascending order and, for each, all entries of that row
//    (lanes = entries, distinct columns u within a row), adding av * a_iu into
//    acc[u] held in a per-warp open-addressing table. Rows are processed one
//    after another, so every acc[u] receives its additions in the reference's
//    order; new keys are appended to a first-touch list in (row, entry) order
//    (ballot prefix), and sum acc^2 runs serially over that list — the
//    reference's `touched` order. (The reference may list a column twice when
//    its accumulator returns to exactly 0.0; the second entry adds +0.0, so
//    the sums agree.)
// Maxima of non-negative doubles use atomicMax on their bit patterns.
#include <algorithm>

#include "kernels.h"

namespace ak {

constexpr int kStatThreads = 256;

__device__ __forceinline__ void max_bits(unsigned long long* dst, double v) {
    atomicMax(dst, (unsigned long long)__double_as_longlong(v));
}

// lane per column over SELL-32 columns (positions; results at the column)
__global__ void __launch_bounds__(kStatThreads) stats_cols_kernel(CscDev C, long long n, const int32_t* __restrict__ row_len,
                                                                  double* __restrict__ col_sq, double* __restrict__ col_norm,
                                                                  StatsDev* out) {
    const long long p = (long long)blockIdx.x * kStatThreads + threadIdx.x;  // position
    if (p >= n) return;
    const long long j = C.col(p);
    const int len = __ldg(C.col_len + p);
    if (len == 0) {
        atomicMin(&out->zero_col, j);
        col_sq[j] = 0.0;
        col_norm[j] = 0.0;
        return;
    }
    const long long base = __ldg(C.grp_off + (p >> 5)) + (p & 31);
    const double* cv = static_cast<const double*>(C.val);
    double c = 0.0;
    long long w = 0;
    for (int t = 0; t < len; ++t) {
        const long long e = base + 32ll * t;
        const double v = __ldg(cv + e);
        c = __dadd_rn(c, __dmul_rn(v, v));
        w += __ldg(row_len + __ldg(C.row + e));
    }
    col_sq[j] = c;
    col_norm[j] = __dsqrt_rn(c);
    atomicMax(&out->nu, (long long)len);
    atomicMax(&out->max_w, w);
    max_bits(&out->l_max_bits, c);
}

// lane per row over SELL-32 rows: alpha = max (theta_i * |v|) * col_norm[c]
__global__ void __launch_bounds__(kStatThreads) stats_alpha_kernel(CscDev R, long long m, const double* __restrict__ col_norm,
                                                                   StatsDev* out) {
    const long long i = (long long)blockIdx.x * kStatThreads + threadIdx.x;
    if (i >= m) return;
    const int len = __ldg(R.col_len + i);
    const long long base = __ldg(R.grp_off + (i >> 5)) + (i & 31);
    const double* rv = static_cast<const double*>(R.val);
    const double th = (double)len;
    double a = 0.0;
    for (int t = 0; t < len; ++t) {
        const long long e = base + 32ll * t;
        const double cand = __dmul_rn(__dmul_rn(th, fabs(__ldg(rv + e))), __ldg(col_norm + __ldg(R.row + e)));
        a = a < cand ? cand : a;
    }
    max_bits(&out->alpha_bits, a);
}

// frob_sq: serial sum of c_t in column order (one warp; lanes load 32 at a time)
__global__ void stats_frob_kernel(const double* __restrict__ col_sq, long long n, StatsDev* out) {
    const int lane = threadIdx.x & 31;
    double s = 0.0;
    for (long long c0 = 0; c0 < n; c0 += 32) {
        const long long k = c0 + lane;
        const double q = k < n ? col_sq[k] : 0.0;
        const int lim = (int)min(32ll, n - c0);
        for (int t = 0; t < lim; ++t) s = __dadd_rn(s, __shfl_sync(FULL, q, t));
    }
    if (lane == 0) out->frob_sq = s;
}

// l_res: warp per column (walked by position: a maximum, order-free), per-warp hash table {key, acc, order} of `cap` slots
// (power of two) in shared memory (tables == nullptr) or global scratch.
__global__ void __launch_bounds__(kStatThreads) stats_lres_kernel(CscDev C, CscDev R, long long n, int cap,
                                                                  unsigned char* tables, StatsDev* out) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int wpb = blockDim.x >> 5;
    const size_t tbytes = (size_t)cap * 16;
    unsigned char* base = tables ? tables + ((size_t)blockIdx.x * wpb + wib) * tbytes : smem + (size_t)wib * tbytes;
    double* acc = reinterpret_cast<double*>(base);
    int32_t* key = reinterpret_cast<int32_t*>(base + (size_t)cap * 8);
    int32_t* order = reinterpret_cast<int32_t*>(base + (size_t)cap * 12);
    for (int q = lane; q < cap; q += 32) key[q] = -1;
    __syncwarp();
    const unsigned mask_cap = (unsigned)cap - 1;
    const double* cval = static_cast<const double*>(C.val);
    const double* rval = static_cast<const double*>(R.val);
    double best = 0.0;
    const long long gw = (long long)blockIdx.x * wpb + wib, nw = (long long)gridDim.x * wpb;
    for (long long t = gw; t < n; t += nw) {
        const int len = __ldg(C.col_len + t);
        const long long cb = __ldg(C.grp_off + (t >> 5)) + (t & 31);
        int cnt = 0;
        for (int k = 0; k < len; ++k) {
            const long long ce = cb + 32ll * k;
            const int i = __ldg(C.row + ce);
            const double av = __ldg(cval + ce);
            const int rl = __ldg(R.col_len + i);
            const long long rb = __ldg(R.grp_off + (i >> 5)) + (i & 31);
            for (int k0 = 0; k0 < rl; k0 += 32) {
                const int kk = k0 + lane;
                const bool act = kk < rl;
                int slot = -1;
                bool fresh = false;
                double p = 0.0;
                if (act) {
                    const long long re = rb + 32ll * kk;
                    const int u = __ldg(R.row + re);
                    p = __dmul_rn(av, __ldg(rval + re));
                    unsigned h = ((unsigned)u * 2654435761u) & mask_cap;
                    for (;;) {
                        const int kv = key[h];
                        if (kv == u) break;
                        if (kv == -1) {
                            const int prev = atomicCAS(key + h, -1, u);
                            if (prev == -1) {
                                fresh = true;
                                break;
                            }
                            if (prev == u) break;
                        }
                        h = (h + 1) & mask_cap;
                    }
                    slot = (int)h;
                }
                const unsigned fm = __ballot_sync(FULL, fresh);
                if (fresh) order[cnt + __popc(fm & ((1u << lane) - 1u))] = slot;
                cnt += __popc(fm);
                if (act) acc[slot] = fresh ? __dadd_rn(0.0, p) : __dadd_rn(acc[slot], p);
                __syncwarp();
            }
        }
        // rs = sum over the first-touch list of acc^2, serially
        double rs = 0.0;
        for (int c0 = 0; c0 < cnt; c0 += 32) {
            const int q = c0 + lane;
            double sq = 0.0;
            if (q < cnt) {
                const double x = acc[order[q]];
                sq = __dmul_rn(x, x);
            }
            const int lim = min(32, cnt - c0);
            for (int u = 0; u < lim; ++u) rs = __dadd_rn(rs, __shfl_sync(FULL, sq, u));
        }
        const double r = __dsqrt_rn(rs);
        best = best < r ? r : best;
        for (int q = lane; q < cnt; q += 32) key[order[q]] = -1;
        __syncwarp();
    }
    if (lane == 0) max_bits(&out->l_res_bits, best);
}

void launch_stats_cols(const CscDev& C, long long n, const int32_t* row_len, double* col_sq, double* col_norm,
                       StatsDev* out, cudaStream_t s) {
    stats_cols_kernel<<<(unsigned)((n + kStatThreads - 1) / kStatThreads), kStatThreads, 0, s>>>(C, n, row_len, col_sq,
                                                                                                 col_norm, out);
}

void launch_stats_rest(const CscDev& C, const CscDev& R, long long m, long long n, const double* col_sq,
                       const double* col_norm, long long max_w, unsigned char* scratch, size_t scratch_bytes,
                       StatsDev* out, cudaStream_t s) {
    stats_alpha_kernel<<<(unsigned)((m + kStatThreads - 1) / kStatThreads), kStatThreads, 0, s>>>(R, m, col_norm, out);
    stats_frob_kernel<<<1, 32, 0, s>>>(col_sq, n, out);
    const int cap = stats_table_cap(max_w, n);
    const size_t tbytes = (size_t)cap * 16;
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    constexpr size_t kSmemBudget = 200u << 10;
    if (tbytes <= kSmemBudget) {
        const int wpb = (int)std::min<size_t>(8, kSmemBudget / tbytes);
        const size_t smem = tbytes * wpb;
        cudaFuncSetAttribute(stats_lres_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        const int per_sm = std::max(1, (int)((227u << 10) / (smem + 1024)));
        const long long blocks = std::min<long long>((n + wpb - 1) / wpb, (long long)sms * per_sm);
        stats_lres_kernel<<<(unsigned)blocks, 32 * wpb, smem, s>>>(C, R, n, cap, nullptr, out);
    } else {
        const int wpb = 8;
        const long long blocks = std::max<long long>(1, (long long)(scratch_bytes / (tbytes * wpb)));
        stats_lres_kernel<<<(unsigned)blocks, 32 * wpb, 0, s>>>(C, R, n, cap, scratch, out);
    }
}

int stats_table_cap(long long max_w, long long n) {
    const long long need = std::max<long long>(32, 2 * std::min<long long>(max_w, n));
    int cap = 32;
    while (cap < need) cap <<= 1;
    return cap;
}

}  // namespace ak
