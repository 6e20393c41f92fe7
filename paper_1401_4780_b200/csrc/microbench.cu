// x-side roofline microbenchmark (SURVEY.md §8d "R_x"): the x traffic of one
// projection with no A stream — theta (<= 128) random L2-resident gathers of x, a warp
// reduction, then theta random red.global.add — at a given warp count and x
// footprint. Modes: 0 gather -> reduce -> red (the worker's dependent chain),
// 1 gathers only, 2 reds only; mode + 16 keeps 2 rows in flight per warp. Indices come from a counter hash, so no memory
// other than x is touched. Used by bench.py to state the L2/atomic-bound
// roofline beside the HBM one.
#include "../../include/asyrk_cuda.h"
#include "capi_common.h"
#include "kernels.h"

namespace ak {

__device__ __forceinline__ uint32_t hash32(uint32_t a) {
    a ^= a >> 16;
    a *= 0x7feb352du;
    a ^= a >> 15;
    a *= 0x846ca68bu;
    a ^= a >> 16;
    return a;
}

// R rows in flight per warp, like the worker (K2 keeps 2): the R rows'
// gathers issue back to back, their reductions interleave, then their reds.
template <class X, int R>
__global__ void __launch_bounds__(256) xside_kernel(X* x, uint32_t n, int theta, long long per_warp, int mode,
                                                    unsigned long long* sink) {
    const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    X acc_all = X(0);
    for (long long q0 = 0; q0 < per_warp; q0 += R) {
        // theta <= 128: lane l owns entries l, l + 32, l + 64, l + 96 (the worker's E slots)
        uint32_t col[R][4];
        bool on[4];
        X s[R];
#pragma unroll
        for (int r = 0; r < R; ++r) {
            s[r] = X(0);
            const uint32_t q = (uint32_t)(q0 + r);
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int k = lane + 32 * e;
                on[e] = k < theta;
                const uint32_t h = hash32(warp * 0x9E3779B9u + q * 0x85EBCA6Bu + (uint32_t)k * 0xC2B2AE35u);
                col[r][e] = (uint32_t)(((uint64_t)h * n) >> 32);
                if (mode != 2 && on[e]) s[r] += __ldcg(x + col[r][e]);
            }
        }
        if (mode == 0) {
#pragma unroll
            for (int o = 16; o > 0; o >>= 1)
#pragma unroll
                for (int r = 0; r < R; ++r) s[r] += __shfl_xor_sync(FULL, s[r], o);
#pragma unroll
            for (int r = 0; r < R; ++r)
#pragma unroll
                for (int e = 0; e < 4; ++e)
                    if (on[e]) atomicAdd(x + col[r][e], X(1e-30) * s[r]);
        } else if (mode == 2) {
#pragma unroll
            for (int r = 0; r < R; ++r)
#pragma unroll
                for (int e = 0; e < 4; ++e)
                    if (on[e]) atomicAdd(x + col[r][e], X(1e-30));
        } else {
#pragma unroll
            for (int r = 0; r < R; ++r) acc_all += s[r];
        }
    }
    if (mode == 1 && acc_all == X(12345.678)) atomicAdd(sink, 1ull);  // keep the gathers alive
}

// Multi-RHS x side (config 5): per "projection" theta (<= 32) random rows of
// X (KL fp32 columns each) gathered as float4 / float2 lanes, the per-column
// warp reduction, then theta red.global.add.v4.f32 / .v2 back into the same
// rows — the K2b worker's X traffic with no A / B stream. Row indices come
// from one multiply-high of a per-lane LCG per element and stay in registers
// between the gather and the reduce phases.
template <int KL>
__global__ void __launch_bounds__(256) xside_mrhs_kernel(float* X, uint32_t n, int theta, long long per_warp) {
    constexpr int VW = KL >= 4 ? 4 : 2, GL = KL / VW, S = 32 / GL, T = (32 + S - 1) / S;
    const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31, slot = lane / GL, cl = lane % GL;
    uint32_t rng = hash32(warp * 0x9E3779B9u + (uint32_t)slot * 0x85EBCA6Bu) | 1u;
    for (long long q = 0; q < per_warp; ++q) {
        uint32_t row[T];
        float acc[VW];
#pragma unroll
        for (int u = 0; u < VW; ++u) acc[u] = 0.f;
#pragma unroll
        for (int j = 0; j < T; ++j) {
            rng = rng * 1664525u + 1013904223u;
            row[j] = __umulhi(rng, n);
            const int t = j * S + slot;
            if (t < theta) {
                const float* p = X + (size_t)row[j] * KL + VW * cl;
                if constexpr (VW == 4) {
                    const float4 v = __ldcg(reinterpret_cast<const float4*>(p));
                    acc[0] += v.x, acc[1] += v.y, acc[2] += v.z, acc[3] += v.w;
                } else {
                    const float2 v = __ldcg(reinterpret_cast<const float2*>(p));
                    acc[0] += v.x, acc[1] += v.y;
                }
            }
        }
#pragma unroll
        for (int o = GL; o < 32; o <<= 1)
#pragma unroll
            for (int u = 0; u < VW; ++u) acc[u] += __shfl_xor_sync(FULL, acc[u], o);
#pragma unroll
        for (int j = 0; j < T; ++j) {
            const int t = j * S + slot;
            if (t < theta) {
                float* p = X + (size_t)row[j] * KL + VW * cl;
                if constexpr (VW == 4)
                    asm volatile("red.relaxed.gpu.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p),
                                 "f"(1e-30f * acc[0]), "f"(1e-30f * acc[1]), "f"(1e-30f * acc[2]), "f"(1e-30f * acc[3])
                                 : "memory");
                else
                    asm volatile("red.relaxed.gpu.global.add.v2.f32 [%0], {%1, %2};" ::"l"(p), "f"(1e-30f * acc[0]),
                                 "f"(1e-30f * acc[1])
                                 : "memory");
            }
        }
    }
}

// the row-parallel worker's pattern (mrhs.cu mrhs_worker_rows_kernel): a group
// of GL lanes owns a row and walks its theta X rows serially, four gathers in
// flight, then theta v4 reds — no cross-lane reduction
template <int KL>
__global__ void __launch_bounds__(256) xside_mrhs_rows_kernel(float* X, uint32_t n, int theta, long long per_row) {
    constexpr int VW = 4, GL = KL / VW;
    const uint32_t gid = (blockIdx.x * blockDim.x + threadIdx.x) / GL;
    const int cl = threadIdx.x % GL;
    uint32_t rng = hash32(gid * 0x9E3779B9u) | 1u;
    for (long long q = 0; q < per_row; ++q) {
        const uint32_t r0 = rng;
        float acc[VW] = {0.f, 0.f, 0.f, 0.f};
        for (int t = 0; t < theta; t += 4) {
            uint32_t c[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                rng = rng * 1664525u + 1013904223u;
                c[j] = __umulhi(rng, n);
            }
            float4 v[4];
#pragma unroll
            for (int j = 0; j < 4; ++j)
                v[j] = t + j < theta ? __ldcg(reinterpret_cast<const float4*>(X + (size_t)c[j] * KL + VW * cl))
                                     : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
            for (int j = 0; j < 4; ++j) acc[0] += v[j].x, acc[1] += v[j].y, acc[2] += v[j].z, acc[3] += v[j].w;
        }
        rng = r0;  // the same theta rows again for the reds
        for (int t = 0; t < theta; ++t) {
            rng = rng * 1664525u + 1013904223u;
            float* p = X + (size_t)__umulhi(rng, n) * KL + VW * cl;
            asm volatile("red.relaxed.gpu.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(1e-30f * acc[0]),
                         "f"(1e-30f * acc[1]), "f"(1e-30f * acc[2]), "f"(1e-30f * acc[3])
                         : "memory");
        }
    }
}

template <class X>
static void xside_launch(int rows, int blocks, int threads, void* x, int64_t n, int theta, int64_t per_warp, int mode,
                         unsigned long long* sink, cudaStream_t s) {
    if (rows == 2)
        xside_kernel<X, 2><<<blocks, threads, 0, s>>>((X*)x, (uint32_t)n, theta, per_warp, mode, sink);
    else
        xside_kernel<X, 1><<<blocks, threads, 0, s>>>((X*)x, (uint32_t)n, theta, per_warp, mode, sink);
}

}  // namespace ak

namespace ak {

// time one launch (after a warm-up launch) of the x-side kernel on buffer x
static asyrk_status xside_time(void* x, int64_t n, int32_t theta, int32_t precision, int32_t warps, int64_t& per_warp,
                               int32_t mode, cudaStream_t stream, float& ms, int& blocks) {
    // mode + 16: the same traffic with 2 rows in flight per warp (the worker's shape)
    const int rows = mode >= 16 ? 2 : 1;
    mode &= 15;
    if (rows == 2) per_warp += per_warp & 1;
    unsigned long long* sink = nullptr;
    if (cudaMalloc(&sink, 8) != cudaSuccess) return ASYRK_E_TooLarge;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int threads = 256;
    blocks = (warps * 32 + threads - 1) / threads;
    ms = 0.f;
    for (int rep = 0; rep < 2; ++rep) {  // first launch warms up
        cudaEventRecord(e0, stream);
        if (precision == P_F32)
            xside_launch<float>(rows, blocks, threads, x, n, theta, per_warp, mode, sink, stream);
        else
            xside_launch<double>(rows, blocks, threads, x, n, theta, per_warp, mode, sink, stream);
        cudaEventRecord(e1, stream);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
    }
    const cudaError_t err = cudaGetLastError();
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(sink);
    return err == cudaSuccess ? ASYRK_OK : ASYRK_E_ThreadSpawnFailure;
}

}  // namespace ak

extern "C" asyrk_status asyrk_microbench_xside(int64_t n, int32_t theta, int32_t precision, int32_t warps,
                                               int64_t proj_per_warp, int32_t mode, double* proj_per_s,
                                               double* kernel_ms) {
    using namespace ak;
    if (n < 1 || theta < 1 || theta > 128 || warps < 1 || proj_per_warp < 1)
        return fail(ASYRK_E_InvalidArgument, "microbench_xside: need n >= 1, 1 <= theta <= 128, warps >= 1");
    // x on a 2 MB page boundary, like the solver's (system.cu dalloc_page_aligned)
    void* base = nullptr;
    const size_t xb = (size_t)n * (precision == P_F32 ? 4 : 8);
    const size_t page = 2u << 20;
    if (cudaMalloc(&base, xb + page) != cudaSuccess) return ASYRK_E_TooLarge;
    void* x = reinterpret_cast<void*>((reinterpret_cast<uintptr_t>(base) + page - 1) & ~(uintptr_t)(page - 1));
    cudaMemset(x, 0, xb);
    float ms = 0.f;
    int blocks = 0;
    const asyrk_status st = xside_time(x, n, theta, precision, warps, proj_per_warp, mode, nullptr, ms, blocks);
    cudaFree(base);
    if (st) return st;
    *proj_per_s = (double)blocks * 256 / 32 * (double)proj_per_warp / (ms * 1e-3);
    if (kernel_ms) *kernel_ms = ms;
    return ASYRK_OK;
}

// The same measurement on a resident system's own x buffer (its address,
// alignment and footprint; the row length of its records as theta) on its
// stream. Leaves x perturbed by ~1e-30 increments: every solve re-initialises x.
asyrk_status xside_on_buffer(void* x, int64_t n, int32_t theta, int32_t precision, int32_t warps, int64_t per_warp,
                             int32_t mode, void* stream, double* proj_per_s, double* kernel_ms) {
    using namespace ak;
    if (theta < 1 || theta > 128 || warps < 1 || per_warp < 1)
        return fail(ASYRK_E_InvalidArgument, "microbench_xside: need rows of 1..128 nonzeros, warps >= 1");
    float ms = 0.f;
    int blocks = 0;
    const asyrk_status st =
        xside_time(x, n, theta, precision, warps, per_warp, mode, static_cast<cudaStream_t>(stream), ms, blocks);
    if (st) return st;
    *proj_per_s = (double)blocks * 256 / 32 * (double)per_warp / (ms * 1e-3);
    if (kernel_ms) *kernel_ms = ms;
    return ASYRK_OK;
}

// R_x of the multi-RHS pattern (config 5): X n x kl fp32 on a 2 MB boundary
namespace ak {
// the multi-RHS x-side kernel timed on an n x kl X buffer (its contents are
// perturbed by reds of ~1e-30 x values)
int32_t xside_mrhs_on_buffer(float* X, int64_t n, int32_t theta, int32_t kl, int32_t warps, int64_t proj_per_warp,
                                  cudaStream_t stream, double* proj_per_s, double* kernel_ms) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int blocks = (warps * 32 + 255) / 256;
    float ms = 0.f;
    const bool rows = mrhs_rowpar((int)kl);  // the worker's own shape at this width
    for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(e0, stream);
        if (rows && kl == 8)
            xside_mrhs_rows_kernel<8><<<blocks, 256, 0, stream>>>(X, (uint32_t)n, theta, proj_per_warp);
        else if (rows && kl == 16)
            xside_mrhs_rows_kernel<16><<<blocks, 256, 0, stream>>>(X, (uint32_t)n, theta, proj_per_warp);
        else if (rows && kl == 32)
            xside_mrhs_rows_kernel<32><<<blocks, 256, 0, stream>>>(X, (uint32_t)n, theta, proj_per_warp);
        else switch (kl) {
            case 2: xside_mrhs_kernel<2><<<blocks, 256, 0, stream>>>(X, (uint32_t)n, theta, proj_per_warp); break;
            case 4: xside_mrhs_kernel<4><<<blocks, 256, 0, stream>>>(X, (uint32_t)n, theta, proj_per_warp); break;
            case 8: xside_mrhs_kernel<8><<<blocks, 256, 0, stream>>>(X, (uint32_t)n, theta, proj_per_warp); break;
            case 16: xside_mrhs_kernel<16><<<blocks, 256, 0, stream>>>(X, (uint32_t)n, theta, proj_per_warp); break;
            case 32: xside_mrhs_kernel<32><<<blocks, 256, 0, stream>>>(X, (uint32_t)n, theta, proj_per_warp); break;
            default: xside_mrhs_kernel<64><<<blocks, 256, 0, stream>>>(X, (uint32_t)n, theta, proj_per_warp); break;
        }
        cudaEventRecord(e1, stream);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
    }
    const cudaError_t err = cudaGetLastError();
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    if (err != cudaSuccess) return fail(ASYRK_E_ThreadSpawnFailure, cudaGetErrorString(err));
    // rows shape: every lane group of a warp projects proj_per_warp rows
    const double per_warp_rows = rows ? (double)(32 / (kl / 4)) : 1.0;
    *proj_per_s = (double)blocks * 8 * per_warp_rows * (double)proj_per_warp / (ms * 1e-3);
    if (kernel_ms) *kernel_ms = ms;
    return ASYRK_OK;
}
}  // namespace ak

extern "C" asyrk_status asyrk_microbench_xside_mrhs(int64_t n, int32_t theta, int32_t kl, int32_t warps,
                                                    int64_t proj_per_warp, double* proj_per_s, double* kernel_ms) {
    using namespace ak;
    if (n < 1 || theta < 1 || theta > 32 || warps < 1 || proj_per_warp < 1 ||
        !(kl == 2 || kl == 4 || kl == 8 || kl == 16 || kl == 32 || kl == 64))
        return fail(ASYRK_E_InvalidArgument,
                    "microbench_xside_mrhs: need n, warps >= 1, 1 <= theta <= 32 and kl a power of two in 2..64");
    void* base = nullptr;
    const size_t xb = (size_t)n * kl * 4, page = 2u << 20;
    if (cudaMalloc(&base, xb + page) != cudaSuccess) return ASYRK_E_TooLarge;
    float* X = reinterpret_cast<float*>((reinterpret_cast<uintptr_t>(base) + page - 1) & ~(uintptr_t)(page - 1));
    cudaMemset(X, 0, xb);
    const asyrk_status st = (asyrk_status)xside_mrhs_on_buffer(X, n, theta, kl, warps, proj_per_warp, 0, proj_per_s, kernel_ms);
    cudaDeviceSynchronize();
    cudaFree(base);
    return st;
}
