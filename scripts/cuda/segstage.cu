// Dev microbenchmark: the monitor's gather SpMV (y = A z, random z indices)
// with z staged through shared memory by segments (bulk copies, double
// buffered) vs gathered from global memory (L2 sectors) — the envelope for
// a segmented monitor pass. Synthetic entries (uniform random indices), one
// persistent CTA per SM.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o segstage segstage.cu
//   ./segstage <z_len> <nnz>    (config 2 rows pass: 100000 6000000; cols: 200000 6000000)
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                              \
    do {                                                                                   \
        cudaError_t e_ = (x);                                                              \
        if (e_ != cudaSuccess) {                                                           \
            fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_));     \
            exit(1);                                                                       \
        }                                                                                  \
    } while (0)

constexpr int kThreads = 1024;
constexpr int kSeg = 12288;  // doubles per segment (96 KB)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
    uint32_t done = 0;
    while (!done)
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                     : "=r"(done)
                     : "r"(smem_u32(bar)), "r"(phase)
                     : "memory");
}

// entries of CTA c, segment s: [off[c*S+s], off[c*S+s+1]); idx local to the segment
__global__ void __launch_bounds__(kThreads, 1) staged(const double* __restrict__ z, long long zlen, int S,
                                                      const long long* __restrict__ off, const uint16_t* __restrict__ idx,
                                                      const double* __restrict__ val, double* out) {
    extern __shared__ __align__(16) unsigned char smem[];
    double* buf = reinterpret_cast<double*>(smem);  // 2 x kSeg
    __shared__ uint64_t bar[2];
    if (threadIdx.x == 0) {
        for (int k = 0; k < 2; ++k) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar + k)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    auto issue = [&](int s) {
        const int k = s & 1;
        const long long z0 = (long long)s * kSeg;
        const long long cnt = min((long long)kSeg, zlen - z0);
        const uint32_t bytes = (uint32_t)(cnt * 8);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar + k)), "r"(bytes)
                     : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                         smem_u32(buf + k * kSeg)),
                     "l"(z + z0), "r"(bytes), "r"(smem_u32(bar + k))
                     : "memory");
    };
    if (threadIdx.x == 0) {
        issue(0);
        if (S > 1) issue(1);
    }
    double acc = 0.0;
    for (int s = 0; s < S; ++s) {
        const int k = s & 1;
        mbar_wait(bar + k, (uint32_t)((s >> 1) & 1));
        const double* zs = buf + k * kSeg;
        const long long e0 = off[(long long)blockIdx.x * S + s], e1 = off[(long long)blockIdx.x * S + s + 1];
        constexpr int U = 8;
        for (long long e = e0 + threadIdx.x; e < e1; e += U * kThreads) {
            double v[U];
            int ix[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const long long q = e + (long long)u * kThreads;
                v[u] = q < e1 ? __ldg(val + q) : 0.0;
                ix[u] = q < e1 ? __ldg(idx + q) : 0;
            }
#pragma unroll
            for (int u = 0; u < U; ++u) acc += v[u] * zs[ix[u]];
        }
        __syncthreads();
        if (threadIdx.x == 0 && s + 2 < S) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            issue(s + 2);
        }
    }
    out[(long long)blockIdx.x * kThreads + threadIdx.x] = acc;
}


// staged, with the next segment's entries prefetched into registers while
// the current segment is processed (one chunk of U entries per thread per segment)
template <int U>
__global__ void __launch_bounds__(kThreads, 1) staged_pipe(const double* __restrict__ z, long long zlen, int S,
                                                           const long long* __restrict__ off,
                                                           const uint16_t* __restrict__ idx,
                                                           const double* __restrict__ val, double* out) {
    extern __shared__ __align__(16) unsigned char smem[];
    double* buf = reinterpret_cast<double*>(smem);  // 2 x kSeg
    __shared__ uint64_t bar[2];
    if (threadIdx.x == 0) {
        for (int k = 0; k < 2; ++k) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar + k)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    auto issue = [&](int s) {
        const int k = s & 1;
        const long long z0 = (long long)s * kSeg;
        const long long cnt = min((long long)kSeg, zlen - z0);
        const uint32_t bytes = (uint32_t)(cnt * 8);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar + k)), "r"(bytes)
                     : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                         smem_u32(buf + k * kSeg)),
                     "l"(z + z0), "r"(bytes), "r"(smem_u32(bar + k))
                     : "memory");
    };
    if (threadIdx.x == 0) {
        issue(0);
        if (S > 1) issue(1);
    }
    double acc = 0.0;
    double v[U];
    int ix[U];
    auto load = [&](int s, double* vv, int* ii) {
        const long long e0 = off[(long long)blockIdx.x * S + s], e1 = off[(long long)blockIdx.x * S + s + 1];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const long long q = e0 + threadIdx.x + (long long)u * kThreads;
            vv[u] = q < e1 ? __ldg(val + q) : 0.0;
            ii[u] = q < e1 ? __ldg(idx + q) : 0;
        }
    };
    load(0, v, ix);
    for (int s = 0; s < S; ++s) {
        const int k = s & 1;
        double vn[U];
        int in[U];
        if (s + 1 < S) load(s + 1, vn, in);
        mbar_wait(bar + k, (uint32_t)((s >> 1) & 1));
        const double* zs = buf + k * kSeg;
#pragma unroll
        for (int u = 0; u < U; ++u) acc += v[u] * zs[ix[u]];
        __syncthreads();
        if (threadIdx.x == 0 && s + 2 < S) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            issue(s + 2);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            v[u] = vn[u];
            ix[u] = in[u];
        }
    }
    out[(long long)blockIdx.x * kThreads + threadIdx.x] = acc;
}

__global__ void __launch_bounds__(kThreads, 1) gathered(const double* __restrict__ z, int S,
                                                        const long long* __restrict__ off,
                                                        const uint16_t* __restrict__ idx, const double* __restrict__ val,
                                                        double* out) {
    double acc = 0.0;
    for (int s = 0; s < S; ++s) {
        const double* zs = z + (long long)s * kSeg;
        const long long e0 = off[(long long)blockIdx.x * S + s], e1 = off[(long long)blockIdx.x * S + s + 1];
        constexpr int U = 8;
        for (long long e = e0 + threadIdx.x; e < e1; e += U * kThreads) {
            double v[U];
            int ix[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const long long q = e + (long long)u * kThreads;
                v[u] = q < e1 ? __ldg(val + q) : 0.0;
                ix[u] = q < e1 ? __ldg(idx + q) : 0;
            }
            double zv[U];
#pragma unroll
            for (int u = 0; u < U; ++u) zv[u] = __ldg(zs + ix[u]);
#pragma unroll
            for (int u = 0; u < U; ++u) acc += v[u] * zv[u];
        }
    }
    out[(long long)blockIdx.x * kThreads + threadIdx.x] = acc;
}

int main(int argc, char** argv) {
    const long long zlen = argc > 1 ? atoll(argv[1]) : 100000;
    const long long nnz = argc > 2 ? atoll(argv[2]) : 6000000;
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    const int S = (int)((zlen + kSeg - 1) / kSeg);
    const long long parts = (long long)sms * S;
    std::vector<long long> off(parts + 1);
    std::vector<uint16_t> idx(nnz);
    std::vector<double> val(nnz);
    uint64_t r = 88172645463325252ull;
    auto rnd = [&] {
        r ^= r << 13;
        r ^= r >> 7;
        r ^= r << 17;
        return r;
    };
    for (long long p = 0; p <= parts; ++p) off[p] = nnz * p / parts;
    for (long long p = 0; p < parts; ++p) {
        const int s = (int)(p % S);
        const long long segn = std::min<long long>(kSeg, zlen - (long long)s * kSeg);
        for (long long e = off[p]; e < off[p + 1]; ++e) {
            idx[e] = (uint16_t)(rnd() % segn);
            val[e] = 1.0 + (double)(rnd() % 1000) * 1e-3;
        }
    }
    double *dz, *dv, *dout;
    long long* doff;
    uint16_t* di;
    CK(cudaMalloc(&dz, zlen * 8));
    CK(cudaMalloc(&dv, nnz * 8));
    CK(cudaMalloc(&di, nnz * 2));
    CK(cudaMalloc(&doff, (parts + 1) * 8));
    CK(cudaMalloc(&dout, (size_t)sms * kThreads * 8));
    CK(cudaMemset(dz, 0, zlen * 8));
    CK(cudaMemcpy(dv, val.data(), nnz * 8, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(di, idx.data(), nnz * 2, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(doff, off.data(), (parts + 1) * 8, cudaMemcpyHostToDevice));
    const int smem = 2 * kSeg * 8;
    CK(cudaFuncSetAttribute(staged, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    void* flush;
    CK(cudaMalloc(&flush, 256 << 20));
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    CK(cudaFuncSetAttribute(staged_pipe<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    const long long per = (nnz + (long long)sms * S - 1) / ((long long)sms * S);
    for (int mode = 0; mode < 3; ++mode) {
        if (mode == 2 && per > 8 * kThreads) continue;
        float tot = 0.f;
        const int reps = 20;
        for (int it = -3; it < reps; ++it) {
            CK(cudaMemsetAsync(flush, it & 0xff, 256 << 20));
            cudaEventRecord(a);
            if (mode == 0)
                staged<<<sms, kThreads, smem>>>(dz, zlen, S, doff, di, dv, dout);
            else if (mode == 1)
                gathered<<<sms, kThreads>>>(dz, S, doff, di, dv, dout);
            else
                staged_pipe<8><<<sms, kThreads, smem>>>(dz, zlen, S, doff, di, dv, dout);
            cudaEventRecord(b);
            CK(cudaEventSynchronize(b));
            float ms = 0.f;
            cudaEventElapsedTime(&ms, a, b);
            if (it >= 0) tot += ms;
        }
        CK(cudaGetLastError());
        const double us = 1e3 * tot / 20;
        printf("%s z=%lld nnz=%lld segments=%d: %.2f us per pass (entry stream %.1f GB/s)\n",
               mode == 0 ? "staged  " : mode == 1 ? "gathered" : "pipe    ", zlen, nnz, S, us, (double)nnz * 10 / us * 1e-3);
    }
    return 0;
}
