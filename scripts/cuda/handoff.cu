// Microbenchmark: latency of a cross-warp dependency hand-off through a
// shared-memory counter (the deterministic dataflow kernel's pattern).
// W warps run a chain of N events round-robin; event q waits until
// flag == q (acquire load poll), does `work` dependent DADDs, then publishes
// flag = q + 1 (release store). Prints cycles per event.
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>
__global__ void chain(int N, int work, int sleep_ns, long long* cycles, double* sink) {
    __shared__ int flag;
    __shared__ double xs[64];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, W = blockDim.x >> 5;
    if (threadIdx.x == 0) flag = 0;
    if (threadIdx.x < 64) xs[threadIdx.x] = 1.0;
    __syncthreads();
    const unsigned fs = (unsigned)__cvta_generic_to_shared(&flag);
    long long t0 = clock64();
    double acc = 1.0 + lane;
    for (int q = w; q < N; q += W) {
        for (;;) {
            int v;
            if (MODE == 0) asm volatile("ld.acquire.cta.shared.b32 %0, [%1];" : "=r"(v) : "r"(fs) : "memory");
            else asm volatile("ld.volatile.shared.b32 %0, [%1];" : "=r"(v) : "r"(fs) : "memory");
            if (__all_sync(0xffffffffu, v == q)) break;
            if (sleep_ns) __nanosleep(sleep_ns);
        }
        double s = xs[lane & 63];
        for (int k = 0; k < work; ++k) s = __dadd_rn(s, acc);
        xs[lane & 63] = s;
        if (MODE == 0) asm volatile("st.release.cta.shared.b32 [%0], %1;" ::"r"(fs), "r"(q + 1) : "memory");
        else {
            __threadfence_block();
            asm volatile("st.volatile.shared.b32 [%0], %1;" ::"r"(fs), "r"(q + 1) : "memory");
        }
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) *cycles = t1 - t0;
    if (threadIdx.x == 0) *sink = xs[0];
}

int main() {
    long long* cyc;
    double* sink;
    cudaMallocManaged(&cyc, 8);
    cudaMallocManaged(&sink, 8);
    const int N = 20000;
    for (int mode = 0; mode < 2; ++mode)
        for (int W : {2, 8, 32})
            for (int work : {0, 16})
                for (int sl : {0, 32}) {
                    if (mode == 0) chain<0><<<1, 32 * W>>>(N, work, sl, cyc, sink);
                    else chain<1><<<1, 32 * W>>>(N, work, sl, cyc, sink);
                    cudaDeviceSynchronize();
                    if (mode == 0) chain<0><<<1, 32 * W>>>(N, work, sl, cyc, sink);
                    else chain<1><<<1, 32 * W>>>(N, work, sl, cyc, sink);
                    cudaDeviceSynchronize();
                    printf("%s warps %2d work %2d sleep %2d: %6.1f cycles per event\n",
                           mode ? "volatile+fence" : "acq/rel", W, work, sl, (double)*cyc / N);
                }
    return 0;
}
