// Dev microbenchmark: random 32-byte X-row gathers (config 5's 8-column
// shard, X = n x 8 fp32) through the TMA engine (cp.async.bulk.tensor
// .tile::gather4, 4 rows per instruction, completion on an mbarrier) against
// the LSU path (float4 loads, 2 lanes per row, 16 rows per warp instruction).
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o gather4 gather4.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>

#define CK(x)                                                                          \
    do {                                                                               \
        cudaError_t e_ = (x);                                                          \
        if (e_ != cudaSuccess) {                                                       \
            fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); \
            exit(1);                                                                   \
        }                                                                              \
    } while (0)

constexpr int KL = 8;
constexpr int D = 4;    // stages per warp
constexpr int RPS = 16; // rows per stage (4 gather4)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void __launch_bounds__(256) tma_gather(const __grid_constant__ CUtensorMap tm, uint32_t n, int iters,
                                                  float* out) {
    __shared__ __align__(128) float buf[8][D][RPS * KL];
    __shared__ __align__(8) uint64_t bar[8][D];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0)
        for (int s = 0; s < D; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[w][s])));
    __syncwarp();
    uint32_t rng = (blockIdx.x * 8 + w) * 0x9E3779B9u | 1u;
    auto issue = [&](int s) {
        if (lane != 0) return;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar[w][s])),
                     "r"((uint32_t)(RPS * KL * 4))
                     : "memory");
        for (int g = 0; g < RPS / 4; ++g) {
            int r[4];
            for (int j = 0; j < 4; ++j) {
                rng = rng * 1664525u + 1013904223u;
                r[j] = (int)__umulhi(rng, n);
            }
            asm volatile(
                "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
                "%3, %4, %5, %6}], [%7];" ::"r"(smem_u32(&buf[w][s][g * 4 * KL])),
                "l"(&tm), "r"(0), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(smem_u32(&bar[w][s]))
                : "memory");
        }
    };
    for (int s = 0; s < D; ++s) issue(s);
    float acc = 0.f;
    for (int it = 0; it < iters; ++it) {
        const int s = it % D;
        const uint32_t par = (uint32_t)((it / D) & 1);
        uint32_t done = 0;
        while (!done)
            asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                         : "=r"(done)
                         : "r"(smem_u32(&bar[w][s])), "r"(par)
                         : "memory");
        const float4 v = reinterpret_cast<const float4*>(buf[w][s])[lane];
        acc += v.x + v.y + v.z + v.w;
        __syncwarp();
        if (it + D < iters) issue(s);
    }
    if (acc == 12345.f) out[0] = acc;
}

__global__ void __launch_bounds__(256) lsu_gather(const float* __restrict__ X, uint32_t n, int iters, float* out) {
    const int lane = threadIdx.x & 31, grp = lane >> 1, cl = lane & 1;
    uint32_t rng = ((blockIdx.x * 256 + threadIdx.x) >> 1) * 0x9E3779B9u | 1u;
    float acc = 0.f;
    for (int it = 0; it < iters; ++it) {  // one X row per lane group per iteration, 4 in flight
        float4 v[4];
        for (int j = 0; j < 4; ++j) {
            rng = rng * 1664525u + 1013904223u;
            v[j] = __ldcg(reinterpret_cast<const float4*>(X + (size_t)__umulhi(rng, n) * KL + 4 * cl));
        }
        for (int j = 0; j < 4; ++j) acc += v[j].x + v[j].y + v[j].z + v[j].w;
        (void)grp;
    }
    if (acc == 12345.f) out[0] = acc;
}

int main() {
    const uint32_t n = 250000;
    float* X;
    float* out;
    CK(cudaMalloc(&X, (size_t)n * KL * 4));
    CK(cudaMalloc(&out, 4));
    CK(cudaMemset(X, 0, (size_t)n * KL * 4));
    CUtensorMap tm;
    cuuint64_t gdim[2] = {KL, n};
    cuuint64_t gstr[1] = {KL * 4};
    cuuint32_t box[2] = {KL, 1};
    cuuint32_t es[2] = {1, 1};
    CUresult r = cuTensorMapEncodeTiled(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, X, gdim, gstr, box, es,
                                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                        CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        fprintf(stderr, "tensor map: %d\n", (int)r);
        return 1;
    }
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int bps : {2, 4, 8}) {
        const int blocks = sms * bps, iters = 2000;
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(a);
            tma_gather<<<blocks, 256>>>(tm, n, iters, out);
            cudaEventRecord(b);
            CK(cudaEventSynchronize(b));
        }
        float ms = 0.f;
        cudaEventElapsedTime(&ms, a, b);
        CK(cudaGetLastError());
        const double rows = (double)blocks * 8 * iters * RPS;
        printf("TMA gather4: %d blocks/SM: %.3f ms, %.2e X rows/s\n", bps, ms, rows / (ms * 1e-3));
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(a);
            lsu_gather<<<blocks, 256>>>(X, n, iters, out);
            cudaEventRecord(b);
            CK(cudaEventSynchronize(b));
        }
        cudaEventElapsedTime(&ms, a, b);
        CK(cudaGetLastError());
        const double rows2 = (double)blocks * 128 * iters * 4;
        printf("LSU float4:  %d blocks/SM: %.3f ms, %.2e X rows/s\n", bps, ms, rows2 / (ms * 1e-3));
    }
    return 0;
}
