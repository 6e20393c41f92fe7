// Exhaustive-ish check of the deterministic path's division: with y = RN(1/b)
// precomputed, q0 = RN(a*y), e = fma(-q0, b, a), q1 = fma(e, y, q0) must equal
// __ddiv_rn(a, b) bit for bit inside the guarded range (|q0| in [2^-800, 2^800],
// b in [2^-100, 2^100]). Prints the mismatch count over the sampled pairs.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t mix(uint64_t z) {
    z += 0x9e3779b97f4a7c15ull;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}

__device__ __forceinline__ double make(uint64_t r, int emin, int emax, int mode) {
    uint64_t mant = r & ((1ull << 52) - 1);
    if (mode == 1) mant = (1ull << 52) - 1 - (r & 0xff);          // mantissa near all ones
    if (mode == 2) mant = r & 0xff;                              // mantissa near zero
    if (mode == 3) mant = ((1ull << 52) - 1) ^ (1ull << (r % 52)); // one bit cleared
    const int e = emin + (int)((r >> 52) % (uint64_t)(emax - emin + 1));
    const uint64_t sign = (r >> 63) << 63;
    return __longlong_as_double((long long)(sign | ((uint64_t)(e + 1023) << 52) | mant));
}

__global__ void check(uint64_t seed, long long per_thread, unsigned long long* bad, unsigned long long* used,
                      double* example) {
    const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    unsigned long long nb = 0, nu = 0;
    for (long long k = 0; k < per_thread; ++k) {
        const uint64_t r1 = mix(seed ^ (uint64_t)(tid * per_thread + k) * 2654435761ull);
        const uint64_t r2 = mix(r1 + 17);
        const int ma = (int)(r2 >> 60) & 3, mb = (int)(r1 >> 58) & 3;
        double b;
        if ((r2 & 7) < 4) {  // row-norm products: b = nrm * nrm with nrm near 1
            const double nrm = 1.0 + ((double)(r1 & 0xfffffff) / 268435456.0 - 0.5) * ((r2 & 8) ? 1e-12 : 0.5);
            b = __dmul_rn(nrm, nrm);
        } else {
            b = fabs(make(r1, -100, 100, mb));
        }
        const double a = make(r2, -700, 700, ma);
        const double y = __drcp_rn(b);
        const double q0 = __dmul_rn(a, y);
        const double aq = fabs(q0);
        if (!(aq >= 0x1p-800 && aq <= 0x1p800 && b >= 0x1p-100 && b <= 0x1p100)) continue;
        const double e = __fma_rn(-q0, b, a);
        const double q1 = __fma_rn(e, y, q0);
        const double ref = __ddiv_rn(a, b);
        ++nu;
        if (__double_as_longlong(q1) != __double_as_longlong(ref)) {
            if (nb == 0) {
                example[0] = a;
                example[1] = b;
            }
            ++nb;
        }
    }
    atomicAdd(bad, nb);
    atomicAdd(used, nu);
}

int main() {
    unsigned long long *bad, *used;
    double* ex;
    cudaMallocManaged(&bad, 8);
    cudaMallocManaged(&used, 8);
    cudaMallocManaged(&ex, 16);
    *bad = *used = 0;
    ex[0] = ex[1] = 0;
    const int blocks = 148 * 16, threads = 256;
    const long long per = 1 << 14;
    for (int rep = 0; rep < 4; ++rep) {
        check<<<blocks, threads>>>(0x1234 + rep * 7919ull, per, bad, used, ex);
        cudaDeviceSynchronize();
    }
    printf("pairs checked %llu, mismatches %llu (first a=%.17g b=%.17g)\n", *used, *bad, ex[0], ex[1]);
    return *bad != 0;
}
