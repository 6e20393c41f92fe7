// Non-temporal staging copies for the pinned upload ring (runtime.cu Stager).
// Compiled by g++ (AVX2 target attribute, chosen at run time).
#include <immintrin.h>

#include <cstddef>
#include <cstdint>

namespace ak {

bool stage_nt_supported() { return __builtin_cpu_supports("avx2"); }

// Staging fills are host-memory bound: streaming (non-temporal) stores into
// the pinned slot skip the read-for-ownership of every destination line.
__attribute__((target("avx2"))) void copy_nt(unsigned char* out, const unsigned char* in, size_t n) {
    size_t k = 0;
    while (k < n && (reinterpret_cast<uintptr_t>(out + k) & 31)) {
        out[k] = in[k];
        ++k;
    }
    for (; k + 128 <= n; k += 128) {
        const __m256i a = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(in + k));
        const __m256i b = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(in + k + 32));
        const __m256i c = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(in + k + 64));
        const __m256i d = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(in + k + 96));
        _mm256_stream_si256(reinterpret_cast<__m256i*>(out + k), a);
        _mm256_stream_si256(reinterpret_cast<__m256i*>(out + k + 32), b);
        _mm256_stream_si256(reinterpret_cast<__m256i*>(out + k + 64), c);
        _mm256_stream_si256(reinterpret_cast<__m256i*>(out + k + 96), d);
    }
    for (; k < n; ++k) out[k] = in[k];
    _mm_sfence();
}

__attribute__((target("avx2"))) void narrow_nt(int32_t* out, const int64_t* in, size_t n) {
    size_t k = 0;
    while (k < n && (reinterpret_cast<uintptr_t>(out + k) & 31)) {
        out[k] = (int32_t)in[k];
        ++k;
    }
    const __m256i pick = _mm256_setr_epi32(0, 2, 4, 6, 0, 2, 4, 6);
    for (; k + 8 <= n; k += 8) {
        const __m256i a = _mm256_permutevar8x32_epi32(_mm256_loadu_si256(reinterpret_cast<const __m256i*>(in + k)), pick);
        const __m256i b =
            _mm256_permutevar8x32_epi32(_mm256_loadu_si256(reinterpret_cast<const __m256i*>(in + k + 4)), pick);
        _mm256_stream_si256(reinterpret_cast<__m256i*>(out + k), _mm256_permute2x128_si256(a, b, 0x20));
    }
    for (; k < n; ++k) out[k] = (int32_t)in[k];
    _mm_sfence();
}

}  // namespace ak
