// Probe: cost of cudaHostRegister / Unregister on a freshly touched 48 MB
// pageable buffer and the H2D rate from it, against a pinned staging copy.
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cuda_runtime.h>

static double ms(std::chrono::steady_clock::time_point a, std::chrono::steady_clock::time_point b) {
    return std::chrono::duration<double, std::milli>(b - a).count();
}

int main() {
    const size_t bytes = 48u << 20;
    void* d;
    cudaMalloc(&d, bytes);
    cudaFree(0);
    for (int rep = 0; rep < 4; ++rep) {
        char* h = static_cast<char*>(std::malloc(bytes));
        std::memset(h, rep + 1, bytes);
        auto t0 = std::chrono::steady_clock::now();
        cudaError_t e = cudaHostRegister(h, bytes, cudaHostRegisterDefault);
        auto t1 = std::chrono::steady_clock::now();
        cudaMemcpy(d, h, bytes, cudaMemcpyHostToDevice);
        auto t2 = std::chrono::steady_clock::now();
        cudaHostUnregister(h);
        auto t3 = std::chrono::steady_clock::now();
        cudaMemcpy(d, h, bytes, cudaMemcpyHostToDevice);  // pageable, driver-staged
        auto t4 = std::chrono::steady_clock::now();
        std::printf("register %.3f ms (%s), H2D registered %.3f ms (%.1f GB/s), unregister %.3f ms, pageable H2D %.3f ms\n",
                    ms(t0, t1), cudaGetErrorString(e), ms(t1, t2), bytes / (ms(t1, t2) * 1e6), ms(t2, t3), ms(t3, t4));
        std::free(h);
    }
    return 0;
}
