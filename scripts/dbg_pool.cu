// dev probe: stream-ordered allocator behaviour on this driver
#include <cstdio>
#include <cuda_runtime.h>
#define C(x) do { cudaError_t e = (x); printf("%-70s -> %s\n", #x, cudaGetErrorString(e)); } while (0)
__global__ void touch(char* p) { p[threadIdx.x] = 1; }
int main() {
    cudaStream_t s; C(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    cudaMemPool_t pool; C(cudaDeviceGetDefaultMemPool(&pool, 0));
    unsigned long long thr = ~0ull; C(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
    void *a = 0, *b = 0, *c = 0, *d = 0;
    C(cudaMallocAsync(&a, 1 << 16, s));
    C(cudaFreeAsync(a, s));
    C(cudaMallocAsync(&b, 12288, s));
    printf("a=%p b=%p\n", a, b);
    touch<<<1, 32, 0, s>>>((char*)b);
    C(cudaStreamSynchronize(s));
    char h[16]; C(cudaMemcpy(h, b, 16, cudaMemcpyDeviceToHost));
    C(cudaFreeAsync(b, s));
    C(cudaMallocAsync(&c, 12288, s));
    cudaEvent_t ev; C(cudaEventCreate(&ev)); C(cudaEventRecord(ev, s)); C(cudaEventSynchronize(ev));
    C(cudaFreeAsync(c, s));
    C(cudaMallocAsync(&d, 12288, 0));
    C(cudaFreeAsync(d, s));
    return 0;
}
