// Process-wide host runtime of the C ABI: the pieces a one-shot
// asyrk_solve_parallel call would otherwise pay for on every call.
//
//  * Stager — host->device upload through a ring of pinned chunks filled by a
//    small persistent thread pool (the caller's arrays are pageable
//    std::vectors). Chunk k+1 is filled while chunk k's DMA runs; int64
//    column indices are narrowed to int32 while staging, so they cross PCIe
//    at 4 bytes/nonzero.
//  * device memory comes from the stream-ordered pool (cudaMallocAsync) with
//    the release threshold lifted, so repeated solves reuse HBM instead of
//    paying cudaMalloc/cudaFree.
//  * a pinned, device-mapped flag slab for the coordinators' stop flags.
//  * HelperThread — one persistent thread for host work that overlaps a
//    create's uploads (the row-length scan), instead of a thread per call.
#pragma once
#include <condition_variable>
#include <deque>
#include <future>
#include <cstddef>
#include <cstdint>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

#include <cuda_runtime.h>

namespace ak {

class ThreadPool {
  public:
    explicit ThreadPool(int n);
    ~ThreadPool();
    int size() const { return (int)workers_.size() + 1; }
    // run f(t) for t in [0, size()) on the pool + the caller; returns when all done
    void run(const std::function<void(int)>& f);

  private:
    std::vector<std::thread> workers_;
    std::mutex mu_;
    std::condition_variable cv_, done_cv_;
    const std::function<void(int)>* task_ = nullptr;
    long long gen_ = 0;
    int pending_ = 0;
    bool stop_ = false;
};

class HelperThread {
  public:
    static HelperThread& get();
    // run f on the helper thread; the future reports completion (and rethrows)
    std::future<void> submit(std::function<void()> f);

  private:
    HelperThread();
    std::mutex mu_;
    std::condition_variable cv_;
    std::deque<std::packaged_task<void()>> q_;
    std::thread t_;
};

// host/stage_copy.cpp: AVX2 streaming-store copies (call only if stage_nt_supported())
bool stage_nt_supported();
void copy_nt(unsigned char* out, const unsigned char* in, size_t n);
void narrow_nt(int32_t* out, const int64_t* in, size_t n);

class Stager {
  public:
    static Stager& get();
    // dst (device) <- src (host, pageable or pinned), bytes
    void upload(void* dst, const void* src, size_t bytes, cudaStream_t s);
    // dst int32 (device) <- src int64 (host), count elements (values must fit)
    void upload_narrow(int32_t* dst, const int64_t* src, size_t count, cudaStream_t s);
    // dst (host, pageable) <- src (device), bytes, after the work queued on s;
    // returns when dst is filled (one pinned slot per chunk, threads copy out)
    void download(void* dst, const void* src, size_t bytes, cudaStream_t s);

  private:
    Stager();
    static constexpr int kSlots = 4;
    size_t chunk_ = 8u << 20;  // bytes per pinned slot (ASYRK_STAGE_CHUNK_KB)
    template <class F>
    void pipeline(size_t out_bytes, size_t out_elem, cudaStream_t s, char* dst, F&& fill);
    std::mutex mu_;
    unsigned char* slot_[kSlots] = {};
    cudaEvent_t ev_[kSlots] = {};
    int next_ = 0;
    ThreadPool pool_;
};

// stream-ordered pool allocation (release threshold lifted once per device)
cudaError_t pool_alloc(void** p, size_t bytes, cudaStream_t s);
cudaError_t pool_free(void* p, cudaStream_t s);

// pinned, device-mapped int flags
int* flag_acquire(int** dev_ptr);
void flag_release(int* host_ptr);

// pinned, device-mapped record mirrors (layout.cuh HostMirror), same slab scheme
struct HostMirror;
HostMirror* mirror_acquire(HostMirror** dev_ptr);
void mirror_release(HostMirror* host_ptr);

}  // namespace ak
