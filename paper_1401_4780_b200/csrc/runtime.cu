// Host runtime of the C ABI (runtime.h).
#include <chrono>
#include "env.h"
#include "runtime.h"
#include "layout.cuh"

#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <stdexcept>

namespace ak {

constexpr int kMaxDevices = 64;  // per-device caches and pools

ThreadPool::ThreadPool(int n) {
    for (int t = 1; t < n; ++t) {
        workers_.emplace_back([this, t] {
            long long seen = 0;
            for (;;) {
                const std::function<void(int)>* task;
                {
                    std::unique_lock<std::mutex> lk(mu_);
                    cv_.wait(lk, [&] { return stop_ || gen_ != seen; });
                    if (stop_) return;
                    seen = gen_;
                    task = task_;
                }
                (*task)(t);
                std::lock_guard<std::mutex> lk(mu_);
                if (--pending_ == 0) done_cv_.notify_one();
            }
        });
    }
}

ThreadPool::~ThreadPool() {
    {
        std::lock_guard<std::mutex> lk(mu_);
        stop_ = true;
    }
    cv_.notify_all();
    for (auto& w : workers_) w.join();
}

void ThreadPool::run(const std::function<void(int)>& f) {
    {
        std::lock_guard<std::mutex> lk(mu_);
        task_ = &f;
        pending_ = (int)workers_.size();
        ++gen_;
    }
    cv_.notify_all();
    f(0);
    std::unique_lock<std::mutex> lk(mu_);
    done_cv_.wait(lk, [&] { return pending_ == 0; });
}

HelperThread::HelperThread() {
    t_ = std::thread([this] {
        for (;;) {
            std::packaged_task<void()> task;
            {
                std::unique_lock<std::mutex> lk(mu_);
                cv_.wait(lk, [&] { return !q_.empty(); });
                task = std::move(q_.front());
                q_.pop_front();
            }
            task();
        }
    });
    t_.detach();  // process lifetime
}

HelperThread& HelperThread::get() {
    static HelperThread* h = new HelperThread();
    return *h;
}

std::future<void> HelperThread::submit(std::function<void()> f) {
    std::packaged_task<void()> task(std::move(f));
    std::future<void> fut = task.get_future();
    {
        std::lock_guard<std::mutex> lk(mu_);
        q_.push_back(std::move(task));
    }
    cv_.notify_one();
    return fut;
}

static int stager_threads() {
    if (const char* e = getenv("ASYRK_STAGER_THREADS")) return std::max(1, atoi(e));
    const unsigned hc = std::thread::hardware_concurrency();
    return (int)std::max(1u, std::min(12u, hc ? hc * 3 / 4 : 1u));  // fills are memory-bound; leave the rest
}

Stager::Stager() : pool_(stager_threads()) {
    if (const char* e = getenv("ASYRK_STAGE_CHUNK_KB")) chunk_ = std::max<size_t>(64, strtoull(e, nullptr, 10)) << 10;
    for (int k = 0; k < kSlots; ++k) {
        if (cudaHostAlloc((void**)&slot_[k], chunk_, cudaHostAllocPortable) != cudaSuccess)
            throw std::runtime_error("pinned staging allocation failed");
        cudaEventCreateWithFlags(&ev_[k], cudaEventDisableTiming);
    }
}

// one Stager per device: its events (and the DMA streams it is used with)
// belong to that device; process lifetime (pinned memory freed at exit)
Stager& Stager::get() {
    static std::mutex mu;
    static Stager* per[kMaxDevices] = {};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices) dev = 0;
    std::lock_guard<std::mutex> lk(mu);
    if (!per[dev]) per[dev] = new Stager();
    return *per[dev];
}

// Fill pinned chunks with fill(dst_chunk, first_elem, n_elems, thread, nthreads)
// and DMA them to dst; out_elem = bytes per staged element.
template <class F>
void Stager::pipeline(size_t out_bytes, size_t out_elem, cudaStream_t s, char* dst, F&& fill) {
    std::lock_guard<std::mutex> lk(mu_);
    const size_t per_chunk = chunk_ / out_elem;
    const size_t total = out_bytes / out_elem;
    static const bool prof = env_flag("ASYRK_STAGE_PROFILE");  // diagnostics: fill vs wait
    double t_wait = 0.0, t_fill = 0.0;
    const auto t_start = std::chrono::steady_clock::now();
    for (size_t e0 = 0; e0 < total; e0 += per_chunk) {
        const size_t ne = std::min(per_chunk, total - e0);
        const int k = next_;
        next_ = (next_ + 1) % kSlots;
        const auto t0 = std::chrono::steady_clock::now();
        cudaEventSynchronize(ev_[k]);  // slot's previous DMA done
        const auto t1 = std::chrono::steady_clock::now();
        t_wait += std::chrono::duration<double, std::milli>(t1 - t0).count();
        unsigned char* slot = slot_[k];
        const int nt = pool_.size();
        std::function<void(int)> task = [&](int t) {
            const size_t a = ne * t / nt, b = ne * (t + 1) / nt;
            if (b > a) fill(slot + a * out_elem, e0 + a, b - a);
        };
        if (ne * out_elem >= (1u << 20))
            pool_.run(task);
        else
            fill(slot, e0, ne);
        t_fill += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t1).count();
        if (cudaMemcpyAsync(dst + e0 * out_elem, slot, ne * out_elem, cudaMemcpyHostToDevice, s) != cudaSuccess)
            throw std::runtime_error("staged upload failed");
        cudaEventRecord(ev_[k], s);
    }
    if (prof)
        fprintf(stderr, "[stage] %9zu B: issue %.3f ms (fill %.3f, slot waits %.3f)\n", out_bytes,
                std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_start).count(), t_fill,
                t_wait);
}

static bool have_avx2() {
    static const bool ok = stage_nt_supported() && !env_flag("ASYRK_NO_NT_STAGING");
    return ok;
}

void Stager::upload(void* dst, const void* src, size_t bytes, cudaStream_t s) {
    const unsigned char* sp = static_cast<const unsigned char*>(src);
    const bool nt = have_avx2();
    pipeline(bytes, 1, s, static_cast<char*>(dst), [sp, nt](unsigned char* out, size_t first, size_t n) {
        if (nt)
            copy_nt(out, sp + first, n);
        else
            std::memcpy(out, sp + first, n);
    });
}

void Stager::download(void* dst, const void* src, size_t bytes, cudaStream_t s) {
    std::lock_guard<std::mutex> lk(mu_);
    unsigned char* out = static_cast<unsigned char*>(dst);
    const unsigned char* in = static_cast<const unsigned char*>(src);
    const size_t chunks = (bytes + chunk_ - 1) / chunk_;
    std::vector<int> slot_of(chunks);
    auto issue = [&](size_t c) {  // DMA chunk c into the next slot
        const int k = next_;
        next_ = (next_ + 1) % kSlots;
        cudaEventSynchronize(ev_[k]);  // the slot's previous transfer is done
        const size_t o = c * chunk_, nb = std::min(chunk_, bytes - o);
        if (cudaMemcpyAsync(slot_[k], in + o, nb, cudaMemcpyDeviceToHost, s) != cudaSuccess ||
            cudaEventRecord(ev_[k], s) != cudaSuccess)
            throw std::runtime_error("staged download failed");
        slot_of[c] = k;
    };
    // chunk c + 1 crosses PCIe while chunk c is copied out of its slot
    if (chunks) issue(0);
    for (size_t c = 0; c < chunks; ++c) {
        if (c + 1 < chunks) issue(c + 1);
        const int k = slot_of[c];
        if (cudaEventSynchronize(ev_[k]) != cudaSuccess) throw std::runtime_error("staged download failed");
        const size_t o = c * chunk_, nb = std::min(chunk_, bytes - o);
        const unsigned char* slot = slot_[k];
        if (nb >= (1u << 20)) {
            const int nt = pool_.size();
            pool_.run([&](int t) {
                const size_t a = nb * t / nt, b = nb * (t + 1) / nt;
                if (b > a) std::memcpy(out + o + a, slot + a, b - a);
            });
        } else {
            std::memcpy(out + o, slot, nb);
        }
    }
}

void Stager::upload_narrow(int32_t* dst, const int64_t* src, size_t count, cudaStream_t s) {
    const bool nt = have_avx2();
    pipeline(count * 4, 4, s, reinterpret_cast<char*>(dst), [src, nt](unsigned char* out, size_t first, size_t n) {
        int32_t* o = reinterpret_cast<int32_t*>(out);
        const int64_t* in = src + first;
        if (nt) {
            narrow_nt(o, in, n);
            return;
        }
        for (size_t k = 0; k < n; ++k) o[k] = (int32_t)in[k];
    });
}

static bool pool_debug() {
    static int d = -1;
    if (d < 0) d = env_flag("ASYRK_DEBUG_POOL") ? 1 : 0;
    return d == 1;
}

static bool no_pool() {
    static int d = -1;
    if (d < 0) d = env_flag("ASYRK_NO_POOL") ? 1 : 0;
    return d == 1;
}

int current_sm_count() {
    static std::atomic<int> cache[kMaxDevices];
    int dev = 0;
    cudaGetDevice(&dev);
    int v = (dev >= 0 && dev < kMaxDevices) ? cache[dev].load(std::memory_order_relaxed) : 0;
    if (!v) {
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
        if (v <= 0) v = 1;
        if (dev >= 0 && dev < kMaxDevices) cache[dev].store(v, std::memory_order_relaxed);
    }
    return v;
}

cudaError_t pool_alloc(void** p, size_t bytes, cudaStream_t s) {
    static std::atomic<uint64_t> configured{0};  // one bit per device ordinal
    int dev = 0;
    cudaGetDevice(&dev);
    const uint64_t bit = (dev >= 0 && dev < kMaxDevices) ? (1ull << dev) : 0;
    if (!bit || !(configured.load(std::memory_order_relaxed) & bit)) {
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
            uint64_t thr = UINT64_MAX;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
        }
        configured.fetch_or(bit, std::memory_order_relaxed);
    }
    const cudaError_t e = no_pool() ? cudaMalloc(p, bytes ? bytes : 1) : cudaMallocAsync(p, bytes ? bytes : 1, s);
    static const bool dbg = env_flag("ASYRK_DEBUG_POOL");
    if (dbg) fprintf(stderr, "[pool] alloc %p %zu\n", *p, bytes);
    return e;
}

cudaError_t pool_free(void* p, cudaStream_t s) {
    if (pool_debug() && p) fprintf(stderr, "[pool] free  %p\n", p);
    if (no_pool()) return p ? cudaFree(p) : cudaSuccess;
    return p ? cudaFreeAsync(p, s) : cudaSuccess;
}

namespace {
std::mutex g_flag_mu;
int* g_flag_host = nullptr;
int* g_flag_dev = nullptr;
std::vector<int> g_flag_free;
constexpr int kFlags = 1024;
}  // namespace

int* flag_acquire(int** dev_ptr) {
    std::lock_guard<std::mutex> lk(g_flag_mu);
    if (!g_flag_host) {
        if (cudaHostAlloc((void**)&g_flag_host, kFlags * sizeof(int), cudaHostAllocMapped | cudaHostAllocPortable) != cudaSuccess)
            return nullptr;
        cudaHostGetDevicePointer((void**)&g_flag_dev, g_flag_host, 0);
        for (int k = kFlags - 1; k >= 0; --k) g_flag_free.push_back(k);
    }
    if (g_flag_free.empty()) return nullptr;
    const int k = g_flag_free.back();
    g_flag_free.pop_back();
    *dev_ptr = g_flag_dev + k;
    return g_flag_host + k;
}

void flag_release(int* host_ptr) {
    if (!host_ptr) return;
    std::lock_guard<std::mutex> lk(g_flag_mu);
    g_flag_free.push_back((int)(host_ptr - g_flag_host));
}

namespace {
constexpr int kMirrors = 256;
std::mutex g_mirror_mu;
HostMirror* g_mirror_host = nullptr;
HostMirror* g_mirror_dev = nullptr;
std::vector<int> g_mirror_free;
}  // namespace

HostMirror* mirror_acquire(HostMirror** dev_ptr) {
    std::lock_guard<std::mutex> lk(g_mirror_mu);
    if (!g_mirror_host) {
        if (cudaHostAlloc((void**)&g_mirror_host, kMirrors * sizeof(HostMirror), cudaHostAllocMapped | cudaHostAllocPortable) != cudaSuccess)
            return nullptr;
        cudaHostGetDevicePointer((void**)&g_mirror_dev, g_mirror_host, 0);
        std::memset(g_mirror_host, 0, kMirrors * sizeof(HostMirror));
        for (int k = kMirrors - 1; k >= 0; --k) g_mirror_free.push_back(k);
    }
    if (g_mirror_free.empty()) return nullptr;
    const int k = g_mirror_free.back();
    g_mirror_free.pop_back();
    *dev_ptr = g_mirror_dev + k;
    return g_mirror_host + k;
}

void mirror_release(HostMirror* host_ptr) {
    if (!host_ptr) return;
    std::lock_guard<std::mutex> lk(g_mirror_mu);
    g_mirror_free.push_back((int)(host_ptr - g_mirror_host));
}

}  // namespace ak
