// The C ABI (include/asyrk_cuda.h): device-resident systems, the solve
// driver (the reference's coordinator, ref/src/parallel.cpp:220-445, moved
// onto the stream) and the one-shot host-buffer entry points.
//
// Solve driver. One "chunk" = span = min(snapshot_interval, epochs - e)
// epochs of row events followed by the residual monitor and a finalize
// kernel that writes the trace record and decides stop/NonFinite on the
// device (DevState). The host only enqueues chunks ahead (bounded lookahead)
// and polls a mapped pinned flag; chunks enqueued after the stop decision
// exit at their first instruction. No host round trip sits between epochs.
#include <algorithm>
#include "env.h"
#include <chrono>
#include <cmath>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include <dlfcn.h>
#include <nccl.h>

#include "capi_common.h"
#include "host_seq.h"
#include "schedule.h"
#include "kernels.h"

using namespace ak;

asyrk_status xside_on_buffer(void* x, int64_t n, int32_t theta, int32_t precision, int32_t warps, int64_t per_warp,
                             int32_t mode, void* stream, double* proj_per_s, double* kernel_ms);  // microbench.cu

namespace ak {
std::string& err_buf() {
    static thread_local std::string e;
    return e;
}
thread_local cudaStream_t g_alloc_stream = nullptr;
}  // namespace ak

namespace {

constexpr int kLookahead = 4;      // chunks in flight beyond the last confirmed one
constexpr int kTimedLaunches = 1024;  // worker launches timed with event pairs per solve
// async drivers time one worker launch in kTimeEvery with an event pair —
// launches 1, 9, 17, ... (launch 0 follows the cold start of a solve): a pair
// between two launches costs ~5.6 us of stream time (0.24 ms per config-2
// solve when every launch was timed); worker_ms scales the sample to all launches
constexpr long long kTimeEvery = 8;
inline bool timed_launch(long long b) { return b % kTimeEvery == 1; }

}  // namespace

struct asyrk_system {
    int64_t m = 0, n = 0, nnz = 0;
    int precision = 0;
    bool normalized = false;
    bool uniform = true;
    uint32_t max_len = 0;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    int dev = 0;  // the device current at create: frees and the stream / scratch pools are per device

    // layout
    unsigned char* rec = nullptr;
    uint2* row_info = nullptr;
    uint32_t stride16 = 0, uniform_len = 0;
    double* row_norm = nullptr;
    size_t rec_bytes = 0;
    long long* grp_off = nullptr;  // SELL-32 columns (CscDev)
    int32_t* col_len = nullptr;
    int32_t* col_perm = nullptr;   // sigma-sorted column copy: position -> column
    int32_t* sell_row = nullptr;
    void* sell_val = nullptr;
    long long* rgrp_off = nullptr;  // SELL-32 rows (monitor pass 1)
    int32_t* row_len = nullptr;
    int32_t* rsell_col = nullptr;
    void* rsell_val = nullptr;
    double* b = nullptr;            // right-hand side (also in the record headers)
    long long* col_ptr = nullptr;   // plain CSC (fp64 and multi-RHS systems)
    int32_t* csc_row = nullptr;
    double* csc_val = nullptr;
    AliasEntry* alias = nullptr;  // device alias table (async norm_proportional), built lazily

    // host copies for sequence generation
    std::vector<int32_t> h_len;
    std::vector<double> h_norm;
    std::unique_ptr<HostAlias> h_alias;

    // solve state
    void* x = nullptr;        // X[n]
    void* x_base = nullptr;   // allocation holding x (x may be offset inside it, ASYRK_X_ALIGN)
    double* xd = nullptr;     // fp64 staging (x0, export, det x)
    void* shadow = nullptr;
    double* x0d = nullptr;
    double* xstar = nullptr;
    double* r = nullptr;
    void* r_base = nullptr;        // allocation holding r (2 MB aligned, see x)
    double* g = nullptr;
    double* part = nullptr;
    DevRecord* recs = nullptr;
    long long rec_cap = 0;
    DevState* st = nullptr;
    unsigned long long* incr = nullptr;
    double* audit_part = nullptr;  // instrumented async solves: per-warp checksums [W][kAuditK] + counts [W]
    long long audit_cap = 0;       // warps audit_part holds
    double* scratch = nullptr;
    int* host_flag = nullptr;      // pinned mapped
    int* host_flag_dev = nullptr;
    HostMirror* mirror = nullptr;  // pinned mapped: latest record for the host-driven monitor schedule
    HostMirror* mirror_dev = nullptr;
    HostMirror* mirror0 = nullptr;  // record 0 taken beside the first workers (its own, so it is never overwritten)
    HostMirror* mirror0_dev = nullptr;
    void* host_scalar = nullptr;   // pinned scratch (kPinBytes): small device -> host reads, the final state + records
    long long pin_recs = -1;       // records of the last solve already copied into host_scalar (-1: none)
    // the monitor's structures (row / column SELL, plain CSC) finish on bstream
    // after create returns; every consumer's stream waits on ev_mon_ready
    cudaStream_t bstream = nullptr;
    cudaEvent_t ev_mon_ready = nullptr;

    // det staging ring
    int32_t* seq_dev[kLookahead + 1] = {};
    int32_t* pick_dev[kLookahead + 1] = {};
    int32_t* seq_host[kLookahead + 1] = {};
    int32_t* pick_host[kLookahead + 1] = {};
    long long* flat_dev[kLookahead + 1] = {};   // ragged rows: event -> offset of its (event, nonzero) pairs
    long long* flat_host[kLookahead + 1] = {};
    // dataflow prepass outputs, double-buffered: chunk k+1's prepass runs on
    // pstream while chunk k's dataflow kernel runs
    int32_t* need[2] = {nullptr, nullptr};
    DetPrep prep[2] = {};
    cudaStream_t pstream = nullptr;
    cudaEvent_t ev_prep[2] = {nullptr, nullptr}, ev_det[2] = {nullptr, nullptr};
    size_t seq_cap = 0;

    cudaEvent_t ev_begin = nullptr, ev_end = nullptr;
    std::vector<cudaEvent_t> ev_w;   // 2 per timed worker launch
    std::vector<cudaEvent_t> ev_chunk;
    // overlapped async solves: monitor stream, x snapshots, slot events
    cudaStream_t mstream = nullptr;
    void* xs[2] = {nullptr, nullptr};
    void* xs_base[2] = {nullptr, nullptr};
    cudaEvent_t snap_ev[2] = {nullptr, nullptr}, mon_ev[2] = {nullptr, nullptr};
    asyrk_solve_stats stats{};
    // event timings of the last solve, read when the stats are asked for
    // (~90 elapsed-time queries at config 2 cost ~0.12 ms of host time that
    // the solve call itself would otherwise pay): worker launches timed
    mutable long long stats_timed = -1;  // -1: nothing pending
    long long spec_launch = -1;          // worker launch queued behind the stopping record (-1: none)
    // scheduled async solves: epochs of work of each worker launch (0: the launch
    // behind the stopping record) and its event pair (-1: not timed)
    std::vector<long long> lw_epochs;
    std::vector<long long> lw_pair;

    Layout layout() const {
        Layout L;
        L.rec = rec;
        L.row_info = uniform ? nullptr : row_info;
        L.stride16 = stride16;
        L.uniform_len = uniform_len;
        L.m = m;
        L.n = n;
        L.rec_bytes = rec_bytes;
        return L;
    }
    CscDev csc() const { return CscDev{grp_off, col_len, sell_row, sell_val, col_perm}; }
    CscDev rsell() const { return CscDev{rgrp_off, row_len, rsell_col, rsell_val}; }
    size_t xbytes() const { return precision == P_F32 ? 4 : 8; }
};

namespace {

// Streams and events of library-owned systems are recycled: the one-shot
// entry points build and drop a system per call, and creating / destroying
// three streams and a dozen events costs ~0.3 ms a call.
struct StreamKit {
    int dev = 0;
    cudaStream_t stream = nullptr, mstream = nullptr;
    cudaEvent_t ev_begin = nullptr, ev_end = nullptr;
    std::vector<cudaEvent_t> ev_w, ev_chunk;
    cudaEvent_t snap_ev[2] = {nullptr, nullptr}, mon_ev[2] = {nullptr, nullptr};
};
std::mutex g_kit_mu;
std::vector<StreamKit> g_kits;
constexpr size_t kMaxKits = 8;

bool kit_take(asyrk_system* s) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return false;
    std::lock_guard<std::mutex> lk(g_kit_mu);
    for (size_t i = 0; i < g_kits.size(); ++i)
        if (g_kits[i].dev == dev) {
            StreamKit k = std::move(g_kits[i]);
            g_kits.erase(g_kits.begin() + (long)i);
            s->stream = k.stream;
            s->mstream = k.mstream;
            s->ev_begin = k.ev_begin;
            s->ev_end = k.ev_end;
            s->ev_w = std::move(k.ev_w);
            s->ev_chunk = std::move(k.ev_chunk);
            for (int q = 0; q < 2; ++q) {
                s->snap_ev[q] = k.snap_ev[q];
                s->mon_ev[q] = k.mon_ev[q];
            }
            return true;
        }
    return false;
}

// after the streams are idle: park them for the next library-owned system
bool kit_put(asyrk_system* s) {
    int dev = 0;
    if (!s->own_stream || !s->stream || cudaGetDevice(&dev) != cudaSuccess) return false;
    std::lock_guard<std::mutex> lk(g_kit_mu);
    if (g_kits.size() >= kMaxKits) return false;
    StreamKit k;
    k.dev = dev;
    k.stream = s->stream;
    k.mstream = s->mstream;
    k.ev_begin = s->ev_begin;
    k.ev_end = s->ev_end;
    k.ev_w = std::move(s->ev_w);
    k.ev_chunk = std::move(s->ev_chunk);
    for (int q = 0; q < 2; ++q) {
        k.snap_ev[q] = s->snap_ev[q];
        k.mon_ev[q] = s->mon_ev[q];
    }
    g_kits.push_back(std::move(k));
    return true;
}

// The build (aux) stream and the pinned scalar of create are recycled the
// same way: a stream creation and a cudaHostAlloc / cudaFreeHost pair per
// one-shot call cost ~0.2 ms of host time.
std::vector<std::pair<int, cudaStream_t>> g_aux_streams;
// pinned scratch per system: [0, 64) small reads; then the solve's DevState and
// its records, copied behind the last kernel so the host's final read is one
// stream synchronization (PinLayout)
constexpr size_t kPinBytes = 64u << 10;
std::vector<void*> g_scalars;

cudaStream_t aux_stream_take() {
    int dev = 0;
    if (cudaGetDevice(&dev) == cudaSuccess) {
        std::lock_guard<std::mutex> lk(g_kit_mu);
        for (size_t i = 0; i < g_aux_streams.size(); ++i)
            if (g_aux_streams[i].first == dev) {
                cudaStream_t a = g_aux_streams[i].second;
                g_aux_streams.erase(g_aux_streams.begin() + (long)i);
                return a;
            }
    }
    cudaStream_t a = nullptr;
    CK(cudaStreamCreateWithFlags(&a, cudaStreamNonBlocking));
    return a;
}

void aux_stream_put(cudaStream_t a) {
    if (!a) return;
    cudaStreamSynchronize(a);
    int dev = 0;
    if (cudaGetDevice(&dev) == cudaSuccess) {
        std::lock_guard<std::mutex> lk(g_kit_mu);
        if (g_aux_streams.size() < kMaxKits) {
            g_aux_streams.emplace_back(dev, a);
            return;
        }
    }
    cudaStreamDestroy(a);
}

void* scalar_take() {
    {
        std::lock_guard<std::mutex> lk(g_kit_mu);
        if (!g_scalars.empty()) {
            void* p = g_scalars.back();
            g_scalars.pop_back();
            return p;
        }
    }
    void* p = nullptr;
    CK(cudaHostAlloc(&p, kPinBytes, cudaHostAllocPortable));
    return p;
}

void scalar_put(void* p) {
    if (!p) return;
    std::lock_guard<std::mutex> lk(g_kit_mu);
    if (g_scalars.size() < 4 * kMaxKits) {
        g_scalars.push_back(p);
        return;
    }
    cudaFreeHost(p);
}

void destroy_det_streams(asyrk_system* s) {
    if (s->pstream) {
        cudaStreamSynchronize(s->pstream);
        cudaStreamDestroy(s->pstream);
        s->pstream = nullptr;
    }
    for (int h = 0; h < 2; ++h) {
        if (s->ev_prep[h]) cudaEventDestroy(s->ev_prep[h]);
        if (s->ev_det[h]) cudaEventDestroy(s->ev_det[h]);
        s->ev_prep[h] = s->ev_det[h] = nullptr;
    }
}

void free_all(asyrk_system* s) {
    // on the system's device (the caller may have another one current), so the
    // frees and the pooled streams / events land on the right device
    struct DeviceGuard {
        int prev = -1;
        explicit DeviceGuard(int d) {
            if (cudaGetDevice(&prev) == cudaSuccess && prev != d) cudaSetDevice(d);
            else prev = -1;
        }
        ~DeviceGuard() {
            if (prev >= 0) cudaSetDevice(prev);
        }
    } on_device(s->dev);
    if (s->bstream) {
        aux_stream_put(s->bstream);  // synchronizes it
        s->bstream = nullptr;
    }
    if (s->ev_mon_ready) {
        cudaEventDestroy(s->ev_mon_ready);
        s->ev_mon_ready = nullptr;
    }
    cudaStream_t fs = s->stream;
    auto F = [fs](void* p) { pool_free(p, fs); };
    F(s->rec);
    F(s->row_info);
    F(s->row_norm);
    F(s->grp_off);
    F(s->col_len);
    F(s->col_perm);
    F(s->sell_row);
    F(s->sell_val);
    F(s->rgrp_off);
    F(s->row_len);
    F(s->rsell_col);
    F(s->rsell_val);
    F(s->b);
    F(s->col_ptr);
    F(s->csc_row);
    F(s->csc_val);
    F(s->alias);
    F(s->x_base ? s->x_base : s->x);
    F(s->xd);
    F(s->shadow);
    F(s->x0d);
    F(s->xstar);
    F(s->r_base ? s->r_base : s->r);
    F(s->g);
    F(s->part);
    F(s->recs);
    F(s->st);
    F(s->incr);
    F(s->audit_part);
    F(s->scratch);
    for (int h = 0; h < 2; ++h) {
        F(s->need[h]);
        F(s->prep[h].keys);
        F(s->prep[h].vals);
        F(s->prep[h].keys_s);
        F(s->prep[h].vals_s);
        F(s->prep[h].start);
        F(s->prep[h].temp);
        F(s->prep[h].ev_val);
        F(s->prep[h].ev_b);
        F(s->prep[h].ev_nn);
        F(s->prep[h].ev_rcp);
    }
    flag_release(s->host_flag);
    mirror_release(s->mirror);
    mirror_release(s->mirror0);
    s->mirror0 = nullptr;
    s->mirror = nullptr;
    for (int k = 0; k <= kLookahead; ++k) {
        F(s->seq_dev[k]);
        F(s->pick_dev[k]);
        F(s->flat_dev[k]);
        if (s->flat_host[k]) cudaFreeHost(s->flat_host[k]);
        if (s->seq_host[k]) cudaFreeHost(s->seq_host[k]);
        if (s->pick_host[k]) cudaFreeHost(s->pick_host[k]);
    }
    for (int q = 0; q < 2; ++q) F(s->xs_base[q] ? s->xs_base[q] : s->xs[q]);
    if (s->mstream) cudaStreamSynchronize(s->mstream);
    if (s->stream) cudaStreamSynchronize(s->stream);  // pool frees are stream-ordered
    scalar_put(s->host_scalar);  // after the streams: no copy into it can still be in flight
    s->host_scalar = nullptr;
    destroy_det_streams(s);
    if (kit_put(s)) return;
    if (s->ev_begin) cudaEventDestroy(s->ev_begin);
    if (s->ev_end) cudaEventDestroy(s->ev_end);
    for (auto e : s->ev_w) cudaEventDestroy(e);
    for (auto e : s->ev_chunk) cudaEventDestroy(e);
    for (int q = 0; q < 2; ++q) {
        if (s->snap_ev[q]) cudaEventDestroy(s->snap_ev[q]);
        if (s->mon_ev[q]) cudaEventDestroy(s->mon_ev[q]);
    }
    if (s->mstream) cudaStreamDestroy(s->mstream);
    if (s->own_stream && s->stream) cudaStreamDestroy(s->stream);
}

// randomly gathered arrays start on a 2 MB page boundary (x, r, the x
// snapshots): an array straddling a page measured 2-3% slower at config 2
void* dalloc_page_aligned(size_t bytes, void** base) {
    constexpr size_t kPage = 2u << 20;
    unsigned char* b = dalloc<unsigned char>(bytes + kPage);
    *base = b;
    return reinterpret_cast<void*>(((uintptr_t)b + kPage - 1) / kPage * kPage);
}

asyrk_status check_view(const asyrk_csr_view* A) {
    if (!A || !A->row_ptr || !A->col_idx || !A->values || !A->row_norm)
        return fail(ASYRK_E_InvalidArgument, "csr view has null arrays");
    if (A->m < 1 || A->n < 1) return fail(ASYRK_E_InvalidArgument, "matrix dimensions must be positive");
    if (A->row_ptr[0] != 0 || A->row_ptr[A->m] != A->nnz)
        return fail(ASYRK_E_DimensionMismatch, "row_ptr does not span nnz");
    if (A->m >= (int64_t)INT32_MAX || A->n >= (int64_t)INT32_MAX || A->nnz >= (int64_t)INT32_MAX)
        return fail(ASYRK_E_TooLarge, "m, n and nnz must each be < 2^31 on the device layout");
    return ASYRK_OK;
}

// Bind the per-solve buffers that depend on cap (records) lazily.
void ensure_records(asyrk_system* s, long long cap) {
    if (cap <= s->rec_cap) return;
    AllocStream as(s->stream);
    CK(cudaGetLastError());
    CK(pool_free(s->recs, s->stream));
    s->recs = dalloc<DevRecord>((size_t)cap);
    s->rec_cap = cap;
}

void ensure_seq(asyrk_system* s, size_t count) {
    if (count <= s->seq_cap) return;
    AllocStream as(s->stream);
    for (int k = 0; k <= kLookahead; ++k) {
        pool_free(s->seq_dev[k], s->stream);
        pool_free(s->pick_dev[k], s->stream);
        pool_free(s->flat_dev[k], s->stream);
        if (s->seq_host[k]) cudaFreeHost(s->seq_host[k]);
        if (s->pick_host[k]) cudaFreeHost(s->pick_host[k]);
        if (s->flat_host[k]) cudaFreeHost(s->flat_host[k]);
        s->seq_dev[k] = dalloc<int32_t>(count);
        s->pick_dev[k] = dalloc<int32_t>(count);
        s->flat_dev[k] = dalloc<long long>(count + 1);
        CK(cudaHostAlloc((void**)&s->seq_host[k], count * 4, cudaHostAllocDefault));
        CK(cudaHostAlloc((void**)&s->pick_host[k], count * 4, cudaHostAllocDefault));
        CK(cudaHostAlloc((void**)&s->flat_host[k], (count + 1) * 8, cudaHostAllocDefault));
    }
    // dataflow prepass buffers: one (event, nonzero) pair per entry
    const size_t pairs = count * (size_t)s->max_len;
    for (int h = 0; h < 2; ++h) {
        DetPrep& P = s->prep[h];
        for (void* p : {(void*)s->need[h], (void*)P.keys, (void*)P.vals, (void*)P.keys_s, (void*)P.vals_s,
                        (void*)P.start, P.temp, (void*)P.ev_val, (void*)P.ev_b, (void*)P.ev_nn, (void*)P.ev_rcp})
            pool_free(p, s->stream);
        s->need[h] = dalloc<int32_t>(pairs);
        P.ev_val = dalloc<double>(pairs);
        P.ev_b = dalloc<double>(count);
        P.ev_nn = dalloc<double>(count);
        P.ev_rcp = dalloc<double>(count);
        P.keys = dalloc<int32_t>(pairs);
        P.vals = dalloc<int32_t>(pairs);
        P.keys_s = dalloc<int32_t>(pairs);
        P.vals_s = dalloc<int32_t>(pairs);
        P.start = dalloc<int32_t>((size_t)s->n);
        P.temp_bytes = det_prepare_temp_bytes((long long)pairs);
        P.temp = dalloc<unsigned char>(P.temp_bytes);
    }
    s->seq_cap = count;
}

// Events are created on demand: `timed` pairs for the worker launches of the
// coming solve (capped at kTimedLaunches), plus the chunk ring.
void ensure_events(asyrk_system* s, long long timed = 0) {
    if (!s->ev_begin) {
        CK(cudaEventCreate(&s->ev_begin));
        CK(cudaEventCreate(&s->ev_end));
        s->ev_chunk.resize(kLookahead + 1);
        for (auto& e : s->ev_chunk) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    const size_t want = (size_t)(2 * std::min<long long>(timed, kTimedLaunches));
    while (s->ev_w.size() < want) {
        cudaEvent_t e;
        CK(cudaEventCreate(&e));
        s->ev_w.push_back(e);
    }
}

void ensure_alias_dev(asyrk_system* s) {
    if (s->alias) return;
    AllocStream as(s->stream);
    if (!s->h_alias) {
        std::vector<double> w(s->h_norm.size());
        for (size_t i = 0; i < w.size(); ++i) w[i] = s->h_norm[i] * s->h_norm[i];
        s->h_alias = std::make_unique<HostAlias>();
        if (!s->h_alias->build(w)) throw CudaFail{fail(ASYRK_E_InvalidArgument, "alias weights invalid")};
    }
    std::vector<AliasEntry> t(s->h_alias->prob.size());
    for (size_t i = 0; i < t.size(); ++i) t[i] = AliasEntry{(float)s->h_alias->prob[i], s->h_alias->alias[i]};
    s->alias = dalloc<AliasEntry>(t.size());
    CK(cudaMemcpyAsync(s->alias, t.data(), t.size() * sizeof(AliasEntry), cudaMemcpyHostToDevice, s->stream));
    CK(cudaStreamSynchronize(s->stream));
}

// sub-allocations of one block: add() every array, allocate off bytes, then assign
struct Carve {
    size_t off = 0;
    std::vector<std::pair<void**, size_t>> parts;
    template <class T>
    void add(T*& p, size_t count) {
        parts.emplace_back(reinterpret_cast<void**>(&p), off);
        off += (count * sizeof(T) + 255) / 256 * 256;
    }
};

asyrk_status create_impl(const asyrk_csr_view* A, const double* b, int32_t precision, void* stream,
                         asyrk_system** out, bool keep_csc = false) {
    asyrk_status v = check_view(A);
    if (v) return v;
    if (precision < 0 || precision > 2) return fail(ASYRK_E_InvalidArgument, "unknown precision");
    auto s = std::make_unique<asyrk_system>();
    CK(cudaGetDevice(&s->dev));
    s->m = A->m;
    s->n = A->n;
    s->nnz = A->nnz;
    s->precision = precision;
    s->normalized = A->normalized != 0;
    if (stream) {
        s->stream = static_cast<cudaStream_t>(stream);
    } else {
        if (!kit_take(s.get())) CK(cudaStreamCreateWithFlags(&s->stream, cudaStreamNonBlocking));
        s->own_stream = true;
    }
    AllocStream alloc_on(s->stream);
    s->host_scalar = scalar_take();
    // ASYRK_PROFILE_CREATE=1: synchronized phase times on stderr (diagnostics)
    static const bool prof = env_flag("ASYRK_PROFILE_CREATE");
    auto t_prev = std::chrono::steady_clock::now();
    auto phase = [&](const char* what) {
        if (!prof) return;
        cudaStreamSynchronize(s->stream);
        const auto t = std::chrono::steady_clock::now();
        fprintf(stderr, "[create] %-14s %8.3f ms\n", what, std::chrono::duration<double, std::milli>(t - t_prev).count());
        t_prev = t;
    };
    const int vbytes = precision == P_F64 ? 8 : 4;
    cudaStream_t st = s->stream;
    // Overlapped build: the host scan of row lengths runs on a thread, and the
    // column sort (CSC / SELL-columns, needs only row_ptr + col_idx) runs on an
    // aux stream while the values are still being staged (runtime.h Stager).
    {
        // x starts on a 2 MB page boundary: the workers' random gathers and reds
        // cover x uniformly, and an x straddling a page boundary measured 2-3%
        // slower at config 2 (ASYRK_X_ALIGN / ASYRK_X_OFFSET: placement experiments)
        static const long long xa = getenv("ASYRK_X_ALIGN") ? atoll(getenv("ASYRK_X_ALIGN")) : (2ll << 20);
        static const long long xo = getenv("ASYRK_X_OFFSET") ? atoll(getenv("ASYRK_X_OFFSET")) : 0;
        if (xa > 0) {
            unsigned char* base = dalloc<unsigned char>((size_t)A->n * s->xbytes() + (size_t)xa + (size_t)xo);
            const uintptr_t u = ((uintptr_t)base + (uintptr_t)xa - 1) / (uintptr_t)xa * (uintptr_t)xa + (uintptr_t)xo;
            s->x_base = base;
            s->x = reinterpret_cast<void*>(u);
        } else {
            s->x = dalloc<unsigned char>((size_t)A->n * s->xbytes());
        }
    }
    s->xd = dalloc<double>((size_t)A->n);
    s->x0d = dalloc<double>((size_t)A->n);
    s->r = static_cast<double*>(dalloc_page_aligned((size_t)A->m * 8, &s->r_base));
    s->g = dalloc<double>((size_t)A->n);
    s->part = dalloc<double>((size_t)monitor_row_blocks(A->m) + 2 * (size_t)monitor_col_blocks(A->n) + 8);
    s->st = dalloc<DevState>(1);
    s->incr = dalloc<unsigned long long>(1);
    s->scratch = dalloc<double>(4096);
    const long long groups = (A->n + 31) / 32;
    const long long rgroups = (A->m + 31) / 32;
    const size_t tb = std::max(csc_sort_temp_bytes(A->nnz), sigma_sort_temp_bytes(A->n));
    const size_t stb = scan_temp_bytes(groups + 1);
    const size_t rstb = scan_temp_bytes(rgroups + 1);
    // the build's scratch: one pool allocation carved into its arrays (a pool
    // call per array measured ~6 us each on the one-shot path)
    Carve cv;
    long long *d_rp = nullptr, *grp_size = nullptr, *rgrp_size = nullptr;
    int32_t *d_col = nullptr, *keys = nullptr, *idx = nullptr, *keys_s = nullptr, *idx_s = nullptr, *row_id = nullptr;
    int32_t *len_tmp = nullptr, *len_sorted = nullptr, *iota_tmp = nullptr;
    double *d_val = nullptr, *d_b = nullptr;
    unsigned char *temp = nullptr, *stemp = nullptr, *rstemp = nullptr;
    cv.add(d_rp, (size_t)A->m + 1);
    cv.add(d_col, (size_t)A->nnz);
    cv.add(d_val, (size_t)A->nnz);
    cv.add(d_b, (size_t)A->m);
    cv.add(keys, (size_t)A->nnz);
    cv.add(idx, (size_t)A->nnz);
    cv.add(keys_s, (size_t)A->nnz);
    cv.add(idx_s, (size_t)A->nnz);
    cv.add(row_id, (size_t)A->nnz);
    cv.add(temp, tb);
    cv.add(len_tmp, (size_t)A->n);
    cv.add(len_sorted, (size_t)A->n);
    cv.add(iota_tmp, (size_t)A->n);
    cv.add(grp_size, (size_t)groups + 1);
    cv.add(stemp, stb);
    cv.add(rgrp_size, (size_t)rgroups + 1);
    cv.add(rstemp, rstb);
    unsigned char* slab = dalloc<unsigned char>(cv.off);
    for (auto& pr : cv.parts) *pr.first = slab + pr.second;
    s->row_norm = dalloc<double>((size_t)A->m);
    // kept by fp64 / multi-RHS systems (plain CSC), so allocated on their own
    long long* col_ptr = dalloc<long long>((size_t)A->n + 1);
    int32_t* csc_row = dalloc<int32_t>((size_t)A->nnz);
    double* csc_val = dalloc<double>((size_t)A->nnz);
    s->col_len = dalloc<int32_t>((size_t)A->n);
    s->col_perm = dalloc<int32_t>((size_t)A->n);
    s->grp_off = dalloc<long long>((size_t)groups + 1);
    s->row_len = dalloc<int32_t>((size_t)A->m);
    s->rgrp_off = dalloc<long long>((size_t)rgroups + 1);
    s->b = dalloc<double>((size_t)A->m);
    phase("device allocs");
    // the build's scratch (col_ptr / csc_row / csc_val are nulled when the system keeps them)
    auto build_temps = [&] { return std::vector<void*>{slab, col_ptr, csc_row, csc_val}; };

    // host scan: row lengths, layout, row-SELL size (sell_len_kernel's 32 * max per group)
    struct Scan {
        int64_t zero_row = -1;
        uint32_t maxl = 0, minl = UINT32_MAX;
        bool too_large = false;
        size_t rec_bytes = 0;
        long long rsell_total = 0;
        std::vector<uint2> info;
    } sc;
    s->h_len.resize((size_t)A->m);
    std::future<void> scan_done = HelperThread::get().submit([&] {
        s->h_norm.assign(A->row_norm, A->row_norm + A->m);
        for (int64_t g = 0; g < rgroups && sc.zero_row < 0; ++g) {
            uint32_t gmax = 0;
            for (int64_t i = g * 32; i < std::min<int64_t>(A->m, g * 32 + 32); ++i) {
                const int64_t l = A->row_ptr[i + 1] - A->row_ptr[i];
                if (l <= 0) {
                    sc.zero_row = i;
                    break;
                }
                s->h_len[(size_t)i] = (int32_t)l;
                gmax = std::max<uint32_t>(gmax, (uint32_t)l);
                sc.minl = std::min<uint32_t>(sc.minl, (uint32_t)l);
            }
            sc.maxl = std::max(sc.maxl, gmax);
            sc.rsell_total += 32ll * gmax;
        }
        if (sc.zero_row >= 0) return;
        if (sc.maxl == sc.minl) {
            sc.rec_bytes = (size_t)A->m * rec_size16(sc.maxl, vbytes) * 16u;
            return;
        }
        sc.info.resize((size_t)A->m);
        uint64_t off = 0;
        for (int64_t i = 0; i < A->m; ++i) {
            sc.info[(size_t)i] = make_uint2((uint32_t)off, (uint32_t)s->h_len[(size_t)i]);
            off += rec_size16((uint32_t)s->h_len[(size_t)i], vbytes);
            if (off >= (1ull << 32)) {
                sc.too_large = true;
                return;
            }
        }
        sc.rec_bytes = (size_t)off * 16u;
    });
    struct Join {
        std::future<void>& f;
        ~Join() {
            if (f.valid()) f.wait();  // the scan reads A and writes s: never outlive them
        }
    } join_scan{scan_done};
    phase("scan thread");

    cudaStream_t aux = nullptr;
    cudaEvent_t ev_cols = nullptr, ev_sorted = nullptr;
    struct AuxGuard {
        cudaStream_t& a;
        cudaEvent_t &e1, &e2;
        ~AuxGuard() {
            if (a) aux_stream_put(a);
            if (e1) cudaEventDestroy(e1);
            if (e2) cudaEventDestroy(e2);
        }
    } aux_guard{aux, ev_cols, ev_sorted};
    aux = aux_stream_take();
    CK(cudaEventCreateWithFlags(&ev_cols, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&ev_sorted, cudaEventDisableTiming));

    phase("alloc+aux");
    // pinned, multithreaded staging; int64 columns cross PCIe as int32 (runtime.h)
    Stager& up = Stager::get();
    up.upload(d_rp, A->row_ptr, ((size_t)A->m + 1) * 8, st);
    up.upload_narrow(d_col, A->col_idx, (size_t)A->nnz, st);
    CK(cudaEventRecord(ev_cols, st));
    // aux: CSC order (stable by column => rows ascending within each column),
    // column histogram, SELL-32 column groups
    CK(cudaStreamWaitEvent(aux, ev_cols, 0));
    launch_iota_cols(d_col, A->nnz, keys, idx, aux);
    launch_row_ids(d_rp, A->m, row_id, aux);
    int end_bit = 1;
    while ((1ll << end_bit) < A->n) ++end_bit;
    csc_sort(temp, tb, keys, keys_s, idx, idx_s, A->nnz, end_bit, aux);
    launch_col_hist(keys_s, A->nnz, A->n, col_ptr, aux);
    CK(cudaMemsetAsync(grp_size, 0, ((size_t)groups + 1) * 8, aux));
    launch_sigma_sort(col_ptr, A->n, temp, tb, len_tmp, len_sorted, iota_tmp, s->col_perm, aux);
    launch_sell_len(col_ptr, A->n, s->col_len, grp_size, aux, s->col_perm);
    exclusive_scan(stemp, stb, grp_size, s->grp_off, groups + 1, aux);
    CK(cudaMemcpyAsync(s->host_scalar, s->grp_off + groups, 8, cudaMemcpyDeviceToHost, aux));  // column-SELL size
    CK(cudaGetLastError());
    CK(cudaEventRecord(ev_sorted, aux));
    // st: the values, norms and b keep streaming meanwhile
    up.upload(d_val, A->values, (size_t)A->nnz * 8, st);
    up.upload(s->row_norm, A->row_norm, (size_t)A->m * 8, st);
    if (b) up.upload(d_b, b, (size_t)A->m * 8, st);
    else CK(cudaMemsetAsync(d_b, 0, (size_t)A->m * 8, st));
    CK(cudaMemcpyAsync(s->b, d_b, (size_t)A->m * 8, cudaMemcpyDeviceToDevice, st));
    if (prof) {
        fprintf(stderr, "[create] upload issued   %8.3f ms\n",
                std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_prev).count());
    }
    phase("upload");

    scan_done.get();
    if (sc.zero_row >= 0 || sc.too_large) {
        cudaStreamSynchronize(aux);  // aux still reads buffers free_all releases
        cudaStreamSynchronize(st);
        for (void* p : build_temps()) pool_free(p, st);
    }
    if (sc.zero_row >= 0) {
        free_all(s.get());
        return fail(ASYRK_E_ZeroRow, "row " + std::to_string(sc.zero_row) + " has no nonzeros");
    }
    if (sc.too_large) {
        free_all(s.get());
        return fail(ASYRK_E_TooLarge, "row records exceed 64 GiB");
    }
    s->max_len = sc.maxl;
    s->uniform = sc.maxl == sc.minl;
    if (s->uniform) {
        s->uniform_len = sc.maxl;
        s->stride16 = rec_size16(sc.maxl, vbytes);
    }
    s->rec = dalloc<unsigned char>(sc.rec_bytes);
    s->rec_bytes = sc.rec_bytes;
    if (!s->uniform) {
        s->row_info = dalloc<uint2>(sc.info.size());
        CK(cudaMemcpyAsync(s->row_info, sc.info.data(), sc.info.size() * sizeof(uint2), cudaMemcpyHostToDevice, st));
    }
    launch_pack_records(d_rp, d_col, d_val, s->row_norm, d_b, A->m, s->uniform ? nullptr : s->row_info, s->stride16,
                        s->uniform_len, precision, s->rec, st);
    CK(cudaGetLastError());
    phase("pack");
    // The monitor's structures are built on the aux (build) stream after the
    // uploads; create returns without waiting for them — the workers need only
    // the packed records, and every monitor consumer waits on ev_mon_ready.
    CK(cudaEventSynchronize(ev_sorted));  // the column sort ran during the value upload
    long long sell_total = 0;
    std::memcpy(&sell_total, s->host_scalar, 8);
    // outputs allocated on the solve stream as before (their placement is what
    // the resident solves measured), then handed to the build stream
    s->rsell_col = dalloc<int32_t>((size_t)sc.rsell_total);
    s->rsell_val = dalloc<unsigned char>((size_t)sc.rsell_total * vbytes);
    s->sell_row = dalloc<int32_t>((size_t)sell_total);
    s->sell_val = dalloc<unsigned char>((size_t)sell_total * vbytes);
    CK(cudaEventRecord(ev_cols, st));  // values, norms, b uploaded and packed; outputs allocated
    CK(cudaStreamWaitEvent(aux, ev_cols, 0));
    {
        // SELL-32 rows for the monitor's coalesced thread-per-row pass (r = Ax - b);
        // keys still holds the CSR-order columns (the sort wrote keys_s)
        CK(cudaMemsetAsync(s->rsell_col, 0, (size_t)std::max<long long>(sc.rsell_total, 1) * 4, aux));
        CK(cudaMemsetAsync(rgrp_size, 0, ((size_t)rgroups + 1) * 8, aux));
        launch_sell_len(d_rp, A->m, s->row_len, rgrp_size, aux);
        exclusive_scan(rstemp, rstb, rgrp_size, s->rgrp_off, rgroups + 1, aux);
        launch_sell_scatter(d_rp, keys, d_val, s->row_len, s->rgrp_off, A->m, precision, s->rsell_col, s->rsell_val,
                            aux);
        phase("sell rows");
        // SELL-32 columns for the monitor's coalesced thread-per-column pass
        launch_gather_csc(idx_s, row_id, d_val, A->nnz, P_F64, csc_row, csc_val, aux);
        CK(cudaMemsetAsync(s->sell_row, 0, (size_t)std::max<long long>(sell_total, 1) * 4, aux));
        launch_sell_scatter(col_ptr, csc_row, csc_val, s->col_len, s->grp_off, A->n, precision, s->sell_row,
                            s->sell_val, aux, s->col_perm);
        phase("sell cols");
        CK(cudaGetLastError());
        if (keep_csc || precision == P_F64) {  // plain CSC: multi-RHS monitor, simulator's serial column walks
            s->col_ptr = col_ptr;
            s->csc_row = csc_row;
            s->csc_val = csc_val;
            col_ptr = nullptr;
            csc_row = nullptr;
            csc_val = nullptr;
        }
        for (void* p : build_temps()) pool_free(p, aux);
        CK(cudaEventCreateWithFlags(&s->ev_mon_ready, cudaEventDisableTiming));
        CK(cudaEventRecord(s->ev_mon_ready, aux));
    }
    s->bstream = aux;  // the build stream now belongs to the system
    aux = nullptr;
    phase("free temps");
    // solve buffers
    s->host_flag = flag_acquire(&s->host_flag_dev);
    if (!s->host_flag) throw CudaFail{fail(ASYRK_E_TooLarge, "no pinned stop flag available")};
    s->mirror = mirror_acquire(&s->mirror_dev);
    s->mirror0 = mirror_acquire(&s->mirror0_dev);
    if (!s->mirror || !s->mirror0) throw CudaFail{fail(ASYRK_E_TooLarge, "no pinned record mirror available")};
    ensure_records(s.get(), 256);
    ensure_events(s.get());
    phase("solve buffers");
    CK(cudaStreamSynchronize(st));
    *out = s.release();
    return ASYRK_OK;
}

// host_scalar layout: [0, 64) scratch, then DevState, then records
constexpr size_t kPinStateOff = 64;
constexpr size_t kPinRecOff = (kPinStateOff + sizeof(DevState) + 63) / 64 * 64;
constexpr long long kPinRecCap = (long long)((kPinBytes - kPinRecOff) / sizeof(DevRecord));
inline DevState* pin_state(asyrk_system* s) {
    return reinterpret_cast<DevState*>(static_cast<unsigned char*>(s->host_scalar) + kPinStateOff);
}
inline DevRecord* pin_records(asyrk_system* s) {
    return reinterpret_cast<DevRecord*>(static_cast<unsigned char*>(s->host_scalar) + kPinRecOff);
}
// enqueue the final state and the first `recs` records into the pinned scratch (stream order)
void pin_final(asyrk_system* s, long long recs, cudaStream_t st) {
    recs = std::min<long long>(std::min<long long>(recs, kPinRecCap), s->rec_cap);
    CK(cudaMemcpyAsync(pin_state(s), s->st, sizeof(DevState), cudaMemcpyDeviceToHost, st));
    if (recs > 0) CK(cudaMemcpyAsync(pin_records(s), s->recs, (size_t)recs * sizeof(DevRecord), cudaMemcpyDeviceToHost, st));
    s->pin_recs = recs;
}

void write_trace(asyrk_system* s, const DevState& hs, asyrk_trace_out* trace, int precision) {
    if (!trace) return;
    const long long k = std::min<long long>(hs.nrec, s->rec_cap);
    std::vector<DevRecord> recs((size_t)k);
    if (k && k <= s->pin_recs)
        std::memcpy(recs.data(), pin_records(s), (size_t)k * sizeof(DevRecord));
    else if (k)
        CK(cudaMemcpy(recs.data(), s->recs, (size_t)k * sizeof(DevRecord), cudaMemcpyDeviceToHost));
    trace->count = hs.nrec;
    const long long w = std::min<long long>(k, trace->cap);
    for (long long i = 0; i < w; ++i) {
        const DevRecord& r = recs[(size_t)i];
        if (trace->epoch_index) trace->epoch_index[i] = r.epoch;
        if (trace->r_sq) trace->r_sq[i] = r.r_sq;
        if (trace->grad_sq) trace->grad_sq[i] = r.grad_sq;
        if (trace->dist_sq) trace->dist_sq[i] = r.dist_sq;
        if (trace->wall_seconds) trace->wall_seconds[i] = 1e-9 * (double)r.t_ns;
        if (trace->updates_applied) trace->updates_applied[i] = r.updates;
    }
    if (trace->final_x) {
        launch_x_export(s->x, s->xd, s->n, precision, s->stream);
        const size_t xb = (size_t)s->n * 8;
        if (xb >= (8u << 20)) {
            Stager::get().download(trace->final_x, s->xd, xb, s->stream);  // large: through the pinned slots
        } else {  // small (config 2: 0.8 MB): one pageable copy is quicker than the bounce
            CK(cudaMemcpyAsync(trace->final_x, s->xd, xb, cudaMemcpyDeviceToHost, s->stream));
            CK(cudaStreamSynchronize(s->stream));
        }
    }
}

// order `stream` after the monitor structures of create (bstream)
void mon_wait(asyrk_system* s, cudaStream_t stream) {
    if (!s->ev_mon_ready) return;
    if (cudaEventQuery(s->ev_mon_ready) == cudaSuccess) {  // built: no cross-stream edge from now on
        cudaEventDestroy(s->ev_mon_ready);
        s->ev_mon_ready = nullptr;
        return;
    }
    CK(cudaStreamWaitEvent(stream, s->ev_mon_ready, 0));
}

MonitorArgs monitor_args(asyrk_system* s, bool exact, int advance, bool with_xstar) {
    MonitorArgs a{};
    a.L = s->layout();
    a.csc = s->csc();
    a.x = s->x;
    a.x_star = with_xstar ? s->xstar : nullptr;
    a.r = s->r;
    a.g = s->g;
    a.part = s->part;
    a.rec = s->recs;
    a.rec_cap = s->rec_cap;
    a.st = s->st;
    a.host_flag = s->host_flag_dev;
    a.exact = exact ? 1 : 0;
    a.advance = advance;
    a.m_rows = s->m;
    a.rows = s->rsell();
    a.b = s->b;
    a.slot = -1;
    a.set_epoch = -1;
    a.mirror = nullptr;
    a.col_out = nullptr;
    a.x_alt = nullptr;
    a.force = 0;
    return a;
}

struct SolveSpec {
    int64_t threads;
    double gamma;
    int64_t epochs;
    double target;
    bool full_row;
    int sampling;           // ASYRK_WITH_REPLACEMENT / SLICE / NORM_PROP
    uint64_t seed;
    int64_t interval;
    const double* x_star;
    int precision;
    bool det;               // deterministic sequence path
    int det_mode;           // SeqGen mode
    bool every_boundary;    // async: record every boundary (run config record_every_boundary)
    bool reassoc;           // deterministic: det_reassociate (tolerance mode)
};

// ASYRK_TIMELINE=path (diagnostics): timing events around the first chunks'
// worker / snapshot / monitor launches on both streams, written as CSV
// (kind, chunk, start_us, end_us relative to the solve's first event).
struct Timeline {
    struct Mark {
        const char* kind;
        long long k;
        cudaEvent_t a, b;
    };
    std::vector<Mark> marks;
    bool on = false;
    static constexpr long long kChunks = 24;
    Mark* begin(const char* kind, long long k, cudaStream_t st) {
        if (!on || k >= kChunks) return nullptr;
        Mark m{kind, k, nullptr, nullptr};
        cudaEventCreate(&m.a);
        cudaEventCreate(&m.b);
        cudaEventRecord(m.a, st);
        marks.push_back(m);
        return &marks.back();
    }
    void end(Mark* m, cudaStream_t st) {
        if (m) cudaEventRecord(m->b, st);
    }
    void dump(const char* path, cudaEvent_t base) {
        if (!on) return;
        if (FILE* f = fopen(path, "w")) {
            fprintf(f, "kind,chunk,start_us,end_us\n");
            for (auto& m : marks) {
                float a = 0.f, b = 0.f;
                cudaEventElapsedTime(&a, base, m.a);
                cudaEventElapsedTime(&b, base, m.b);
                fprintf(f, "%s,%lld,%.2f,%.2f\n", m.kind, m.k, 1e3 * a, 1e3 * b);
            }
            fclose(f);
        }
        for (auto& m : marks) {
            cudaEventDestroy(m.a);
            cudaEventDestroy(m.b);
        }
    }
};

// Stats, trace and instrument report of a finished solve (the stream is idle).
// worker time of a solve from its sampled launches (timed_launch): the mean
// sampled duration times the launches that did work; spec = index of the
// launch queued behind the stopping record (it exits at once; -1: none), which
// is neither a sample nor work
double sampled_worker_ms(asyrk_system* s, long long timed, long long launches, long long spec) {
    std::vector<double> w((size_t)std::max<long long>(timed, 0));
    for (long long t = 0; t < timed; ++t) {
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, s->ev_w[(size_t)(2 * t)], s->ev_w[(size_t)(2 * t + 1)]));
        w[(size_t)t] = ms;
    }
    long long used = timed, work = launches;
    if (spec >= 0 && spec < launches) {
        --work;
        if (timed_launch(spec) && used > 0) --used;  // it is the last launch, so the last sample
    }
    double sum = 0.0;
    for (long long t = 0; t < used; ++t) sum += w[(size_t)t];
    return used > 0 ? sum * (double)work / (double)used : 0.0;
}

// the last async solve's event timings (its events stay untouched until the next solve)
void resolve_stats(asyrk_system* s) {
    if (s->stats_timed < 0) return;
    const long long timed = s->stats_timed;
    s->stats_timed = -1;
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, s->ev_begin, s->ev_end));
    s->stats.solve_ms = ms;
    if (!s->lw_epochs.empty()) {  // scheduled solve: timed launches' ms per epoch x all epochs of work
        double t_ms = 0.0, t_ep = 0.0, all_ep = 0.0;
        for (size_t i = 0; i < s->lw_epochs.size(); ++i) {
            all_ep += (double)s->lw_epochs[i];
            const long long p = s->lw_pair[i];
            if (p < 0 || s->lw_epochs[i] <= 0) continue;
            float lm = 0.f;
            CK(cudaEventElapsedTime(&lm, s->ev_w[(size_t)(2 * p)], s->ev_w[(size_t)(2 * p + 1)]));
            t_ms += lm;
            t_ep += (double)s->lw_epochs[i];
        }
        s->stats.worker_ms = t_ep > 0.0 ? t_ms * all_ep / t_ep : 0.0;
        return;
    }
    s->stats.worker_ms = sampled_worker_ms(s, timed, s->stats.worker_launches, s->spec_launch);
}

// ASYRK_PROFILE_SOLVE=1: host timestamps of the async solve's phases on stderr (diagnostics)
struct SolveClock {
    bool on = env_flag("ASYRK_PROFILE_SOLVE");
    std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
    void mark(const char* what) const {
        if (on)
            fprintf(stderr, "[solve] %-18s %8.1f us\n", what,
                    std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count());
    }
};
thread_local SolveClock* g_solve_clock = nullptr;
inline void solve_mark(const char* what) {
    if (g_solve_clock) g_solve_clock->mark(what);
}

asyrk_status finish_solve(asyrk_system* s, const SolveSpec& sp, int prec, long long timed, long long launches,
                          const std::vector<unsigned long long>& chunk_incr, asyrk_trace_out* trace,
                          asyrk_instrument_out* instr) {
    cudaStream_t st = s->stream;
    DevState hs;
    if (s->pin_recs >= 0)  // copied behind the last kernel (pin_final), the stream is idle
        std::memcpy(&hs, pin_state(s), sizeof(DevState));
    else
        CK(cudaMemcpy(&hs, s->st, sizeof(DevState), cudaMemcpyDeviceToHost));
    solve_mark("state read");
    s->stats_timed = timed;  // solve_ms / worker_ms: resolve_stats, on demand
    s->stats.kernel_launches = launches;
    s->stats.projections = hs.updates;
    solve_mark("stats");
    if (hs.status == ASYRK_E_NonFinite) return fail(ASYRK_E_NonFinite, "iterate became non-finite");

    write_trace(s, hs, trace, prec);
    solve_mark("trace");
    if (instr) {
        instr->row_updates = hs.updates;
        unsigned long long inc = 0;
        if (sp.det) {
            const long long done = sp.interval > 0 ? (hs.epoch + sp.interval - 1) / sp.interval : 0;
            for (long long c = 0; c < done && c < (long long)chunk_incr.size(); ++c) inc += chunk_incr[(size_t)c];
            launch_instrument_check(s->x, s->x0d, s->shadow, s->n, prec, s->scratch, st);
        } else {
            launch_audit_check(s->x, s->x0d, s->n, prec, s->audit_part,
                               reinterpret_cast<const unsigned long long*>(s->audit_part + sp.threads * kAuditK),
                               sp.threads, s->scratch + 16, s->scratch, s->incr, st);
            CK(cudaMemcpyAsync(&inc, s->incr, sizeof(inc), cudaMemcpyDeviceToHost, st));
        }
        double mx = 0.0;
        CK(cudaMemcpyAsync(&mx, s->scratch, sizeof(double), cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        instr->increments = (int64_t)inc;
        instr->max_abs_error = mx;
        instr->tolerance = 1e-9 * (double)std::max<int64_t>(instr->increments, 1);
        instr->consistent = mx <= instr->tolerance ? 1 : 0;
    }
    return ASYRK_OK;
}

// The async driver with the host-driven monitor schedule (schedule.h). One
// stream: worker launches of the unmonitored boundaries back to back; at a
// scheduled boundary the residual monitor (rows + columns/finalize) runs
// in-stream and writes the record + stop decision; the next boundary's worker
// launch is enqueued right behind it (it runs only if the record did not stop
// the solve: st->go) while the host waits for the record's event and reads
// the mirror to place the next evaluation. So the host's read overlaps a
// worker epoch, no epoch runs past the stopping boundary, and the returned
// iterate is the one whose record met the target (parallel.cpp:415-426: the
// final record is that of the final iterate).
asyrk_status run_scheduled(asyrk_system* s, const SolveSpec& sp, WorkerArgs& wa, int E, int prec, long long max_chunks,
                           long long launches, asyrk_trace_out* trace, asyrk_instrument_out* instr) {
    cudaStream_t st = s->stream;
    const bool xs = sp.x_star != nullptr;
    auto epoch_of = [&](long long b) { return std::min<long long>(b * sp.interval, sp.epochs); };
    cudaEvent_t ev_rec = s->ev_chunk[0];
    std::memset(s->mirror, 0, sizeof(HostMirror));
    // Boundary 0 is x0, which the workers do not read back: its record is taken
    // from the fp64 copy x0d on the monitor stream while the first workers run
    // (x is fp64 for P_F64 / P_F32X64 systems), and only the monitors of later
    // boundaries (on the worker stream) wait for it — and for the monitor
    // structures create builds on its build stream. fp32 systems record x0 in-stream.
    const bool side0 = prec != P_F32 && max_chunks > 0 && !instr;  // (an audit must see every increment)
    MonitorSchedule sch;
    sch.reset(sp.target, sp.every_boundary);
    // boundary whose record (main mirror) the host has not read yet (-1: none);
    // with side0, record 0 (its own mirror) is read together with record 1: the
    // evaluation of boundary 1 is unconditional, so it and the next worker are
    // enqueued at once instead of after the host has seen record 0
    long long pending = side0 ? -1 : 0;
    bool r0_pending = side0;
    long long stop_b = -1;   // boundary whose record stopped the solve (-1: the budget ran out)
    long long next_mon = 1;  // next boundary to evaluate
    long long timed = 0;
    // Worker launches: boundary b -> b_end in one launch. Between the boundary
    // after an evaluation and the next scheduled evaluation no record is taken,
    // so those chunks run as ONE launch (each warp walks its slice once per
    // epoch without waiting for the others at the unrecorded boundaries, as the
    // reference's workers do, parallel.cpp:306-373; the launch still ends
    // exactly at the next evaluated boundary): config 2 runs ~10 launches for 42
    // epochs instead of 43, without the drain and ramp of every epoch. The
    // launch behind an evaluation is one chunk (the gap after it is not known
    // until the host has read the record). Fused launches and a sample of the
    // one-chunk ones (timed_launch) are timed with event pairs; worker_ms =
    // their ms per epoch x all epochs of work (resolve_stats).
    s->lw_epochs.clear();
    s->lw_pair.clear();
    // Fused only while the records stream within about twice the L2 per epoch:
    // configs 2 and 4 (77 / 130 MB of records) gain 7% / 3%, config 3 (832 MB
    // streamed from HBM every epoch) loses 1-2% (profiles/r02_ab_fuse_*.json,
    // r02_fuse_cfg34.txt) — its epochs are 1.35 ms, so the per-launch drain is
    // negligible there and warps drifting apart across unrecorded boundaries
    // scatter the record stream
    static const bool no_fuse_env = env_flag("ASYRK_NO_FUSE");
    static const size_t l2_bytes = [] {
        int dev = 0, l2 = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, dev);
        return (size_t)(l2 > 0 ? l2 : 126 << 20);
    }();
    const bool no_fuse = no_fuse_env || s->rec_bytes > 2 * l2_bytes;
    auto enqueue_worker = [&](long long b, long long b_end) {
        wa.epoch0 = epoch_of(b);
        wa.span0 = epoch_of(b_end) - wa.epoch0;
        const bool time_it = timed < kTimedLaunches && (b_end - b > 1 || timed_launch(b));
        if (time_it) CK(cudaEventRecord(s->ev_w[(size_t)(2 * timed)], st));
        launch_worker(wa, prec, E, st);
        s->lw_epochs.push_back(wa.span0);
        s->lw_pair.push_back(time_it ? timed : -1);
        if (time_it) {
            CK(cudaEventRecord(s->ev_w[(size_t)(2 * timed + 1)], st));
            ++timed;
        }
        ++launches;
        s->stats.worker_launches++;
    };
    if (side0) {
        if (!s->mstream) {
            int lo = 0, hi = 0;
            CK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
            CK(cudaStreamCreateWithPriority(&s->mstream, cudaStreamNonBlocking, hi));
            for (int q = 0; q < 2; ++q) {
                CK(cudaEventCreateWithFlags(&s->snap_ev[q], cudaEventDisableTiming));
                CK(cudaEventCreateWithFlags(&s->mon_ev[q], cudaEventDisableTiming));
            }
        }
        launch_state_init(s->st, sp.epochs, sp.interval, sp.target, st, /*go=*/1);
        CK(cudaEventRecord(s->snap_ev[0], st));
        enqueue_worker(0, 1);  // first: the GPU starts on the workers while the host enqueues record 0
        CK(cudaStreamWaitEvent(s->mstream, s->snap_ev[0], 0));
        mon_wait(s, s->mstream);
        std::memset(s->mirror0, 0, sizeof(HostMirror));
        MonitorArgs m0 = monitor_args(s, false, 0, xs);
        m0.x = s->x0d;
        m0.mirror = s->mirror0_dev;
        launch_monitor(m0, prec, s->mstream);
        CK(cudaEventRecord(s->mon_ev[0], s->mstream));
    } else {
        mon_wait(s, st);
        MonitorArgs m0 = monitor_args(s, false, 0, xs);
        m0.mirror = s->mirror_dev;
        launch_monitor(m0, prec, st);
        CK(cudaEventRecord(ev_rec, st));
        if (max_chunks > 0) enqueue_worker(0, 1);
    }
    launches += side0 ? 3 : 2;
    s->stats.monitor_launches++;
    bool waited0 = !side0;  // the worker stream is ordered after record 0
    solve_mark("first worker");
    for (long long b = 0; b < max_chunks; ++b) {
        // here the worker of chunk b (b -> b + 1) is enqueued; read the pending
        // record while it runs, then place the next evaluation
        if (pending >= 0) {
            if (r0_pending) {  // record 0 first (long done: boundary 1's evaluation waited for it)
                CK(cudaEventSynchronize(s->mon_ev[0]));
                r0_pending = false;
                const volatile HostMirror* h0 = s->mirror0;
                if (h0->stop) {
                    // x0 met the target (or was non-finite) while the first workers
                    // already ran (their later launches and record 1 skip on the device's
                    // stop): the solve returns x0 (epoch 0, no updates)
                    CK(cudaStreamWaitEvent(st, s->mon_ev[0], 0));
                    launch_x_init(s->x0d, s->x, s->n, prec, st);
                    stop_b = 0;
                    for (auto& e : s->lw_epochs) e = 0;  // (their updates are discarded)
                    break;
                }
                sch.push(0, h0->r_sq);
            }
            CK(cudaEventSynchronize(ev_rec));
            solve_mark("record read");
            const volatile HostMirror* hm = s->mirror;
            if (hm->stop) {  // the enqueued worker sees go = 0 and exits
                stop_b = pending;
                if (!s->lw_epochs.empty()) s->lw_epochs.back() = 0;
                break;
            }
            next_mon = sch.push(pending, hm->r_sq);
            pending = -1;
        }
        const long long b1 = b + 1;
        if (b1 >= next_mon || b1 == max_chunks) {
            if (!waited0) {  // record 0 (monitor stream) precedes every later record
                CK(cudaStreamWaitEvent(st, s->mon_ev[0], 0));
                waited0 = true;
            }
            MonitorArgs ma = monitor_args(s, false, 1, xs);
            ma.set_epoch = epoch_of(b1);
            ma.mirror = s->mirror_dev;
            launch_monitor(ma, prec, st);
            launches += 2;
            s->stats.monitor_launches++;
            CK(cudaEventRecord(ev_rec, st));
            pending = b1;
        }
        if (b1 < max_chunks) {
            // no record unread: the next evaluation is known, run up to it in one launch
            const long long b_end = (pending < 0 && !no_fuse) ? std::min(std::max(next_mon, b1 + 1), max_chunks) : b1 + 1;
            enqueue_worker(b1, b_end);
            b = b_end - 2;  // (++b: the next iteration handles boundary b_end)
        }
        CK(cudaGetLastError());
    }
    if (r0_pending) {  // a one-chunk solve ends before the loop reads record 0
        CK(cudaEventSynchronize(s->mon_ev[0]));
        const volatile HostMirror* h0 = s->mirror0;
        if (h0->stop) {
            CK(cudaStreamWaitEvent(st, s->mon_ev[0], 0));
            launch_x_init(s->x0d, s->x, s->n, prec, st);
            stop_b = 0;
        }
    }
    solve_mark("loop done");
    CK(cudaEventRecord(s->ev_end, st));
    pin_final(s, s->stats.monitor_launches, st);  // every record of this solve came from one monitor launch
    CK(cudaStreamSynchronize(st));
    solve_mark("stream idle");
    CK(cudaGetLastError());
    const asyrk_status fs = finish_solve(s, sp, prec, timed, launches, {}, trace, instr);
    // the launch queued behind the stopping record exits at once (lw_epochs 0)
    s->spec_launch = stop_b > 0 ? s->stats.worker_launches - 1 : -1;
    return fs;
}

asyrk_status run_solve(asyrk_system* s, const double* x0, const SolveSpec& sp, asyrk_trace_out* trace,
                       asyrk_instrument_out* instr) {
    cudaStream_t st = s->stream;
    SolveClock clk;
    g_solve_clock = clk.on ? &clk : nullptr;
    struct ClockReset {
        ~ClockReset() { g_solve_clock = nullptr; }
    } clock_reset;
    AllocStream alloc_on(st);
    const int prec = sp.det ? P_F64 : sp.precision;
    if (sp.det && s->precision != P_F64)
        return fail(ASYRK_E_InvalidArgument, "the deterministic path needs an fp64 system");
    if (!sp.det && sp.precision != s->precision)
        return fail(ASYRK_E_InvalidArgument, "config precision differs from the system's");
    const long long max_chunks = sp.epochs > 0 ? (sp.epochs + sp.interval - 1) / sp.interval : 0;
    ensure_records(s, std::max<long long>(256, max_chunks + 2));
    ensure_events(s, max_chunks);
    s->stats = asyrk_solve_stats{};
    s->stats_timed = -1;
    s->spec_launch = -1;
    s->pin_recs = -1;
    s->lw_epochs.clear();  // (filled by the scheduled driver only)
    s->lw_pair.clear();

    // x0, x_star
    if (x0) CK(cudaMemcpyAsync(s->x0d, x0, (size_t)s->n * 8, cudaMemcpyHostToDevice, st));
    else CK(cudaMemsetAsync(s->x0d, 0, (size_t)s->n * 8, st));
    launch_x_init(s->x0d, s->x, s->n, prec, st);
    if (sp.x_star) {
        if (!s->xstar) s->xstar = dalloc<double>((size_t)s->n);
        CK(cudaMemcpyAsync(s->xstar, sp.x_star, (size_t)s->n * 8, cudaMemcpyHostToDevice, st));
    }
    if (instr) {
        if (sp.det) {  // the reference's per-component shadow (bitwise audit report)
            if (!s->shadow) s->shadow = dalloc<unsigned char>((size_t)s->n * 8);
            CK(cudaMemsetAsync(s->shadow, 0, (size_t)s->n * 8, st));
        } else {  // the workers' per-warp signed checksums (layout.cuh kAuditK) and increment counts
            if (s->audit_cap < sp.threads) {
                pool_free(s->audit_part, st);
                s->audit_part = dalloc<double>((size_t)sp.threads * (kAuditK + 1));
                s->audit_cap = sp.threads;
            }
            CK(cudaMemsetAsync(s->audit_part, 0, (size_t)sp.threads * (kAuditK + 1) * sizeof(double), st));
        }
        CK(cudaMemsetAsync(s->incr, 0, sizeof(unsigned long long), st));
    }
    *s->host_flag = 0;

    solve_mark("setup");
    CK(cudaEventRecord(s->ev_begin, st));
    launch_state_init(s->st, sp.epochs, sp.interval, sp.target, st);
    long long launches = 1;
    const int mon_kernels = sp.det ? 3 : 2;  // rows + columns (+ exact finalize); fast finalize is fused

    // worker setup
    WorkerArgs wa{};
    DetArgs da{};
    int E = 0;
    std::unique_ptr<SeqGen> gen;
    std::vector<unsigned long long> chunk_incr;
    if (sp.det) {
        const bool picks = !sp.full_row;
        if (sp.det_mode == 1 && !s->h_alias) {
            std::vector<double> w(s->h_norm.size());
            for (size_t i = 0; i < w.size(); ++i) w[i] = s->h_norm[i] * s->h_norm[i];
            s->h_alias = std::make_unique<HostAlias>();
            if (!s->h_alias->build(w)) {
                s->h_alias.reset();
                return fail(ASYRK_E_InvalidArgument, "alias weights invalid");
            }
        }
        gen = std::make_unique<SeqGen>(sp.seed, sp.det_mode, s->m, &s->h_len, s->h_alias.get(), picks);
        ensure_seq(s, (size_t)(std::min<int64_t>(sp.interval, std::max<int64_t>(sp.epochs, 1)) * s->m));
        da.L = s->layout();
        da.row_norm = s->row_norm;
        da.x = static_cast<double*>(s->x);
        da.shadow = instr ? static_cast<double*>(s->shadow) : nullptr;
        da.st = s->st;
        da.gamma = sp.gamma;
        da.full_row = sp.full_row ? 1 : 0;
        da.x_in_smem = (det_fits_smem(s->n) && s->max_len <= 128) ? 1 : 0;
        // waiting warps spin: any polling back-off costs more than the issue slots
        // it frees (config 1, profiles/r02_det_forward_grid.txt: bitwise 21.0 ms
        // spinning vs 21.3 at 16 ns; tolerance mode 12.15 vs 12.6 — ASYRK_DET_POLL_NS)
        static const int poll_env = getenv("ASYRK_DET_POLL_NS") ? atoi(getenv("ASYRK_DET_POLL_NS")) : -1;
        da.poll_ns = poll_env >= 0 ? poll_env : 0;
        da.max_len = s->max_len;
        da.reassoc = sp.reassoc ? 1 : 0;
        if (!s->pstream) {
            CK(cudaStreamCreateWithFlags(&s->pstream, cudaStreamNonBlocking));
            for (int h = 0; h < 2; ++h) {
                CK(cudaEventCreateWithFlags(&s->ev_prep[h], cudaEventDisableTiming));
                CK(cudaEventCreateWithFlags(&s->ev_det[h], cudaEventDisableTiming));
            }
        }
        // the pstream work of this solve follows everything queued on st before it
        CK(cudaEventRecord(s->ev_det[0], st));
        CK(cudaStreamWaitEvent(s->pstream, s->ev_det[0], 0));
        s->stats.warps = 1;
        s->stats.resident_warps = 1;
    } else {
        if (sp.sampling == ASYRK_NORM_PROPORTIONAL) ensure_alias_dev(s);
        E = worker_elems_per_lane(s->max_len);
        wa.L = s->layout();
        wa.x = s->x;
        wa.audit = instr ? s->audit_part : nullptr;
        wa.alias = s->alias;
        wa.st = s->st;
        wa.increments = instr ? reinterpret_cast<unsigned long long*>(s->audit_part + sp.threads * kAuditK) : nullptr;
        wa.W = sp.threads;
        wa.gamma = sp.gamma;
        const uint64_t k = splitmix64(sp.seed ^ 0xA5A5A5A5DEADBEEFull);
        wa.key0 = (uint32_t)k;
        wa.key1 = (uint32_t)(k >> 32);
        wa.sampling = sp.sampling == ASYRK_SLICE_SHUFFLE ? S_SLICE
                      : sp.sampling == ASYRK_NORM_PROPORTIONAL ? S_ALIAS
                                                                : S_UNIFORM;
        wa.full_row = sp.full_row ? 1 : 0;
        s->stats.warps = (int32_t)std::min<int64_t>(sp.threads, INT32_MAX);
        s->stats.resident_warps =
            (int32_t)std::min<int64_t>(sp.threads, worker_max_resident_warps(prec, E, wa.full_row));
    }
    CK(cudaGetLastError());

    // Async solves (default): the host-driven monitor schedule (schedule.h) —
    // the residual monitor runs in-stream at the boundaries the schedule picks,
    // the workers of the other boundaries run back to back. ASYRK_OVERLAP=1
    // selects the round-1 driver instead (a monitor of every boundary it can
    // take, on its own stream, overlapped with the next epochs).
    static const bool overlap_env = env_flag("ASYRK_OVERLAP");
    if (!sp.det && !overlap_env)
        return run_scheduled(s, sp, wa, E, prec, max_chunks, launches, trace, instr);
    static const bool no_overlap = env_flag("ASYRK_NO_OVERLAP");
    // (instrumented runs keep the in-stream monitor: restoring the stopping
    // snapshot would desynchronize x from the shadow increments)
    // The deterministic path overlaps too: its exact monitor (serial sums,
    // ~150 us per record at config 1) reads a boundary snapshot on the monitor
    // stream while the next chunk runs; a chunk that ran past the stopping
    // boundary is undone by restoring that snapshot, so records and the
    // returned iterate are the in-order ones (bit-identical either way).
    static const bool no_det_overlap = env_flag("ASYRK_NO_DET_OVERLAP");
    const bool overlap = !no_overlap && !instr && (!sp.det || !no_det_overlap);
    if (overlap && !s->mstream) {
        // highest priority: monitor blocks take SM slots ahead of queued worker blocks
        int lo = 0, hi = 0;
        CK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
        static const bool low_prio = env_flag("ASYRK_MON_LOWPRIO");
        CK(cudaStreamCreateWithPriority(&s->mstream, cudaStreamNonBlocking, low_prio ? lo : hi));
        for (int q = 0; q < 2; ++q) {
            CK(cudaEventCreateWithFlags(&s->snap_ev[q], cudaEventDisableTiming));
            CK(cudaEventCreateWithFlags(&s->mon_ev[q], cudaEventDisableTiming));
        }
    }
    if (overlap && !s->xs[0])  // (a recycled stream kit brings the stream and events, not the buffers)
        for (int q = 0; q < 2; ++q) s->xs[q] = dalloc_page_aligned((size_t)s->n * s->xbytes(), &s->xs_base[q]);
    // record_every_boundary (or ASYRK_EXACT_RECORDS=1): a record at every boundary
    // (the workers wait for the monitor); default: the monitor takes the latest
    // boundary it can, like the reference's coordinator, and the workers never wait
    static const bool exact_env = env_flag("ASYRK_EXACT_RECORDS");
    const bool exact_records = exact_env || sp.every_boundary || sp.det;  // deterministic: every boundary
    // boundary 0 (x0): the overlapped modes take it through the same snapshot ->
    // monitor-stream path as every later boundary, so the first workers start
    // at once; a stop decided there is undone like any other (restore). Only
    // the monitor's stream waits for create's build stream.
    mon_wait(s, overlap ? s->mstream : st);
    if (overlap) {
        MonitorArgs ma = monitor_args(s, sp.det, 0, sp.x_star != nullptr);
        if (exact_records) {
            launch_snapshot(s->st, s->x, s->xs[1], s->n, prec, 1, s->st, s->m, st, 0);
            ma.x = s->xs[1];
            ma.slot = 1;
        } else {
            launch_snapshot_dyn(s->st, s->x, s->xs[0], s->xs[1], s->n, prec, s->m, st, 0);
        }
        CK(cudaEventRecord(s->snap_ev[1], st));
        CK(cudaStreamWaitEvent(s->mstream, s->snap_ev[1], 0));
        if (!exact_records) {
            launch_claim(s->st, s->mstream);
            ma.x = s->xs[0];
            ma.x_alt = s->xs[1];
            ma.slot = kDynSlot;
        }
        launch_monitor(ma, prec, s->mstream);
        CK(cudaEventRecord(s->mon_ev[1], s->mstream));
        launches += 1 + mon_kernels + (exact_records ? 0 : 1);
    } else {
        launch_monitor(monitor_args(s, sp.det, 0, sp.x_star != nullptr), prec, st);
        launches += mon_kernels;
    }
    s->stats.monitor_launches++;
    static const char* tl_path = getenv("ASYRK_TIMELINE");
    Timeline tl;
    tl.marks.reserve(4 * Timeline::kChunks);
    tl.on = tl_path != nullptr;
    long long timed = 0;
    long long k = 0;
    for (; k < max_chunks; ++k) {
        if (k >= kLookahead) {
            CK(cudaEventSynchronize(s->ev_chunk[(size_t)(k % (kLookahead + 1))]));
            if (*reinterpret_cast<volatile int*>(s->host_flag)) break;
        }
        const bool time_it = timed < kTimedLaunches && (!sp.det || timed_launch(k) || max_chunks == 1);  // det: sampled (event pairs cost stream time)
        if (sp.det) {
            const long long e0 = k * sp.interval;
            const long long span = std::min<long long>(sp.interval, sp.epochs - e0);
            const int slot = (int)(k % (kLookahead + 1));
            // slot reuse: the copy of chunk k-(L+1) completed before chunk k-L's event (synced above)
            unsigned long long inc = 0;
            for (long long e = 0; e < span; ++e) {
                int32_t* sq = s->seq_host[slot] + e * s->m;
                int32_t* pk = s->pick_host[slot] + e * s->m;
                gen->epoch(sq, pk);
                if (instr) {
                    if (sp.full_row)
                        for (int64_t q = 0; q < s->m; ++q) inc += (unsigned long long)s->h_len[(size_t)sq[q]];
                    else
                        inc += (unsigned long long)s->m;
                }
            }
            chunk_incr.push_back(inc);
            const size_t cnt = (size_t)(span * s->m);
            // uploads and the dataflow prepass go on pstream, one chunk ahead of
            // the dataflow kernel on st; prepass set h was last read by chunk k-2
            const int h = (int)(k & 1);
            cudaStream_t ps = s->pstream;
            if (k >= 2) CK(cudaStreamWaitEvent(ps, s->ev_det[h], 0));
            CK(cudaMemcpyAsync(s->seq_dev[slot], s->seq_host[slot], cnt * 4, cudaMemcpyHostToDevice, ps));
            if (!sp.full_row)
                CK(cudaMemcpyAsync(s->pick_dev[slot], s->pick_host[slot], cnt * 4, cudaMemcpyHostToDevice, ps));
            da.seq = s->seq_dev[slot];
            da.picks = s->pick_dev[slot];
            da.count = (long long)cnt;
            da.need = s->need[h];
            da.ev_col = s->prep[h].keys;
            da.ev_val = s->prep[h].ev_val;
            da.ev_b = s->prep[h].ev_b;
            da.ev_nn = s->prep[h].ev_nn;
            da.ev_rcp = s->prep[h].ev_rcp;
            long long pairs = (long long)cnt * (long long)s->uniform_len;
            da.flat_off = nullptr;
            if (!s->uniform) {  // ragged rows: offsets of each event's (event, nonzero) pairs
                long long* fo = s->flat_host[slot];
                fo[0] = 0;
                for (size_t q = 0; q < cnt; ++q) fo[q + 1] = fo[q] + s->h_len[(size_t)s->seq_host[slot][q]];
                pairs = fo[cnt];
                CK(cudaMemcpyAsync(s->flat_dev[slot], fo, (cnt + 1) * 8, cudaMemcpyHostToDevice, ps));
                da.flat_off = s->flat_dev[slot];
            }
            if (da.x_in_smem) launch_det_prepare(da, s->prep[h], pairs, ps);
            CK(cudaEventRecord(s->ev_prep[h], ps));
            CK(cudaStreamWaitEvent(st, s->ev_prep[h], 0));
            if (time_it) CK(cudaEventRecord(s->ev_w[(size_t)(2 * timed)], st));
            static const char* dbg_path = getenv("ASYRK_DET_DEBUG");
            long long* dbg = nullptr;
            if (dbg_path && k == 0) {
                CK(cudaMalloc(&dbg, (size_t)cnt * 4 * 8));
                CK(cudaMemset(dbg, 0, (size_t)cnt * 4 * 8));
            }
            da.dbg = dbg;
            launch_det(da, 0, st);
            CK(cudaEventRecord(s->ev_det[h], st));
            if (dbg) {
                std::vector<long long> hd((size_t)cnt * 4);
                CK(cudaStreamSynchronize(st));
                CK(cudaMemcpy(hd.data(), dbg, hd.size() * 8, cudaMemcpyDeviceToHost));
                if (FILE* f = fopen(dbg_path, "wb")) {
                    fwrite(hd.data(), 8, hd.size(), f);
                    fclose(f);
                }
                cudaFree(dbg);
                da.dbg = nullptr;
            }
        } else {
            if (time_it) CK(cudaEventRecord(s->ev_w[(size_t)(2 * timed)], st));
            Timeline::Mark* tm = tl.begin("worker", k, st);
            launch_worker(wa, prec, E, st);
            tl.end(tm, st);
        }
        if (time_it) {
            CK(cudaEventRecord(s->ev_w[(size_t)(2 * timed + 1)], st));
            ++timed;
        }
        launches += 1;
        s->stats.worker_launches++;
        if (overlap) {
            // epoch-boundary snapshot on the worker stream; the residual monitor
            // of that snapshot runs on the monitor stream while the next epoch's
            // workers already go (the reference's coordinator thread,
            // parallel.cpp:388-408, without its torn reads)
            const int slot2 = (int)(k & 1);
            Timeline::Mark* ts = tl.begin("snapshot", k, st);
            if (exact_records) {  // every boundary recorded: slot reuse waits for monitor k-2
                if (k >= 1) CK(cudaStreamWaitEvent(st, s->mon_ev[slot2], 0));  // (k = 1: boundary 0's monitor)
                launch_snapshot(s->st, s->x, s->xs[slot2], s->n, prec, slot2, s->st, s->m, st);
            } else {  // latest boundary the monitor can take (parallel.cpp:388-399)
                launch_snapshot_dyn(s->st, s->x, s->xs[0], s->xs[1], s->n, prec, s->m, st);
            }
            tl.end(ts, st);
            CK(cudaEventRecord(s->snap_ev[slot2], st));
            CK(cudaStreamWaitEvent(s->mstream, s->snap_ev[slot2], 0));
            MonitorArgs ma = monitor_args(s, sp.det, 0, sp.x_star != nullptr);
            if (exact_records) {
                ma.x = s->xs[slot2];
                ma.slot = slot2;
            } else {
                launch_claim(s->st, s->mstream);
                ma.x = s->xs[0];
                ma.x_alt = s->xs[1];
                ma.slot = kDynSlot;
            }
            Timeline::Mark* tmo = tl.begin("monitor", k, s->mstream);
            launch_monitor(ma, prec, s->mstream);
            tl.end(tmo, s->mstream);
            CK(cudaEventRecord(s->mon_ev[slot2], s->mstream));
            launches += 1 + mon_kernels + (exact_records ? 0 : 1);  // snapshot (+ claim) + monitor
        } else {
            launch_monitor(monitor_args(s, sp.det, 1, sp.x_star != nullptr), prec, st);
            launches += mon_kernels;
        }
        s->stats.monitor_launches++;
        CK(cudaEventRecord(s->ev_chunk[(size_t)(k % (kLookahead + 1))], st));
        CK(cudaGetLastError());
    }
    if (overlap) {
        // join the monitor stream, then the exact record of the final iterate
        // (parallel.cpp:415-426: epoch = the epochs actually run)
        CK(cudaEventRecord(s->snap_ev[0], s->mstream));
        CK(cudaStreamWaitEvent(st, s->snap_ev[0], 0));
        // the epochs that ran past the stopping snapshot are discarded: the
        // solve returns the iterate whose residual met the target
        launch_restore(s->st, s->x, s->xs[0], s->xs[1], s->n, prec, st);
        launches += 1;
        // the final record of the returned iterate: when the run stopped at a
        // monitored snapshot, x was just restored from it and its record
        // (same bits, same monitor) is already the last one; otherwise (the
        // last boundaries went unmonitored, or NonFinite) record it now
        int stop_slot = -1;
        CK(cudaMemcpyAsync(s->host_scalar, &s->st->stop_slot, sizeof(int), cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        std::memcpy(&stop_slot, s->host_scalar, sizeof(int));
        static const bool always_final = env_flag("ASYRK_ALWAYS_FINAL_RECORD");
        if (stop_slot < 0 || always_final) {
            MonitorArgs fa = monitor_args(s, sp.det, 0, sp.x_star != nullptr);
            fa.force = 1;
            launch_monitor(fa, prec, st);
            launches += mon_kernels;
            s->stats.monitor_launches++;
        }
        CK(cudaGetLastError());
    }
    CK(cudaEventRecord(s->ev_end, st));
    CK(cudaStreamSynchronize(st));
    CK(cudaGetLastError());
    tl.dump(tl_path, s->ev_begin);
    return finish_solve(s, sp, prec, timed, launches, chunk_incr, trace, instr);
}

// validate_config, ref/src/parallel.cpp:56-80 (+ device extensions)
asyrk_status validate_run(const asyrk_system* s, const asyrk_run_config* c) {
    if (!c) return fail(ASYRK_E_InvalidArgument, "null config");
    const bool raw_ok = c->allow_unnormalized || c->sampling == ASYRK_NORM_PROPORTIONAL;
    if (!s->normalized && !raw_ok) return fail(ASYRK_E_NotNormalized, "solve_parallel requires normalized rows");
    if (c->threads < 1) return fail(ASYRK_E_InvalidArgument, "threads must be >= 1");
    if (!(c->gamma > 0.0)) return fail(ASYRK_E_InvalidGamma, "gamma must be positive");
    if (c->epochs < 0 || c->snapshot_interval < 1)
        return fail(ASYRK_E_InvalidArgument, "epochs must be >= 0 and snapshot_interval >= 1");
    if (c->sampling == ASYRK_SLICE_SHUFFLE && s->m < c->threads)
        return fail(ASYRK_E_InvalidArgument, "slice_shuffle needs at least one row per worker");
    if (c->sampling < 0 || c->sampling > 2) return fail(ASYRK_E_InvalidArgument, "unknown sampling");
    if (c->variant != ASYRK_FULL_ROW && c->variant != ASYRK_SINGLE_COMPONENT)
        return fail(ASYRK_E_InvalidArgument, "unknown variant");
    return ASYRK_OK;
}

asyrk_status system_solve_impl(asyrk_system* s, const double* x0, const asyrk_run_config* c,
                               asyrk_trace_out* trace, asyrk_instrument_out* instr) {
    asyrk_status v = validate_run(s, c);
    if (v) return v;
    SolveSpec sp{};
    sp.threads = c->threads;
    sp.gamma = c->gamma;
    sp.epochs = c->epochs;
    sp.target = c->target_r_sq;
    sp.full_row = c->variant == ASYRK_FULL_ROW;
    sp.sampling = c->sampling;
    sp.seed = c->seed;
    sp.interval = c->snapshot_interval;
    sp.x_star = c->x_star;
    sp.precision = c->precision;
    sp.det = c->threads == 1;
    sp.det_mode = c->sampling == ASYRK_SLICE_SHUFFLE ? 2 : (c->sampling == ASYRK_NORM_PROPORTIONAL ? 1 : 0);
    sp.every_boundary = c->record_every_boundary != 0;
    sp.reassoc = c->det_reassociate != 0;
    return run_solve(s, x0, sp, trace, instr);
}

asyrk_status system_rk_impl(asyrk_system* s, const double* x0, const asyrk_rk_config* c, asyrk_trace_out* trace) {
    if (!c) return fail(ASYRK_E_InvalidArgument, "null config");
    if (c->sampling == ASYRK_RK_UNIFORM && !s->normalized)
        return fail(ASYRK_E_NotNormalized,
                    "uniform row sampling is only unbiased on normalized rows; use norm_proportional or normalize first");
    if (c->max_epochs < 0) return fail(ASYRK_E_InvalidArgument, "max_epochs must be >= 0");
    if (c->sampling < 0 || c->sampling > 2) return fail(ASYRK_E_InvalidArgument, "unknown sampling");
    SolveSpec sp{};
    sp.threads = 1;
    sp.gamma = 1.0;
    sp.epochs = c->max_epochs;
    sp.target = c->target_r_sq;
    sp.full_row = true;
    sp.seed = c->seed;
    sp.interval = 1;
    sp.x_star = c->x_star;
    sp.precision = P_F64;
    sp.det = true;
    sp.det_mode = c->sampling == ASYRK_RK_UNIFORM ? 0 : (c->sampling == ASYRK_RK_NORM_PROPORTIONAL ? 1 : 2);
    sp.reassoc = c->det_reassociate != 0;
    return run_solve(s, x0, sp, trace, nullptr);
}

// Deterministic multi-RHS rk_solve (SURVEY.md §8c "config 5 per column"):
// k right-hand sides, ONE row sequence (the reference's make_stream(seed, 0)
// stream of rk_solve, kaczmarz.cpp:128-227), column j's iterate bit-identical
// to rk_solve(A, B[:, j], X0[:, j]) with the same seed. One dataflow CTA per
// column over the shared event prepass; a record per epoch whose r_sq /
// grad_sq / dist_sq are the per-column exact sums added in column order; the
// stop is global (sum r_sq <= target_r_sq or max_epochs).
asyrk_status rk_multi_impl(asyrk_system* s, const double* B, int64_t k, const double* X0, const asyrk_rk_config* c,
                           double* X_out, asyrk_trace_out* trace) {
    if (!c || !B || k < 1) return fail(ASYRK_E_InvalidArgument, "rk_solve_multi: need a config, B and k >= 1");
    if (s->precision != P_F64) return fail(ASYRK_E_InvalidArgument, "the deterministic path needs an fp64 system");
    if (c->sampling == ASYRK_RK_UNIFORM && !s->normalized)
        return fail(ASYRK_E_NotNormalized,
                    "uniform row sampling is only unbiased on normalized rows; use norm_proportional or normalize first");
    if (c->max_epochs < 0) return fail(ASYRK_E_InvalidArgument, "max_epochs must be >= 0");
    if (c->sampling < 0 || c->sampling > 2) return fail(ASYRK_E_InvalidArgument, "unknown sampling");
    if (k > 65535) return fail(ASYRK_E_TooLarge, "rk_solve_multi: at most 65535 right-hand sides");
    cudaStream_t st = s->stream;
    AllocStream alloc_on(st);
    mon_wait(s, st);
    const int64_t m = s->m, n = s->n;
    const int det_mode = c->sampling == ASYRK_RK_UNIFORM ? 0 : (c->sampling == ASYRK_RK_NORM_PROPORTIONAL ? 1 : 2);
    if (det_mode == 1 && !s->h_alias) {
        std::vector<double> w(s->h_norm.size());
        for (size_t i = 0; i < w.size(); ++i) w[i] = s->h_norm[i] * s->h_norm[i];
        s->h_alias = std::make_unique<HostAlias>();
        if (!s->h_alias->build(w)) {
            s->h_alias.reset();
            return fail(ASYRK_E_InvalidArgument, "alias weights invalid");
        }
    }
    // column-major device copies: column j of X / B / X* contiguous
    std::vector<double> tmp((size_t)(k * std::max(m, n)));
    auto to_cols = [&](const double* src, int64_t rows) {
        for (int64_t i = 0; i < rows; ++i)
            for (int64_t j = 0; j < k; ++j) tmp[(size_t)(j * rows + i)] = src[i * k + j];
    };
    double* Xc = dalloc<double>((size_t)(k * n));
    double* Bc = dalloc<double>((size_t)(k * m));
    double* Xs = c->x_star ? dalloc<double>((size_t)(k * n)) : nullptr;
    double* colres = dalloc<double>((size_t)(3 * k));
    double* evb = dalloc<double>((size_t)(k * m));  // the prepass's per-column b of each event
    struct Free {
        cudaStream_t st;
        std::vector<void*> p;
        ~Free() {
            for (void* q : p) pool_free(q, st);
        }
    } fr{st, {Xc, Bc, Xs, colres, evb}};
    to_cols(B, m);
    CK(cudaMemcpyAsync(Bc, tmp.data(), (size_t)(k * m) * 8, cudaMemcpyHostToDevice, st));
    CK(cudaStreamSynchronize(st));
    if (X0) {
        to_cols(X0, n);
        CK(cudaMemcpyAsync(Xc, tmp.data(), (size_t)(k * n) * 8, cudaMemcpyHostToDevice, st));
        CK(cudaStreamSynchronize(st));
    } else {
        CK(cudaMemsetAsync(Xc, 0, (size_t)(k * n) * 8, st));
    }
    if (Xs) {
        to_cols(c->x_star, n);
        CK(cudaMemcpyAsync(Xs, tmp.data(), (size_t)(k * n) * 8, cudaMemcpyHostToDevice, st));
        CK(cudaStreamSynchronize(st));
    }
    ensure_records(s, std::max<long long>(256, c->max_epochs + 2));
    ensure_events(s, 0);
    ensure_seq(s, (size_t)m);
    s->stats = asyrk_solve_stats{};
    s->stats_timed = -1;
    s->pin_recs = -1;
    std::memset(s->mirror, 0, sizeof(HostMirror));
    *s->host_flag = 0;
    CK(cudaEventRecord(s->ev_begin, st));
    launch_state_init(s->st, c->max_epochs, 1, c->target_r_sq, st);
    long long launches = 1;
    auto record = [&](long long epoch) {  // boundary `epoch` of every column -> one record
        for (int64_t j = 0; j < k; ++j) {
            MonitorArgs ma = monitor_args(s, true, 0, Xs != nullptr);
            ma.x = Xc + j * n;
            ma.b = Bc + j * m;
            ma.x_star = Xs ? Xs + j * n : nullptr;
            ma.col_out = colres + 3 * j;
            launch_monitor(ma, P_F64, st);
            launches += 3;
        }
        MonitorArgs mc = monitor_args(s, true, epoch > 0 ? 1 : 0, Xs != nullptr);
        mc.x_star = Xs;  // (records dist_sq when given)
        mc.set_epoch = epoch;
        mc.mirror = s->mirror_dev;
        launch_multi_commit(mc, colres, (int)k, st);
        launches += 1;
        s->stats.monitor_launches++;
        CK(cudaEventRecord(s->ev_chunk[0], st));
        CK(cudaEventSynchronize(s->ev_chunk[0]));
        return *const_cast<volatile int*>(&s->mirror->stop) != 0;
    };
    SeqGen gen(c->seed, det_mode, m, &s->h_len, s->h_alias.get(), false);
    DetArgs da{};
    da.L = s->layout();
    da.row_norm = s->row_norm;
    da.x = Xc;
    da.st = s->st;
    da.gamma = 1.0;
    da.full_row = 1;
    da.x_in_smem = (det_fits_smem(n) && s->max_len <= 128) ? 1 : 0;
    static const int poll_env = getenv("ASYRK_DET_POLL_NS") ? atoi(getenv("ASYRK_DET_POLL_NS")) : -1;
    da.poll_ns = poll_env >= 0 ? poll_env : 0;
    da.max_len = s->max_len;
    da.ncols = (int)k;
    da.b_cols = Bc;
    da.reassoc = c->det_reassociate ? 1 : 0;
    bool stop = record(0);
    for (long long e = 1; e <= c->max_epochs && !stop; ++e) {
        int32_t* sq = s->seq_host[0];
        gen.epoch(sq, s->pick_host[0]);
        CK(cudaMemcpyAsync(s->seq_dev[0], sq, (size_t)m * 4, cudaMemcpyHostToDevice, st));
        da.seq = s->seq_dev[0];
        da.picks = s->pick_dev[0];
        da.count = m;
        da.need = s->need[0];
        da.ev_col = s->prep[0].keys;
        da.ev_val = s->prep[0].ev_val;
        da.ev_b = evb;
        da.ev_nn = s->prep[0].ev_nn;
        da.ev_rcp = s->prep[0].ev_rcp;
        long long pairs = m * (long long)s->uniform_len;
        da.flat_off = nullptr;
        if (!s->uniform) {
            long long* fo = s->flat_host[0];
            fo[0] = 0;
            for (int64_t q = 0; q < m; ++q) fo[q + 1] = fo[q] + s->h_len[(size_t)sq[q]];
            pairs = fo[m];
            CK(cudaMemcpyAsync(s->flat_dev[0], fo, (size_t)(m + 1) * 8, cudaMemcpyHostToDevice, st));
            da.flat_off = s->flat_dev[0];
        }
        if (da.x_in_smem) launch_det_prepare(da, s->prep[0], pairs, st);
        launch_det(da, 0, st);
        launches += da.x_in_smem ? 5 : 1;
        s->stats.worker_launches++;
        stop = record(e);
        CK(cudaGetLastError());
    }
    CK(cudaEventRecord(s->ev_end, st));
    CK(cudaStreamSynchronize(st));
    DevState hs;
    CK(cudaMemcpy(&hs, s->st, sizeof(DevState), cudaMemcpyDeviceToHost));
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, s->ev_begin, s->ev_end));
    s->stats.solve_ms = ms;
    s->stats.kernel_launches = launches;
    s->stats.projections = hs.updates;
    s->stats.warps = (int32_t)std::min<int64_t>(k, INT32_MAX);
    if (hs.status == ASYRK_E_NonFinite) return fail(ASYRK_E_NonFinite, "iterate became non-finite");
    if (trace) {
        asyrk_trace_out t = *trace;
        t.final_x = nullptr;
        write_trace(s, hs, &t, P_F64);
        trace->count = t.count;
    }
    if (X_out) {
        CK(cudaMemcpy(tmp.data(), Xc, (size_t)(k * n) * 8, cudaMemcpyDeviceToHost));
        for (int64_t i = 0; i < n; ++i)
            for (int64_t j = 0; j < k; ++j) X_out[i * k + j] = tmp[(size_t)(j * n + i)];
    }
    return ASYRK_OK;
}

asyrk_status residuals_impl(asyrk_system* s, const double* x, double* r_sq, double* grad_sq) {
    cudaStream_t st = s->stream;
    mon_wait(s, st);
    CK(cudaMemcpyAsync(s->x0d, x, (size_t)s->n * 8, cudaMemcpyHostToDevice, st));
    launch_x_init(s->x0d, s->x, s->n, s->precision, st);
    launch_state_init(s->st, 0, 1, -1.0, st);
    MonitorArgs a = monitor_args(s, s->precision == P_F64, 0, false);
    a.host_flag = nullptr;
    launch_monitor(a, s->precision, st);
    CK(cudaGetLastError());
    DevRecord rec;
    DevState hs;
    CK(cudaMemcpyAsync(&rec, s->recs, sizeof(rec), cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(&hs, s->st, sizeof(hs), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (hs.status) {
        *r_sq = NAN;
        *grad_sq = NAN;
        return ASYRK_OK;
    }
    *r_sq = rec.r_sq;
    *grad_sq = rec.grad_sq;
    return ASYRK_OK;
}

// power_iteration_lambda_max, ref/src/stats.cpp:15-50
asyrk_status power_impl(asyrk_system* s, double tol, int64_t max_iters, double* lambda, int64_t* iters) {
    cudaStream_t st = s->stream;
    mon_wait(s, st);
    const int64_t n = s->n;
    RefStream gen(0x5ca1ab1eULL, 0);
    std::vector<double> v((size_t)n);
    for (auto& e : v) e = gen.normal();
    double ss = 0.0;
    for (double e : v) ss += e * e;
    double vn = std::sqrt(ss);
    if (vn == 0.0) v[0] = 1.0, vn = 1.0;
    for (auto& e : v) e /= vn;
    double* dv = s->xd;   // v
    double* dav = s->r;   // A v
    double* dw = s->g;    // A^T A v
    double* dots = s->scratch + 2048;
    CK(cudaMemcpyAsync(dv, v.data(), (size_t)n * 8, cudaMemcpyHostToDevice, st));
    double lam = 0.0;
    double h[2];
    for (int64_t it = 0; it < max_iters; ++it) {
        launch_spmv_rows(s->rsell(), s->precision, s->m, dv, dav, st);
        launch_spmv_cols(s->csc(), s->precision, n, dav, dw, st);
        launch_dot(dw, dw, n, s->scratch, dots, st);
        launch_dot(dv, dw, n, s->scratch + 1024, dots + 1, st);
        CK(cudaMemcpyAsync(h, dots, 16, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        const double wn = std::sqrt(h[0]);
        if (wn == 0.0) {
            *lambda = 0.0;
            if (iters) *iters = it + 1;
            return ASYRK_OK;
        }
        const double next = h[1];
        launch_power_update(dv, dw, dots, n, st);
        if (it > 0 && std::abs(next - lam) <= tol * std::max(1.0, std::abs(next))) {
            *lambda = next;
            if (iters) *iters = it + 1;
            CK(cudaStreamSynchronize(st));
            return ASYRK_OK;
        }
        lam = next;
    }
    return fail(ASYRK_E_PowerIterationDiverged,
                "power iteration did not converge within " + std::to_string(max_iters) + " iterations");
}

// compute_stats (ref/src/stats.cpp:52-130, exact_spectral = false), stats.cu
asyrk_status stats_impl(asyrk_system* s, double tol, int64_t max_iters, asyrk_stats_out* out) {
    if (!out) return fail(ASYRK_E_InvalidArgument, "null stats output");
    if (!s->normalized)
        return fail(ASYRK_E_NotNormalized,
                    "stats are defined for row-normalized matrices; call normalize_rows first");
    if (s->precision != P_F64) return fail(ASYRK_E_InvalidArgument, "compute_stats needs an fp64 system");
    cudaStream_t st = s->stream;
    mon_wait(s, st);
    AllocStream as(st);
    double* col_sq = dalloc<double>((size_t)s->n);
    double* col_norm = dalloc<double>((size_t)s->n);
    StatsDev* dres = dalloc<StatsDev>(1);
    unsigned char* scratch = nullptr;
    struct Free {
        std::vector<void*> p;
        cudaStream_t s;
        ~Free() {
            for (void* q : p) pool_free(q, s);
        }
    } fr{{col_sq, col_norm, dres}, st};
    StatsDev h{};
    h.zero_col = LLONG_MAX;
    CK(cudaMemcpyAsync(dres, &h, sizeof h, cudaMemcpyHostToDevice, st));
    launch_stats_cols(s->csc(), s->n, s->row_len, col_sq, col_norm, dres, st);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(&h, dres, sizeof h, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (h.zero_col != LLONG_MAX)
        return fail(ASYRK_E_ZeroColumn, "column " + std::to_string(h.zero_col) + " has no nonzeros");
    const size_t tbytes = (size_t)stats_table_cap(h.max_w, s->n) * 16;
    size_t scratch_bytes = 0;
    if (tbytes > (200u << 10)) {  // tables past shared memory live in global scratch (8 warps per block)
        scratch_bytes = std::max<size_t>(8 * tbytes, std::min<size_t>((size_t)1 << 30, 8 * tbytes * 148));
        scratch = dalloc<unsigned char>(scratch_bytes);
        fr.p.push_back(scratch);
    }
    launch_stats_rest(s->csc(), s->rsell(), s->m, s->n, col_sq, col_norm, h.max_w, scratch, scratch_bytes, dres, st);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(&h, dres, sizeof h, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    asyrk_stats_out o = *out;
    o.m = s->m;
    o.n = s->n;
    o.delta = (double)s->nnz / ((double)s->m * (double)s->n);
    o.mu = s->max_len;
    o.nu = h.nu;
    auto bits = [](unsigned long long b) {
        double d;
        std::memcpy(&d, &b, 8);
        return d;
    };
    o.alpha = bits(h.alpha_bits);
    o.frob_sq = h.frob_sq;
    o.l_max = bits(h.l_max_bits);
    o.l_res = bits(h.l_res_bits);
    if (o.theta)
        for (int64_t i = 0; i < s->m; ++i) o.theta[i] = s->h_len[(size_t)i];
    o.lambda_max = 0.0;
    o.power_iterations = 0;
    if (max_iters >= 0) {  // (< 0: the caller takes lambda_max from the dense spectrum)
        asyrk_status ps = power_impl(s, tol, max_iters, &o.lambda_max, &o.power_iterations);
        if (ps) return ps;
    }
    *out = o;
    return ASYRK_OK;
}

// ---- bounded-delay simulator (ref/src/delay_sim.cpp:71-270), delay.cu
asyrk_status sim_validate(const asyrk_system* s, const asyrk_sim_config* c) {
    if (!c) return fail(ASYRK_E_InvalidArgument, "null simulator config");
    if (!s->normalized) return fail(ASYRK_E_NotNormalized, "simulate requires normalized rows");
    if (s->precision != P_F64) return fail(ASYRK_E_InvalidArgument, "the simulator needs an fp64 system");
    if (c->gamma < 0.0) return fail(ASYRK_E_InvalidGamma, "gamma must be >= 0");
    if (c->iterations < 1) return fail(ASYRK_E_InvalidArgument, "need at least one iteration");
    if (c->tau < 0) return fail(ASYRK_E_InvalidArgument, "tau must be >= 0");
    if (c->probe_dist_sq && !c->dist_point)
        return fail(ASYRK_E_InvalidArgument, "probe_dist_sq needs a SolutionProjector");
    if (c->delay < 0 || c->delay > 2) return fail(ASYRK_E_InvalidArgument, "unknown delay model");
    if (c->variant < 0 || c->variant > 1) return fail(ASYRK_E_InvalidArgument, "unknown update variant");
    return ASYRK_OK;
}

SimArgs sim_args(asyrk_system* s, const asyrk_sim_config* c) {
    SimArgs a{};
    a.L = s->layout();
    a.R = s->rsell();
    a.C = s->csc();
    a.col_ptr = s->col_ptr;
    a.csc_row = s->csc_row;
    a.csc_val = s->csc_val;
    a.row_norm = s->row_norm;
    a.b = s->b;
    a.x0 = s->x0d;
    a.m = s->m;
    a.n = s->n;
    a.gamma = c->gamma;
    a.tau = c->tau;
    a.delay_kind = c->delay;
    a.variant = c->variant;
    a.iterations = c->iterations;
    a.seed0 = c->seed;
    return a;
}

void sim_upload_x0(asyrk_system* s, const double* x0) {
    if (x0)
        CK(cudaMemcpyAsync(s->x0d, x0, (size_t)s->n * 8, cudaMemcpyHostToDevice, s->stream));
    else
        CK(cudaMemsetAsync(s->x0d, 0, (size_t)s->n * 8, s->stream));
}

asyrk_status sim_impl(asyrk_system* s, const double* x0, const asyrk_sim_config* c, asyrk_sim_out* out) {
    if (asyrk_status v = sim_validate(s, c)) return v;
    if (!out) return fail(ASYRK_E_InvalidArgument, "null simulator output");
    cudaStream_t st = s->stream;
    mon_wait(s, st);
    AllocStream as(st);
    const long long m = s->m, n = s->n, K = c->iterations;
    const bool probing = c->probe_every > 0 && (c->probe_r_sq || c->probe_dist_sq);
    const long long nprobe_max = probing ? K / c->probe_every + 1 : 0;
    const long long rec_cap = K / m + 2;
    const long long ev_cap = std::min<long long>(c->max_events, K);
    const size_t wd = sim_work_doubles(m, n, c->tau);
    double* work = dalloc<double>(wd);
    double* probe = dalloc<double>((size_t)std::max<long long>(nprobe_max, 1));
    double* probe_d = dalloc<double>((size_t)std::max<long long>(nprobe_max, 1));
    double* xdist = c->dist_point ? dalloc<double>((size_t)n) : nullptr;
    DevRecord* rec = dalloc<DevRecord>((size_t)rec_cap);
    SimEventDev* ev = dalloc<SimEventDev>((size_t)std::max<long long>(ev_cap, 1));
    long long* cnt = dalloc<long long>(4);  // nrec, nev, nprobe, fail_updates
    int* status = dalloc<int>(1);
    struct Free {
        std::vector<void*> p;
        cudaStream_t s;
        ~Free() {
            for (void* q : p) pool_free(q, s);
        }
    } fr{{work, probe, probe_d, xdist, rec, ev, cnt, status}, st};
    sim_upload_x0(s, x0);
    if (xdist) CK(cudaMemcpyAsync(xdist, c->dist_point, (size_t)n * 8, cudaMemcpyHostToDevice, st));
    CK(cudaMemsetAsync(cnt, 0, 4 * 8, st));
    CK(cudaMemsetAsync(status, 0, 4, st));
    SimArgs a = sim_args(s, c);
    a.probe_every = c->probe_every;
    a.probe_r_sq = c->probe_r_sq;
    a.xdist = xdist;
    a.probe_d = c->probe_dist_sq ? probe_d : nullptr;
    a.max_events = ev_cap;
    a.runs = 1;
    a.work = work;
    a.work_stride = (long long)wd;
    a.probe = (probing && c->probe_r_sq) ? probe : nullptr;
    a.probe_stride = nprobe_max;
    a.rec = rec;
    a.rec_cap = rec_cap;
    a.nrec = cnt;
    a.nev = cnt + 1;
    a.nprobe = cnt + 2;
    a.ev = ev;
    a.status = status;
    a.fail_updates = cnt + 3;
    launch_sim(a, true, st);
    CK(cudaGetLastError());
    long long hc[4];
    int hst = 0;
    CK(cudaMemcpyAsync(hc, cnt, sizeof hc, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(&hst, status, 4, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (hst) return fail(ASYRK_E_NonFinite, "iterate became non-finite at iteration " + std::to_string(hc[3]));
    // trace records (one per epoch boundary + a trailing partial epoch)
    std::vector<DevRecord> recs((size_t)std::min(hc[0], rec_cap));
    if (!recs.empty()) CK(cudaMemcpy(recs.data(), rec, recs.size() * sizeof(DevRecord), cudaMemcpyDeviceToHost));
    asyrk_trace_out& tr = out->trace;
    tr.count = hc[0];
    for (long long k = 0; k < std::min<long long>((long long)recs.size(), tr.cap); ++k) {
        const DevRecord& r = recs[(size_t)k];
        if (tr.epoch_index) tr.epoch_index[k] = r.epoch;
        if (tr.r_sq) tr.r_sq[k] = r.r_sq;
        if (tr.grad_sq) tr.grad_sq[k] = r.grad_sq;
        if (tr.dist_sq) tr.dist_sq[k] = r.dist_sq;
        if (tr.wall_seconds) tr.wall_seconds[k] = 1e-9 * (double)r.t_ns;
        if (tr.updates_applied) tr.updates_applied[k] = r.updates;
    }
    if (tr.final_x) CK(cudaMemcpy(tr.final_x, work, (size_t)n * 8, cudaMemcpyDeviceToHost));
    // events
    out->ev_count = hc[1];
    const long long ne = std::min<long long>(hc[1], out->ev_cap);
    if (ne > 0) {
        std::vector<SimEventDev> e((size_t)ne);
        CK(cudaMemcpy(e.data(), ev, (size_t)ne * sizeof(SimEventDev), cudaMemcpyDeviceToHost));
        for (long long k = 0; k < ne; ++k) {
            if (out->ev_j) out->ev_j[k] = e[(size_t)k].j;
            if (out->ev_i) out->ev_i[k] = e[(size_t)k].i;
            if (out->ev_t) out->ev_t[k] = e[(size_t)k].t;
            if (out->ev_k) out->ev_k[k] = e[(size_t)k].k;
            if (out->ev_step) out->ev_step[k] = e[(size_t)k].step;
        }
    }
    // history: the last min(tau+1, K+1) iterates, oldest first (delay_sim.cpp:223-227)
    const long long ring_len = c->tau + 1;
    const long long kept = std::min(ring_len, K + 1);
    out->history_rows = kept;
    if (out->history) {
        const double* ring = c->tau == 0 ? work : work + n;
        long long row = 0;
        for (long long idx = K - kept + 1; idx <= K && row < out->history_cap; ++idx, ++row)
            CK(cudaMemcpy(out->history + row * n, ring + (idx % ring_len) * n, (size_t)n * 8,
                          cudaMemcpyDeviceToHost));
    }
    // probes at iterations 0, probe_every, 2 probe_every, ...
    out->probe_count = probing ? hc[2] : 0;
    const long long np = std::min<long long>(out->probe_count, out->probe_cap);
    if (np > 0) {
        if (out->probe_r_sq && c->probe_r_sq)
            CK(cudaMemcpy(out->probe_r_sq, probe, (size_t)np * 8, cudaMemcpyDeviceToHost));
        if (out->probe_dist_sq && c->probe_dist_sq)
            CK(cudaMemcpy(out->probe_dist_sq, probe_d, (size_t)np * 8, cudaMemcpyDeviceToHost));
        if (out->probe_iteration)
            for (long long k = 0; k < np; ++k) out->probe_iteration[k] = k * c->probe_every;
    }
    return ASYRK_OK;
}

asyrk_status mc_impl(asyrk_system* s, const double* x0, const asyrk_sim_config* c, int64_t runs, double* mean_r_sq,
                     double* ratios) {
    if (runs < 100) return fail(ASYRK_E_InsufficientData, "need >= 100 runs for stable ratio estimates");
    asyrk_sim_config cc = *c;  // monte_carlo_ratios probes every iteration (delay_sim.cpp:239-241)
    cc.probe_every = 1;
    cc.probe_r_sq = 1;
    cc.probe_dist_sq = 0;
    cc.max_events = 0;
    if (asyrk_status v = sim_validate(s, &cc)) return v;
    if (!mean_r_sq || (!ratios && cc.iterations > 0)) return fail(ASYRK_E_InvalidArgument, "null output");
    cudaStream_t st = s->stream;
    mon_wait(s, st);
    AllocStream as(st);
    const long long K = cc.iterations;
    const size_t wd = sim_work_doubles(s->m, s->n, cc.tau);
    if ((double)wd * (double)runs * 8.0 + (double)(K + 1) * (double)runs * 8.0 > 64e9)
        return fail(ASYRK_E_TooLarge, "Monte-Carlo working set exceeds 64 GB");
    double* work = dalloc<double>(wd * (size_t)runs);
    double* probe = dalloc<double>((size_t)(K + 1) * (size_t)runs);
    double* mean = dalloc<double>((size_t)K + 1);
    double* rat = dalloc<double>((size_t)std::max<long long>(K, 1));
    int* status = dalloc<int>((size_t)runs);
    long long* failu = dalloc<long long>((size_t)runs);
    struct Free {
        std::vector<void*> p;
        cudaStream_t s;
        ~Free() {
            for (void* q : p) pool_free(q, s);
        }
    } fr{{work, probe, mean, rat, status, failu}, st};
    sim_upload_x0(s, x0);
    CK(cudaMemsetAsync(status, 0, (size_t)runs * 4, st));
    SimArgs a = sim_args(s, &cc);
    a.probe_every = 1;
    a.probe_r_sq = 1;
    a.runs = runs;
    a.work = work;
    a.work_stride = (long long)wd;
    a.probe = probe;
    a.probe_stride = K + 1;
    a.status = status;
    a.fail_updates = failu;
    launch_sim(a, false, st);
    launch_sim_mean(probe, K + 1, runs, K, mean, rat, st);
    CK(cudaGetLastError());
    std::vector<int> hs((size_t)runs);
    CK(cudaMemcpyAsync(hs.data(), status, (size_t)runs * 4, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    for (int64_t r = 0; r < runs; ++r)
        if (hs[(size_t)r]) {  // the reference throws from the first failing run
            long long u = 0;
            CK(cudaMemcpy(&u, failu + r, 8, cudaMemcpyDeviceToHost));
            return fail(ASYRK_E_NonFinite, "iterate became non-finite at iteration " + std::to_string(u));
        }
    CK(cudaMemcpy(mean_r_sq, mean, (size_t)(K + 1) * 8, cudaMemcpyDeviceToHost));
    if (K > 0) CK(cudaMemcpy(ratios, rat, (size_t)K * 8, cudaMemcpyDeviceToHost));
    return ASYRK_OK;
}

struct SysGuard {
    asyrk_system* s = nullptr;
    ~SysGuard() {
        if (s) {
            free_all(s);
            delete s;
        }
    }
};

}  // namespace

extern "C" {

const char* asyrk_last_error(void) { return err_buf().c_str(); }
int asyrk_abi_version(void) { return ASYRK_ABI_VERSION; }

asyrk_status asyrk_set_device(int32_t device) {
    return guarded([&] {
        CK(cudaSetDevice(device));
        return ASYRK_OK;
    });
}

asyrk_status asyrk_system_create(const asyrk_csr_view* A, const double* b, int32_t precision, void* stream,
                                 asyrk_system** out) {
    return guarded([&] { return create_impl(A, b, precision, stream, out); });
}

asyrk_status asyrk_system_destroy(asyrk_system* sys) {
    if (!sys) return ASYRK_OK;
    cudaStreamSynchronize(sys->stream);
    free_all(sys);
    delete sys;
    return ASYRK_OK;
}

asyrk_status asyrk_system_solve(asyrk_system* sys, const double* x0, const asyrk_run_config* cfg,
                                asyrk_trace_out* trace, asyrk_instrument_out* instrument) {
    if (!sys) return fail(ASYRK_E_InvalidArgument, "null system");
    return guarded([&] { return system_solve_impl(sys, x0, cfg, trace, instrument); });
}

asyrk_status asyrk_system_rk_solve(asyrk_system* sys, const double* x0, const asyrk_rk_config* cfg,
                                   asyrk_trace_out* trace) {
    if (!sys) return fail(ASYRK_E_InvalidArgument, "null system");
    return guarded([&] { return system_rk_impl(sys, x0, cfg, trace); });
}

asyrk_status asyrk_system_residuals(asyrk_system* sys, const double* x, double* r_sq, double* grad_sq) {
    if (!sys) return fail(ASYRK_E_InvalidArgument, "null system");
    return guarded([&] { return residuals_impl(sys, x, r_sq, grad_sq); });
}

asyrk_status asyrk_system_power_iteration(asyrk_system* sys, double tol, int64_t max_iters, double* lambda_max,
                                          int64_t* iterations) {
    if (!sys) return fail(ASYRK_E_InvalidArgument, "null system");
    return guarded([&] { return power_impl(sys, tol, max_iters, lambda_max, iterations); });
}

asyrk_status asyrk_system_compute_stats(asyrk_system* sys, double tol, int64_t max_iters, asyrk_stats_out* out) {
    if (!sys) return fail(ASYRK_E_InvalidArgument, "null system");
    return guarded([&] { return stats_impl(sys, tol, max_iters, out); });
}

asyrk_status asyrk_compute_stats(const asyrk_csr_view* A, double tol, int64_t max_iters, asyrk_stats_out* out) {
    return guarded([&] {
        SysGuard g;
        asyrk_status s = create_impl(A, nullptr, P_F64, nullptr, &g.s);
        if (s) return s;
        return stats_impl(g.s, tol, max_iters, out);
    });
}

asyrk_status asyrk_system_simulate(asyrk_system* sys, const double* x0, const asyrk_sim_config* cfg,
                                   asyrk_sim_out* out) {
    if (!sys) return fail(ASYRK_E_InvalidArgument, "null system");
    return guarded([&] { return sim_impl(sys, x0, cfg, out); });
}

asyrk_status asyrk_system_monte_carlo_ratios(asyrk_system* sys, const double* x0, const asyrk_sim_config* cfg,
                                             int64_t runs, double* mean_r_sq, double* ratios) {
    if (!sys || !cfg) return fail(ASYRK_E_InvalidArgument, "null argument");
    return guarded([&] { return mc_impl(sys, x0, cfg, runs, mean_r_sq, ratios); });
}

asyrk_status asyrk_simulate(const asyrk_csr_view* A, const double* b, const double* x0, const asyrk_sim_config* cfg,
                            asyrk_sim_out* out) {
    return guarded([&] {
        SysGuard g;
        asyrk_status s = create_impl(A, b, P_F64, nullptr, &g.s);
        if (s) return s;
        return sim_impl(g.s, x0, cfg, out);
    });
}

asyrk_status asyrk_monte_carlo_ratios(const asyrk_csr_view* A, const double* b, const double* x0,
                                      const asyrk_sim_config* cfg, int64_t runs, double* mean_r_sq, double* ratios) {
    if (!cfg) return fail(ASYRK_E_InvalidArgument, "null simulator config");
    if (runs < 100) return fail(ASYRK_E_InsufficientData, "need >= 100 runs for stable ratio estimates");
    return guarded([&] {
        SysGuard g;
        asyrk_status s = create_impl(A, b, P_F64, nullptr, &g.s);
        if (s) return s;
        return mc_impl(g.s, x0, cfg, runs, mean_r_sq, ratios);
    });
}

asyrk_status asyrk_monitor_schedule_next(double target_r_sq, int32_t every, int64_t max_gap, const int64_t* boundaries,
                                         const double* r_sq, int64_t count, int64_t* next) {
    if (!next || count < 1 || !boundaries || !r_sq)
        return fail(ASYRK_E_InvalidArgument, "monitor_schedule_next: need at least one record");
    MonitorSchedule sch;
    sch.reset(target_r_sq, every != 0);
    if (max_gap > 0) sch.max_gap = max_gap;
    long long nx = 0;
    for (int64_t i = std::max<int64_t>(0, count - 2); i < count; ++i) nx = sch.push(boundaries[i], r_sq[i]);
    *next = nx;
    return ASYRK_OK;
}

// rate_fit (ref/src/delay_sim.cpp:272-338): least-squares slope of log(y[k])
// against k * stride, in the reference's summation order. Host arithmetic.
asyrk_status asyrk_rate_fit(const double* y, int64_t count, double stride, double* slope, double* r2) {
    if (!slope || !r2 || (count > 0 && !y)) return fail(ASYRK_E_InvalidArgument, "null argument");
    if (count < 20) return fail(ASYRK_E_InsufficientData, "rate_fit needs >= 20 points");
    if (!(stride > 0.0)) return fail(ASYRK_E_InvalidArgument, "stride must be positive");
    std::vector<double> ly((size_t)count);
    for (int64_t k = 0; k < count; ++k) {
        if (!(y[k] > 0.0))
            return fail(ASYRK_E_NonPositiveData,
                        "rate_fit needs strictly positive values (index " + std::to_string(k) + ")");
        ly[(size_t)k] = std::log(y[k]);
    }
    const double shift = ly[0];
    for (double& v : ly) v -= shift;
    double sx = 0.0, sy = 0.0;
    for (int64_t k = 0; k < count; ++k) {
        sx += static_cast<double>(k);
        sy += ly[(size_t)k];
    }
    const double mx = sx / static_cast<double>(count), my = sy / static_cast<double>(count);
    double sxx = 0.0, sxy = 0.0, syy = 0.0;
    for (int64_t k = 0; k < count; ++k) {
        const double dx = static_cast<double>(k) - mx, dy = ly[(size_t)k] - my;
        sxx += dx * dx;
        sxy += dx * dy;
        syy += dy * dy;
    }
    *slope = sxy / sxx / stride;
    *r2 = syy == 0.0 ? 1.0 : 1.0 - (syy - sxy * sxy / sxx) / syy;
    return ASYRK_OK;
}

asyrk_status asyrk_system_set_rhs(asyrk_system* sys, const double* b) {
    if (!sys || !b) return fail(ASYRK_E_InvalidArgument, "null argument");
    return guarded([&] {
        CK(cudaMemcpyAsync(sys->r, b, (size_t)sys->m * 8, cudaMemcpyHostToDevice, sys->stream));
        launch_set_rhs(sys->layout(), sys->r, sys->stream);
        CK(cudaMemcpyAsync(sys->b, sys->r, (size_t)sys->m * 8, cudaMemcpyDeviceToDevice, sys->stream));
        CK(cudaStreamSynchronize(sys->stream));
        CK(cudaGetLastError());
        return ASYRK_OK;
    });
}

asyrk_status asyrk_system_multiply(asyrk_system* sys, const double* x, double* y) {
    if (!sys || !x || !y) return fail(ASYRK_E_InvalidArgument, "null argument");
    return guarded([&] {
        mon_wait(sys, sys->stream);
        CK(cudaMemcpyAsync(sys->xd, x, (size_t)sys->n * 8, cudaMemcpyHostToDevice, sys->stream));
        launch_spmv_rows(sys->rsell(), sys->precision, sys->m, sys->xd, sys->r, sys->stream);
        CK(cudaMemcpyAsync(y, sys->r, (size_t)sys->m * 8, cudaMemcpyDeviceToHost, sys->stream));
        CK(cudaStreamSynchronize(sys->stream));
        CK(cudaGetLastError());
        return ASYRK_OK;
    });
}

asyrk_status asyrk_system_multiply_transpose(asyrk_system* sys, const double* x, double* y) {
    if (!sys || !x || !y) return fail(ASYRK_E_InvalidArgument, "null argument");
    return guarded([&] {
        mon_wait(sys, sys->stream);
        CK(cudaMemcpyAsync(sys->r, x, (size_t)sys->m * 8, cudaMemcpyHostToDevice, sys->stream));
        launch_spmv_cols(sys->csc(), sys->precision, sys->n, sys->r, sys->g, sys->stream);
        CK(cudaMemcpyAsync(y, sys->g, (size_t)sys->n * 8, cudaMemcpyDeviceToHost, sys->stream));
        CK(cudaStreamSynchronize(sys->stream));
        CK(cudaGetLastError());
        return ASYRK_OK;
    });
}

asyrk_status asyrk_system_sample_rows(asyrk_system* sys, int32_t sampling, uint64_t seed, int64_t warps, int64_t epoch,
                                      int64_t per_warp, int32_t* rows_out) {
    if (!sys || !rows_out || warps < 1 || per_warp < 1 || epoch < 0)
        return fail(ASYRK_E_InvalidArgument, "sample_rows: need a system, warps >= 1, per_warp >= 1, epoch >= 0");
    if (sampling < 0 || sampling > 2) return fail(ASYRK_E_InvalidArgument, "unknown sampling");
    if (sampling == ASYRK_SLICE_SHUFFLE && sys->m < warps)
        return fail(ASYRK_E_InvalidArgument, "slice_shuffle needs at least one row per worker");
    return guarded([&] {
        AllocStream as(sys->stream);
        if (sampling == ASYRK_NORM_PROPORTIONAL) ensure_alias_dev(sys);
        WorkerArgs wa{};
        wa.L = sys->layout();
        wa.alias = sys->alias;
        wa.W = warps;
        const uint64_t k = splitmix64(seed ^ 0xA5A5A5A5DEADBEEFull);  // the solve's key derivation
        wa.key0 = (uint32_t)k;
        wa.key1 = (uint32_t)(k >> 32);
        wa.sampling = sampling == ASYRK_SLICE_SHUFFLE ? S_SLICE : sampling == ASYRK_NORM_PROPORTIONAL ? S_ALIAS : S_UNIFORM;
        const size_t cnt = (size_t)(warps * per_warp);
        int32_t* d = dalloc<int32_t>(cnt);
        launch_sample_rows(wa, epoch, per_warp, d, sys->stream);
        CK(cudaGetLastError());
        CK(cudaMemcpyAsync(rows_out, d, cnt * 4, cudaMemcpyDeviceToHost, sys->stream));
        CK(cudaStreamSynchronize(sys->stream));
        pool_free(d, sys->stream);
        return ASYRK_OK;
    });
}

asyrk_status asyrk_system_microbench_xside(asyrk_system* sys, int32_t warps, int64_t proj_per_warp, int32_t mode,
                                           double* proj_per_s, double* kernel_ms) {
    if (!sys || !proj_per_s) return fail(ASYRK_E_InvalidArgument, "null argument");
    const int32_t theta = (int32_t)(sys->uniform ? sys->uniform_len : sys->max_len);
    const int32_t prec = sys->precision == P_F32 ? P_F32 : P_F64;  // x's element type
    return xside_on_buffer(sys->x, sys->n, theta, prec, warps, proj_per_warp, mode, sys->stream, proj_per_s, kernel_ms);
}

asyrk_status asyrk_system_rk_solve_multi(asyrk_system* sys, const double* B, int64_t k, const double* X0,
                                         const asyrk_rk_config* cfg, double* X_out, asyrk_trace_out* trace) {
    if (!sys) return fail(ASYRK_E_InvalidArgument, "null system");
    return guarded([&] { return rk_multi_impl(sys, B, k, X0, cfg, X_out, trace); });
}

asyrk_status asyrk_system_last_stats(const asyrk_system* sys, asyrk_solve_stats* out) {
    if (!sys || !out) return fail(ASYRK_E_InvalidArgument, "null argument");
    return guarded([&] {
        resolve_stats(const_cast<asyrk_system*>(sys));
        *out = sys->stats;
        return ASYRK_OK;
    });
}

asyrk_status asyrk_system_max_resident_warps(const asyrk_system* sys, int32_t precision, int32_t* out) {
    if (!sys || !out) return fail(ASYRK_E_InvalidArgument, "null argument");
    return guarded([&] {
        *out = worker_max_resident_warps(precision, worker_elems_per_lane(sys->max_len), 1);
        return ASYRK_OK;
    });
}

asyrk_status asyrk_solve_parallel(const asyrk_csr_view* A, const double* b, const double* x0,
                                  const asyrk_run_config* cfg, asyrk_trace_out* trace,
                                  asyrk_instrument_out* instrument) {
    if (!cfg) return fail(ASYRK_E_InvalidArgument, "null config");
    return guarded([&] {
        static const bool prof = env_flag("ASYRK_PROFILE_CREATE");
        const auto t0 = std::chrono::steady_clock::now();
        asyrk_status s;
        {
            SysGuard g;
            const int prec = cfg->threads == 1 ? P_F64 : cfg->precision;
            s = create_impl(A, b, prec, nullptr, &g.s);
            if (s) return s;
            const auto t1 = std::chrono::steady_clock::now();
            s = system_solve_impl(g.s, x0, cfg, trace, instrument);
            if (prof) resolve_stats(g.s);
            if (prof)
                fprintf(stderr, "[one-shot] create %.3f ms solve %.3f ms (device %.3f ms)\n",
                        std::chrono::duration<double, std::milli>(t1 - t0).count(),
                        std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t1).count(),
                        g.s->stats.solve_ms);
        }
        if (prof)
            fprintf(stderr, "[one-shot] total %.3f ms\n",
                    std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
        return s;
    });
}

asyrk_status asyrk_rk_solve(const asyrk_csr_view* A, const double* b, const double* x0, const asyrk_rk_config* cfg,
                            asyrk_trace_out* trace) {
    return guarded([&] {
        SysGuard g;
        asyrk_status s = create_impl(A, b, P_F64, nullptr, &g.s);
        if (s) return s;
        return system_rk_impl(g.s, x0, cfg, trace);
    });
}

asyrk_status asyrk_residuals(const asyrk_csr_view* A, const double* x, const double* b, double* r_sq,
                             double* grad_sq) {
    return guarded([&] {
        SysGuard g;
        asyrk_status s = create_impl(A, b, P_F64, nullptr, &g.s);
        if (s) return s;
        return residuals_impl(g.s, x, r_sq, grad_sq);
    });
}

asyrk_status asyrk_power_iteration_lambda_max(const asyrk_csr_view* A, double tol, int64_t max_iters,
                                              double* lambda_max) {
    return guarded([&] {
        SysGuard g;
        asyrk_status s = create_impl(A, nullptr, P_F64, nullptr, &g.s);
        if (s) return s;
        return power_impl(g.s, tol, max_iters, lambda_max, nullptr);
    });
}

// sweep_threads, ref/src/parallel.cpp:447-481
asyrk_status asyrk_sweep_threads(const asyrk_csr_view* A, const double* b, const double* x0,
                                 const asyrk_run_config* cfg, const int64_t* thread_list, int64_t n_threads,
                                 double* wall_seconds, int64_t* epochs, double* final_r_sq, double* speedup) {
    if (!cfg || !thread_list) return fail(ASYRK_E_InvalidArgument, "null argument");
    if (n_threads <= 0) return fail(ASYRK_E_InvalidArgument, "thread list is empty");
    if (std::find(thread_list, thread_list + n_threads, (int64_t)1) == thread_list + n_threads)
        return fail(ASYRK_E_InvalidArgument, "thread list must contain 1 (the speedup reference)");
    return guarded([&] {
        SysGuard g64, g;
        asyrk_status s = create_impl(A, b, P_F64, nullptr, &g64.s);
        if (s) return s;
        if (cfg->precision != P_F64) {
            s = create_impl(A, b, cfg->precision, nullptr, &g.s);
            if (s) return s;
        }
        const long long cap = 1 + (cfg->epochs + cfg->snapshot_interval - 1) / std::max<int64_t>(1, cfg->snapshot_interval);
        std::vector<int64_t> ep((size_t)cap);
        std::vector<double> rs((size_t)cap), wall((size_t)cap);
        for (int64_t t = 0; t < n_threads; ++t) {
            asyrk_run_config c = *cfg;
            c.threads = thread_list[t];
            asyrk_trace_out tr{};
            tr.cap = cap;
            tr.epoch_index = ep.data();
            tr.r_sq = rs.data();
            tr.wall_seconds = wall.data();
            asyrk_system* sys = (c.threads == 1 || cfg->precision == P_F64) ? g64.s : g.s;
            s = system_solve_impl(sys, x0, &c, &tr, nullptr);
            if (s) return s;
            const int64_t last = std::min<int64_t>(tr.count, cap) - 1;
            wall_seconds[t] = wall[(size_t)last];
            epochs[t] = ep[(size_t)last];
            final_r_sq[t] = rs[(size_t)last];
        }
        double w1 = 0.0;
        for (int64_t t = 0; t < n_threads; ++t)
            if (thread_list[t] == 1) {
                w1 = wall_seconds[t];
                break;
            }
        for (int64_t t = 0; t < n_threads; ++t) speedup[t] = wall_seconds[t] > 0.0 ? w1 / wall_seconds[t] : 0.0;
        return ASYRK_OK;
    });
}

}  // extern "C"

// ===========================================================================
// Multi-right-hand-side AsyRK (BASELINE config 5): asyrk_mrhs_* (asyrk_cuda.h)
// ===========================================================================
struct asyrk_mrhs {
    asyrk_system* sys = nullptr;  // fp32 records + plain CSC of A
    mutable long long stats_timed = -1;  // worker launches whose event times are still to be read
    long long timed = 0;                  // worker launches of the current solve timed with an event pair
    long long spec_launch = -1;           // the launch queued behind the stopping record (-1: none)
    std::vector<long long> lw_epochs, lw_pair;  // mrhs_run: epochs of work / event pair of each worker launch
    int64_t k_total = 0, c0 = 0, c1 = 0, kl = 0;
    float* X = nullptr;           // n x kl
    float* B = nullptr;           // m x kl
    float* R = nullptr;           // m x kl (CSC monitor, ASYRK_MRHS_CSC_MONITOR=1)
    float* G = nullptr;           // n x kl (scatter monitor, default)
    double* Xstar = nullptr;      // n x kl (optional)
    double* part = nullptr;
    double* norms = nullptr;      // device {r_sq, g_sq, d_sq}
    bool have_xstar = false;
    int64_t threads = 0;
    double gamma = 1.0;
    uint64_t seed = 0;
    int sampling = S_UNIFORM;
    int64_t interval = 1, epochs = 0;
    long long max_chunks = 0;
    // host-driven schedule (schedule.h): b = boundaries reached by the enqueued
    // workers, `due` = the last step ended at an evaluated boundary (its norms
    // are what the ranks all-reduce), `pending` = boundary of the last commit
    // whose record the host has not read yet
    MonitorSchedule sch;
    long long b = 0, next_mon = 1, pending = -1;
    bool due = false, stop_seen = false;
    cudaEvent_t ev_commit = nullptr;
    asyrk_solve_stats stats{};
};

namespace {

MrhsArgs mrhs_args(asyrk_mrhs* h) {
    asyrk_system* s = h->sys;
    MrhsArgs a{};
    a.L = s->layout();
    a.X = h->X;
    a.B = h->B;
    a.R = h->R;
    a.G = h->G;
    a.Xstar = h->have_xstar ? h->Xstar : nullptr;
    a.col_ptr = s->col_ptr;
    a.csc_row = s->csc_row;
    a.csc_val = s->csc_val;
    a.part = h->part;
    a.norms = h->norms;
    a.rec = s->recs;
    a.rec_cap = s->rec_cap;
    a.st = s->st;
    a.host_flag = s->host_flag_dev;
    a.W = h->threads;
    a.gamma = h->gamma;
    const uint64_t k = splitmix64(h->seed ^ 0x3C6EF372FE94F82Bull);
    a.key0 = (uint32_t)k;
    a.key1 = (uint32_t)(k >> 32);
    a.KL = (int)h->kl;
    a.sampling = h->sampling;
    a.mirror = s->mirror_dev;
    a.max_len = s->max_len;
    return a;
}

void mrhs_free(asyrk_mrhs* h) {
    if (!h) return;
    if (h->ev_commit) cudaEventDestroy(h->ev_commit);
    if (h->sys) {
        cudaStream_t st = h->sys->stream;
        for (void* p : {(void*)h->X, (void*)h->B, (void*)h->R, (void*)h->G, (void*)h->Xstar, (void*)h->part,
                        (void*)h->norms})
            pool_free(p, st);
        free_all(h->sys);
        delete h->sys;
    }
    delete h;
}

asyrk_status mrhs_create_impl(const asyrk_csr_view* A, const float* B, int64_t k_total, int64_t c0, int64_t c1,
                              void* stream, asyrk_mrhs** out) {
    if (!B || k_total < 1 || c0 < 0 || c1 > k_total || c1 <= c0)
        return fail(ASYRK_E_InvalidArgument, "mrhs: need 0 <= c0 < c1 <= k_total and B");
    const int64_t kl = c1 - c0;
    if (!mrhs_supported_kl(kl))
        return fail(ASYRK_E_InvalidArgument, "mrhs: columns per GPU must be a power of two in [2, 64]");
    auto h = std::unique_ptr<asyrk_mrhs, void (*)(asyrk_mrhs*)>(new asyrk_mrhs, mrhs_free);
    asyrk_status st = create_impl(A, nullptr, P_F32, stream, &h->sys, true);
    if (st) return st;
    asyrk_system* s = h->sys;
    AllocStream as(s->stream);
    h->k_total = k_total;
    h->c0 = c0;
    h->c1 = c1;
    h->kl = kl;
    h->X = dalloc<float>((size_t)s->n * kl);
    h->B = dalloc<float>((size_t)s->m * kl);
    // the monitor's G = A^T R: scattered by the rows pass into G (n x kl, default:
    // one pass over A, no CSC gather of R), or gathered from R over the CSC
    static const bool csc_monitor = env_flag("ASYRK_MRHS_CSC_MONITOR");
    if (csc_monitor)
        h->R = dalloc<float>((size_t)s->m * kl);
    else
        h->G = dalloc<float>((size_t)s->n * kl);
    h->norms = dalloc<double>(4);
    h->part = dalloc<double>((size_t)mrhs_row_blocks(s->m) + 2 * (size_t)mrhs_col_blocks(s->n) + 8);
    // this shard's columns of B, contiguous (host gather, then staged upload)
    std::vector<float> bl((size_t)s->m * kl);
    for (int64_t i = 0; i < s->m; ++i)
        std::memcpy(&bl[(size_t)(i * kl)], B + i * k_total + c0, (size_t)kl * sizeof(float));
    Stager::get().upload(h->B, bl.data(), bl.size() * sizeof(float), s->stream);
    CK(cudaEventCreateWithFlags(&h->ev_commit, cudaEventDisableTiming));
    CK(cudaStreamSynchronize(s->stream));
    *out = h.release();
    return ASYRK_OK;
}

long long mrhs_epoch_of(const asyrk_mrhs* h, long long b) { return std::min<long long>(b * h->interval, h->epochs); }

// X0 / Xstar are full n x k_total host arrays (row-major); this shard takes its columns.
// Leaves the initial residual's norms (this shard) in h->norms: the caller
// all-reduces them, then commits boundary 0.
asyrk_status mrhs_begin_impl(asyrk_mrhs* h, const asyrk_run_config* cfg, const float* X0, const double* Xstar) {
    if (!cfg) return fail(ASYRK_E_InvalidArgument, "null config");
    asyrk_system* s = h->sys;
    if (!s->normalized && !cfg->allow_unnormalized)
        return fail(ASYRK_E_NotNormalized, "solve_parallel requires normalized rows");
    if (cfg->threads < 1) return fail(ASYRK_E_InvalidArgument, "threads must be >= 1");
    if (!(cfg->gamma > 0.0)) return fail(ASYRK_E_InvalidGamma, "gamma must be positive");
    if (cfg->epochs < 0 || cfg->snapshot_interval < 1)
        return fail(ASYRK_E_InvalidArgument, "epochs must be >= 0 and snapshot_interval >= 1");
    if (cfg->sampling != ASYRK_WITH_REPLACEMENT && cfg->sampling != ASYRK_SLICE_SHUFFLE)
        return fail(ASYRK_E_InvalidArgument, "mrhs: sampling must be with_replacement or slice_shuffle");
    if (cfg->sampling == ASYRK_SLICE_SHUFFLE && s->m < cfg->threads)
        return fail(ASYRK_E_InvalidArgument, "slice_shuffle needs at least one row per worker");
    cudaStream_t st = s->stream;
    mon_wait(s, st);
    AllocStream as(st);
    h->threads = cfg->threads;
    h->gamma = cfg->gamma;
    h->seed = cfg->seed;
    h->sampling = cfg->sampling == ASYRK_SLICE_SHUFFLE ? S_SLICE : S_UNIFORM;
    h->interval = cfg->snapshot_interval;
    h->epochs = cfg->epochs;
    h->max_chunks = cfg->epochs > 0 ? (cfg->epochs + cfg->snapshot_interval - 1) / cfg->snapshot_interval : 0;
    h->sch.reset(cfg->target_r_sq, cfg->record_every_boundary != 0);
    h->b = 0;
    h->next_mon = 1;
    h->pending = -1;
    h->stop_seen = false;
    h->stats = asyrk_solve_stats{};
    h->stats_timed = -1;
    h->timed = 0;
    h->spec_launch = -1;
    s->pin_recs = -1;
    ensure_records(s, std::max<long long>(256, h->max_chunks + 2));
    ensure_events(s, h->max_chunks);
    const int64_t kl = h->kl;
    if (X0) {
        std::vector<float> xl((size_t)s->n * kl);
        for (int64_t j = 0; j < s->n; ++j)
            std::memcpy(&xl[(size_t)(j * kl)], X0 + j * h->k_total + h->c0, (size_t)kl * sizeof(float));
        CK(cudaMemcpyAsync(h->X, xl.data(), xl.size() * sizeof(float), cudaMemcpyHostToDevice, st));
        CK(cudaStreamSynchronize(st));
    } else {
        CK(cudaMemsetAsync(h->X, 0, (size_t)s->n * kl * sizeof(float), st));
    }
    h->have_xstar = Xstar != nullptr;
    if (Xstar) {
        if (!h->Xstar) h->Xstar = dalloc<double>((size_t)s->n * kl);
        std::vector<double> xs((size_t)s->n * kl);
        for (int64_t j = 0; j < s->n; ++j)
            std::memcpy(&xs[(size_t)(j * kl)], Xstar + j * h->k_total + h->c0, (size_t)kl * sizeof(double));
        CK(cudaMemcpyAsync(h->Xstar, xs.data(), xs.size() * sizeof(double), cudaMemcpyHostToDevice, st));
        CK(cudaStreamSynchronize(st));
    }
    *s->host_flag = 0;
    std::memset(s->mirror, 0, sizeof(HostMirror));
    h->lw_epochs.clear();
    h->lw_pair.clear();
    CK(cudaEventRecord(s->ev_begin, st));
    launch_state_init(s->st, cfg->epochs, cfg->snapshot_interval, cfg->target_r_sq, st);
    launch_mrhs_monitor(mrhs_args(h), st);  // initial residual -> norms (this shard)
    h->due = true;
    h->stats.kernel_launches += 4;
    h->stats.monitor_launches++;
    CK(cudaGetLastError());
    return ASYRK_OK;
}

// record of the boundary the last step reached (only at evaluated boundaries)
void mrhs_commit_impl(asyrk_mrhs* h) {
    if (!h->due) return;
    launch_mrhs_commit(mrhs_args(h), h->b == 0 ? -1 : mrhs_epoch_of(h, h->b), h->sys->stream);
    CK(cudaEventRecord(h->ev_commit, h->sys->stream));
    h->pending = h->b;
    h->due = false;
    h->stats.kernel_launches += 1;
    CK(cudaGetLastError());
}

// read the pending record (waits for its commit): stop flag + next evaluation
bool mrhs_read_pending(asyrk_mrhs* h) {
    if (h->pending < 0) return h->stop_seen;
    CK(cudaEventSynchronize(h->ev_commit));
    const volatile HostMirror* hm = h->sys->mirror;
    if (hm->stop) h->stop_seen = true;
    else h->next_mon = h->sch.push(h->pending, hm->r_sq);
    h->pending = -1;
    return h->stop_seen;
}

// workers of chunks b .. b_end - 1 in one launch (boundary b -> b_end; b_end <= 0:
// one chunk). mrhs_run fuses the chunks up to the next scheduled evaluation as
// run_scheduled does (per-launch epochs in lw_epochs; those launches and the
// sampled single ones are timed)
void mrhs_enqueue_worker(asyrk_mrhs* h, long long b_end = 0, bool track = false) {
    asyrk_system* s = h->sys;
    cudaStream_t st = s->stream;
    if (b_end <= h->b) b_end = h->b + 1;
    MrhsArgs a = mrhs_args(h);
    a.epoch0 = mrhs_epoch_of(h, h->b);
    a.span0 = mrhs_epoch_of(h, b_end) - a.epoch0;
    const long long t = h->stats.worker_launches;
    const long long k = h->timed;
    const bool time_it = (timed_launch(t) || (track && b_end - h->b > 1)) && k < kTimedLaunches &&
                         (size_t)(2 * k + 1) < s->ev_w.size();
    if (time_it) CK(cudaEventRecord(s->ev_w[(size_t)(2 * k)], st));
    launch_mrhs_worker(a, st);
    if (track) {
        h->lw_epochs.push_back(a.span0);
        h->lw_pair.push_back(time_it ? k : -1);
    }
    if (time_it) {
        CK(cudaEventRecord(s->ev_w[(size_t)(2 * k + 1)], st));
        h->timed++;
    }
    h->b = b_end;
    h->stats.worker_launches++;
    h->stats.kernel_launches++;
    CK(cudaGetLastError());
}

// the monitor of boundary b if the schedule evaluates it (always the last one)
void mrhs_maybe_monitor(asyrk_mrhs* h) {
    h->due = h->b >= h->next_mon || h->b >= h->max_chunks;
    if (!h->due) return;
    launch_mrhs_monitor(mrhs_args(h), h->sys->stream);
    h->stats.monitor_launches++;
    h->stats.kernel_launches += 3;
    CK(cudaGetLastError());
}

// the last solve's event times (its events are untouched until the next solve)
void mrhs_resolve_stats(asyrk_mrhs* h) {
    if (h->stats_timed < 0) return;
    asyrk_system* s = h->sys;
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, s->ev_begin, s->ev_end));
    h->stats.solve_ms = ms;
    const long long timed = h->stats_timed;
    h->stats_timed = -1;
    if (!h->lw_epochs.empty()) {  // mrhs_run: timed launches' ms per epoch x all epochs of work
        double t_ms = 0.0, t_ep = 0.0, all_ep = 0.0;
        for (size_t i = 0; i < h->lw_epochs.size(); ++i) {
            all_ep += (double)h->lw_epochs[i];
            const long long p = h->lw_pair[i];
            if (p < 0 || h->lw_epochs[i] <= 0) continue;
            float lm = 0.f;
            CK(cudaEventElapsedTime(&lm, s->ev_w[(size_t)(2 * p)], s->ev_w[(size_t)(2 * p + 1)]));
            t_ms += lm;
            t_ep += (double)h->lw_epochs[i];
        }
        h->stats.worker_ms = t_ep > 0.0 ? t_ms * all_ep / t_ep : 0.0;
        return;
    }
    h->stats.worker_ms = sampled_worker_ms(s, timed, h->stats.worker_launches, h->spec_launch);
}

asyrk_status mrhs_finish_impl(asyrk_mrhs* h, asyrk_trace_out* trace, float* X_out) {
    asyrk_system* s = h->sys;
    cudaStream_t st = s->stream;
    CK(cudaEventRecord(s->ev_end, st));
    pin_final(s, h->stats.monitor_launches, st);  // state + records behind the last kernel
    CK(cudaStreamSynchronize(st));
    DevState hs;
    std::memcpy(&hs, pin_state(s), sizeof(DevState));
    h->stats_timed = h->timed;  // sampled launches (mrhs_resolve_stats)
    h->stats.projections = hs.updates;
    h->stats.warps = (int32_t)std::min<int64_t>(h->threads, INT32_MAX);
    if (hs.status == ASYRK_E_NonFinite) return fail(ASYRK_E_NonFinite, "iterate became non-finite");
    if (trace) {
        const long long k = std::min<long long>(hs.nrec, s->rec_cap);
        std::vector<DevRecord> recs((size_t)k);
        if (k && k <= s->pin_recs)
            std::memcpy(recs.data(), pin_records(s), (size_t)k * sizeof(DevRecord));
        else if (k)
            CK(cudaMemcpy(recs.data(), s->recs, (size_t)k * sizeof(DevRecord), cudaMemcpyDeviceToHost));
        trace->count = hs.nrec;
        const long long w = std::min<long long>(k, trace->cap);
        for (long long i = 0; i < w; ++i) {
            const DevRecord& r = recs[(size_t)i];
            if (trace->epoch_index) trace->epoch_index[i] = r.epoch;
            if (trace->r_sq) trace->r_sq[i] = r.r_sq;
            if (trace->grad_sq) trace->grad_sq[i] = r.grad_sq;
            if (trace->dist_sq) trace->dist_sq[i] = r.dist_sq;
            if (trace->wall_seconds) trace->wall_seconds[i] = 1e-9 * (double)r.t_ns;
            if (trace->updates_applied) trace->updates_applied[i] = r.updates;
        }
    }
    if (X_out) {
        const size_t xb = (size_t)s->n * h->kl * sizeof(float);
        static const bool plain = env_flag("ASYRK_PLAIN_DOWNLOAD");  // (A/B)
        if (xb >= (8u << 20) && !plain) {
            Stager::get().download(X_out, h->X, xb, st);  // large: through the pinned slots
        } else {
            CK(cudaMemcpyAsync(X_out, h->X, xb, cudaMemcpyDeviceToHost, st));
            CK(cudaStreamSynchronize(st));
        }
    }
    return ASYRK_OK;
}

// ---- NCCL, resolved at run time (libnccl.so.2: the copy already loaded in
// the process — e.g. PyTorch's — if there is one, else the system library), so
// the library itself has no link-time NCCL dependency.
struct NcclApi {
    bool ok = false;
    std::string why;
    decltype(&ncclGetUniqueId) getUniqueId = nullptr;
    decltype(&ncclCommInitRank) commInitRank = nullptr;
    decltype(&ncclCommInitAll) commInitAll = nullptr;
    decltype(&ncclCommDestroy) commDestroy = nullptr;
    decltype(&ncclAllReduce) allReduce = nullptr;
    decltype(&ncclGroupStart) groupStart = nullptr;
    decltype(&ncclGroupEnd) groupEnd = nullptr;
    decltype(&ncclGetErrorString) errorString = nullptr;
    decltype(&ncclGetVersion) getVersion = nullptr;
};

const NcclApi& nccl() {
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            api.why = std::string("libnccl.so.2 not loadable: ") + (dlerror() ? dlerror() : "?");
            return;
        }
#define AK_NCCL_SYM(field, name)                                                   \
    api.field = reinterpret_cast<decltype(api.field)>(dlsym(h, name));            \
    if (!api.field) {                                                              \
        api.why = std::string("libnccl.so.2 lacks ") + name;                       \
        return;                                                                    \
    }
        AK_NCCL_SYM(getUniqueId, "ncclGetUniqueId")
        AK_NCCL_SYM(commInitRank, "ncclCommInitRank")
        AK_NCCL_SYM(commInitAll, "ncclCommInitAll")
        AK_NCCL_SYM(commDestroy, "ncclCommDestroy")
        AK_NCCL_SYM(allReduce, "ncclAllReduce")
        AK_NCCL_SYM(groupStart, "ncclGroupStart")
        AK_NCCL_SYM(groupEnd, "ncclGroupEnd")
        AK_NCCL_SYM(errorString, "ncclGetErrorString")
        AK_NCCL_SYM(getVersion, "ncclGetVersion")
#undef AK_NCCL_SYM
        api.ok = true;
    });
    return api;
}

#define NK(call)                                                                                      \
    do {                                                                                              \
        ncclResult_t r_ = (call);                                                                     \
        if (r_ != ncclSuccess) {                                                                      \
            ::ak::err_buf() = std::string("NCCL: ") + nccl().errorString(r_) + " at " #call;          \
            throw ::ak::CudaFail{ASYRK_E_ThreadSpawnFailure};                                         \
        }                                                                                             \
    } while (0)

asyrk_status need_nccl() {
    if (!nccl().ok) return fail(ASYRK_E_ThreadSpawnFailure, nccl().why);
    return ASYRK_OK;
}

// The whole sharded solve in C++ for G shards (one per device; G = 1 without
// NCCL). Per boundary: every shard's workers; at an evaluated boundary the
// shards' monitors, one all-reduce of {r_sq, g_sq, d_sq} over the shards (a
// grouped ncclAllReduce on each shard's stream), the commits (identical global
// record + stop on every shard). The worker launches of the next boundary are
// enqueued behind the commits before the host reads the record, so the read
// overlaps an epoch; they run only if the record did not stop the solve.
asyrk_status mrhs_run(std::vector<asyrk_mrhs*>& hs, const std::vector<int>& devs, const std::vector<ncclComm_t>& comms,
                      const asyrk_run_config* cfg, const float* X0, const double* Xstar) {
    const size_t G = hs.size();
    auto on = [&](size_t g) {
        if (!devs.empty()) CK(cudaSetDevice(devs[g]));
    };
    auto allreduce = [&] {
        if (comms.empty()) return;
        NK(nccl().groupStart());
        for (size_t g = 0; g < G; ++g) {
            on(g);
            NK(nccl().allReduce(hs[g]->norms, hs[g]->norms, 3, ncclDouble, ncclSum, comms[g], hs[g]->sys->stream));
        }
        NK(nccl().groupEnd());
    };
    auto commit_all = [&] {
        allreduce();
        for (size_t g = 0; g < G; ++g) {
            on(g);
            mrhs_commit_impl(hs[g]);
        }
    };
    for (size_t g = 0; g < G; ++g) {
        on(g);
        asyrk_status st = mrhs_begin_impl(hs[g], cfg, X0, Xstar);
        if (st) return st;
    }
    commit_all();  // boundary 0
    asyrk_mrhs* h0 = hs[0];
    // fused launches up to the next evaluation (ASYRK_MRHS_FUSE=1) are off by
    // default here: at config 5 (0.57 ms epochs) they measured 22.6 vs 22.2 ms
    // per solve and the same per-rank shard times (profiles/r02_ab_c5*.json)
    static const bool fuse = env_flag("ASYRK_MRHS_FUSE") && !env_flag("ASYRK_NO_FUSE");
    while (h0->b < h0->max_chunks) {
        // with every record read, the next evaluation is known: one launch up to it
        // (the same on every shard and rank: the schedule follows the all-reduced records)
        const long long b_end = (h0->pending < 0 && fuse)
                                    ? std::min(std::max(h0->next_mon, h0->b + 1), h0->max_chunks)
                                    : h0->b + 1;
        for (size_t g = 0; g < G; ++g) {
            on(g);
            mrhs_enqueue_worker(hs[g], b_end, true);
        }
        // the record of the last commit (if any) is read while these workers run
        on(0);
        const bool stop = mrhs_read_pending(h0);
        for (size_t g = 1; g < G; ++g) {
            hs[g]->stop_seen = stop;
            hs[g]->next_mon = h0->next_mon;
            hs[g]->pending = -1;
        }
        if (stop) {  // the workers just enqueued see go = 0 and exit
            for (size_t g = 0; g < G; ++g) {
                hs[g]->spec_launch = hs[g]->stats.worker_launches - 1;
                if (!hs[g]->lw_epochs.empty()) hs[g]->lw_epochs.back() = 0;
            }
            break;
        }
        for (size_t g = 0; g < G; ++g) {
            on(g);
            mrhs_maybe_monitor(hs[g]);
        }
        if (h0->due) commit_all();
    }
    return ASYRK_OK;
}

}  // namespace

extern "C" {

asyrk_status asyrk_mrhs_create(const asyrk_csr_view* A, const float* B, int64_t k_total, int64_t c0, int64_t c1,
                               void* stream, asyrk_mrhs** out) {
    return guarded([&] { return mrhs_create_impl(A, B, k_total, c0, c1, stream, out); });
}

asyrk_status asyrk_mrhs_destroy(asyrk_mrhs* h) {
    mrhs_free(h);
    return ASYRK_OK;
}

asyrk_status asyrk_mrhs_begin(asyrk_mrhs* h, const asyrk_run_config* cfg, const float* X0, const double* Xstar) {
    if (!h) return fail(ASYRK_E_InvalidArgument, "null mrhs");
    return guarded([&] { return mrhs_begin_impl(h, cfg, X0, Xstar); });
}

asyrk_status asyrk_mrhs_norms(asyrk_mrhs* h, double** dev_norms) {
    if (!h || !dev_norms) return fail(ASYRK_E_InvalidArgument, "null argument");
    *dev_norms = h->norms;
    return ASYRK_OK;
}

asyrk_status asyrk_mrhs_due(asyrk_mrhs* h, int32_t* due) {
    if (!h || !due) return fail(ASYRK_E_InvalidArgument, "null argument");
    *due = h->due ? 1 : 0;
    return ASYRK_OK;
}

asyrk_status asyrk_mrhs_commit(asyrk_mrhs* h, int32_t advance) {
    if (!h) return fail(ASYRK_E_InvalidArgument, "null mrhs");
    (void)advance;  // the boundary is the one the last step reached (or 0 after begin)
    return guarded([&] {
        mrhs_commit_impl(h);
        return ASYRK_OK;
    });
}

asyrk_status asyrk_mrhs_step(asyrk_mrhs* h) {
    if (!h) return fail(ASYRK_E_InvalidArgument, "null mrhs");
    return guarded([&] {
        mrhs_read_pending(h);
        mrhs_enqueue_worker(h);
        mrhs_maybe_monitor(h);
        return ASYRK_OK;
    });
}

asyrk_status asyrk_mrhs_stopped(asyrk_mrhs* h, int32_t* stopped) {
    if (!h || !stopped) return fail(ASYRK_E_InvalidArgument, "null argument");
    return guarded([&] {
        // the decision of the latest commit (each commit's record is read on
        // its own, after its event): every rank sees the same sequence
        const bool st = mrhs_read_pending(h);
        *stopped = (st || h->b >= h->max_chunks) ? 1 : 0;
        return ASYRK_OK;
    });
}

asyrk_status asyrk_mrhs_finish(asyrk_mrhs* h, asyrk_trace_out* trace, float* X_out) {
    if (!h) return fail(ASYRK_E_InvalidArgument, "null mrhs");
    return guarded([&] { return mrhs_finish_impl(h, trace, X_out); });
}

asyrk_status asyrk_mrhs_solve(asyrk_mrhs* h, const asyrk_run_config* cfg, const float* X0, const double* Xstar,
                              asyrk_trace_out* trace, float* X_out) {
    if (!h) return fail(ASYRK_E_InvalidArgument, "null mrhs");
    return guarded([&] {
        std::vector<asyrk_mrhs*> hs{h};
        asyrk_status st = mrhs_run(hs, {}, {}, cfg, X0, Xstar);
        if (st) return st;
        return mrhs_finish_impl(h, trace, X_out);
    });
}

asyrk_status asyrk_mrhs_microbench_xside(asyrk_mrhs* h, int32_t warps, int64_t proj_per_warp, double* proj_per_s,
                                         double* kernel_ms) {
    if (!h || !proj_per_s) return fail(ASYRK_E_InvalidArgument, "null argument");
    if (warps < 1 || proj_per_warp < 1) return fail(ASYRK_E_InvalidArgument, "warps and proj_per_warp must be >= 1");
    return guarded([&] {
        asyrk_system* s = h->sys;
        const int32_t theta = (int32_t)(s->uniform ? s->uniform_len : s->max_len);
        if (theta > 32) return fail(ASYRK_E_InvalidArgument, "mrhs microbench: rows of at most 32 nonzeros");
        // the shard's own X (re-initialized by every solve), as config 2's R_x uses the solver's x
        return (asyrk_status)xside_mrhs_on_buffer(h->X, s->n, theta, (int32_t)h->kl, warps, proj_per_warp, s->stream, proj_per_s,
                                    kernel_ms);
    });
}

asyrk_status asyrk_mrhs_max_resident_warps(const asyrk_mrhs* h, int32_t* out) {
    if (!h || !out) return fail(ASYRK_E_InvalidArgument, "null argument");
    return guarded([&] {
        *out = mrhs_max_resident_warps((int)h->kl, h->sys->max_len);
        return ASYRK_OK;
    });
}

asyrk_status asyrk_mrhs_last_stats(const asyrk_mrhs* h, asyrk_solve_stats* out) {
    if (!h || !out) return fail(ASYRK_E_InvalidArgument, "null argument");
    return guarded([&] {
        mrhs_resolve_stats(const_cast<asyrk_mrhs*>(h));
        *out = h->stats;
        return ASYRK_OK;
    });
}

// ---- multi-GPU (NCCL)
asyrk_status asyrk_nccl_available(int32_t* version) {
    if (!version) return fail(ASYRK_E_InvalidArgument, "null argument");
    *version = 0;
    if (!nccl().ok) return fail(ASYRK_E_ThreadSpawnFailure, nccl().why);
    int v = 0;
    nccl().getVersion(&v);
    *version = v;
    return ASYRK_OK;
}

asyrk_status asyrk_nccl_get_unique_id(char* id) {
    if (!id) return fail(ASYRK_E_InvalidArgument, "null argument");
    return guarded([&] {
        asyrk_status st = need_nccl();
        if (st) return st;
        ncclUniqueId u;
        NK(nccl().getUniqueId(&u));
        static_assert(sizeof(ncclUniqueId) == ASYRK_NCCL_UNIQUE_ID_BYTES, "ncclUniqueId size");
        std::memcpy(id, &u, sizeof(u));
        return ASYRK_OK;
    });
}

asyrk_status asyrk_nccl_comm_init_rank(void** comm, int32_t nranks, const char* id, int32_t rank) {
    if (!comm || !id || nranks < 1 || rank < 0 || rank >= nranks)
        return fail(ASYRK_E_InvalidArgument, "nccl_comm_init_rank: need comm, id and 0 <= rank < nranks");
    return guarded([&] {
        asyrk_status st = need_nccl();
        if (st) return st;
        ncclUniqueId u;
        std::memcpy(&u, id, sizeof(u));
        ncclComm_t c = nullptr;
        NK(nccl().commInitRank(&c, nranks, u, rank));
        *comm = c;
        return ASYRK_OK;
    });
}

asyrk_status asyrk_nccl_comm_destroy(void* comm) {
    if (!comm) return ASYRK_OK;
    return guarded([&] {
        asyrk_status st = need_nccl();
        if (st) return st;
        NK(nccl().commDestroy(static_cast<ncclComm_t>(comm)));
        return ASYRK_OK;
    });
}

asyrk_status asyrk_mrhs_solve_nccl(asyrk_mrhs* h, const asyrk_run_config* cfg, void* comm, const float* X0,
                                   const double* Xstar, asyrk_trace_out* trace, float* X_out) {
    if (!h || !comm) return fail(ASYRK_E_InvalidArgument, "null mrhs or communicator");
    return guarded([&] {
        asyrk_status st = need_nccl();
        if (st) return st;
        std::vector<asyrk_mrhs*> hs{h};
        st = mrhs_run(hs, {}, {static_cast<ncclComm_t>(comm)}, cfg, X0, Xstar);
        if (st) return st;
        return mrhs_finish_impl(h, trace, X_out);
    });
}

asyrk_status asyrk_mrhs_solve_devices(const asyrk_csr_view* A, const float* B, int64_t k_total, const int32_t* devices,
                                      int32_t ndev, const asyrk_run_config* cfg, const float* X0, const double* Xstar,
                                      asyrk_trace_out* trace, float* X_out, asyrk_solve_stats* stats) {
    if (!A || !B || !devices || ndev < 1 || !cfg) return fail(ASYRK_E_InvalidArgument, "null argument or ndev < 1");
    if (k_total % ndev) return fail(ASYRK_E_InvalidArgument, "mrhs: k_total must split evenly over the devices");
    return guarded([&] {
        asyrk_status st = need_nccl();
        if (st) return st;
        int prev = 0;
        CK(cudaGetDevice(&prev));
        std::vector<int> devs(devices, devices + ndev);
        std::vector<asyrk_mrhs*> hs((size_t)ndev, nullptr);
        std::vector<ncclComm_t> comms((size_t)ndev, nullptr);
        auto cleanup = [&] {
            for (size_t g = 0; g < hs.size(); ++g) {
                cudaSetDevice(devs[g]);
                if (comms[g]) nccl().commDestroy(comms[g]);
                mrhs_free(hs[g]);
            }
            cudaSetDevice(prev);
        };
        try {
            const int64_t kl = k_total / ndev;
            for (int g = 0; g < ndev; ++g) {
                CK(cudaSetDevice(devs[(size_t)g]));
                st = mrhs_create_impl(A, B, k_total, g * kl, (g + 1) * kl, nullptr, &hs[(size_t)g]);
                if (st) {
                    cleanup();
                    return st;
                }
            }
            NK(nccl().commInitAll(comms.data(), ndev, devs.data()));
            st = mrhs_run(hs, devs, comms, cfg, X0, Xstar);
            std::vector<float> xl;
            for (int g = 0; g < ndev && !st; ++g) {
                CK(cudaSetDevice(devs[(size_t)g]));
                asyrk_mrhs* h = hs[(size_t)g];
                xl.assign((size_t)h->sys->n * kl, 0.f);
                st = mrhs_finish_impl(h, g == 0 ? trace : nullptr, X_out ? xl.data() : nullptr);
                if (!st && X_out)
                    for (int64_t j = 0; j < h->sys->n; ++j)
                        std::memcpy(X_out + j * k_total + g * kl, &xl[(size_t)(j * kl)], (size_t)kl * sizeof(float));
                if (!st && stats && g == 0) {
                    mrhs_resolve_stats(h);
                    *stats = h->stats;
                }
            }
        } catch (...) {
            cleanup();
            throw;
        }
        cleanup();
        return st;
    });
}

}  // extern "C"
