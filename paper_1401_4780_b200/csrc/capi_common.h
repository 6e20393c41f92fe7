// Shared plumbing of the C-ABI translation units (system.cu, mrhs_system.cu):
// the thread-local error message, CUDA error mapping onto the reference's
// ErrorCode numbering, and stream-ordered device allocation.
#pragma once
#include <new>
#include <stdexcept>
#include <string>

#include <cuda_runtime.h>

#include "../../include/asyrk_cuda.h"
#include "runtime.h"

namespace ak {

std::string& err_buf();  // message returned by asyrk_last_error()

inline asyrk_status fail(asyrk_status s, const std::string& msg) {
    err_buf() = msg;
    return s;
}

struct CudaFail {
    asyrk_status st;
};

// CUDA failures: out of memory -> TooLarge, anything else -> ThreadSpawnFailure
// (the reference's "could not start the workers"); the message names the call.
#define CK(call)                                                                                       \
    do {                                                                                               \
        cudaError_t e_ = (call);                                                                       \
        if (e_ != cudaSuccess) {                                                                       \
            ::ak::err_buf() = std::string("CUDA: ") + cudaGetErrorString(e_) + " at " #call " (" +    \
                              __FILE__ + ":" + std::to_string(__LINE__) + ")";                         \
            throw ::ak::CudaFail{e_ == cudaErrorMemoryAllocation ? ASYRK_E_TooLarge                    \
                                                                 : ASYRK_E_ThreadSpawnFailure};        \
        }                                                                                              \
    } while (0)

template <class F>
asyrk_status guarded(F&& f) {
    try {
        return f();
    } catch (const CudaFail& c) {
        return c.st;
    } catch (const std::bad_alloc&) {
        return fail(ASYRK_E_TooLarge, "host allocation failed");
    } catch (const std::exception& e) {
        return fail(ASYRK_E_InvalidArgument, e.what());
    }
}

// Device allocations are stream-ordered pool allocations on the owning
// object's stream (runtime.h), selected per entry point with AllocStream.
extern thread_local cudaStream_t g_alloc_stream;

template <class T>
T* dalloc(size_t count) {
    void* p = nullptr;
    if (count == 0) count = 1;
    CK(pool_alloc(&p, count * sizeof(T), g_alloc_stream));
    return static_cast<T*>(p);
}

struct AllocStream {
    cudaStream_t prev;
    explicit AllocStream(cudaStream_t s) : prev(g_alloc_stream) { g_alloc_stream = s; }
    ~AllocStream() { g_alloc_stream = prev; }
};

}  // namespace ak
