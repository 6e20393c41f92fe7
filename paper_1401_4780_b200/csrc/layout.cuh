// Device data layout of the AsyRK hot path and the device-side helpers every
// kernel shares. See DESIGN.md §"Data layout in HBM".
//
// Row records. Row i of A (ref CsrMatrix, csr.hpp:69-75) is stored as ONE
// contiguous, 16-byte aligned record so a worker warp fetches everything a
// projection needs with a single dependent round trip:
//
//     +0   double b_i            (right-hand side)
//     +8   double inv_nrm2_i     (1 / (row_norm_i * row_norm_i))
//     +16  V      vals[len]      (V = double | float)
//     +16+len*sizeof(V)  int32 cols[len]
//     ... zero pad to 16 B
//
// When every row has the same nonzero count (all BASELINE configs) the record
// address is i * stride and no row_ptr is read at all; ragged matrices carry a
// uint2 {offset/16, len} per row.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace ak {

constexpr unsigned FULL = 0xffffffffu;

struct Layout {
    const unsigned char* rec;  // records
    const uint2* row_info;     // {off16, len} per row, or nullptr when uniform
    uint32_t stride16;         // uniform record stride / 16 B
    uint32_t uniform_len;      // uniform nonzeros per row
    int64_t m, n;
    size_t rec_bytes;          // total record bytes
};

struct RowRef {
    const unsigned char* base;
    int len;
};

__device__ __forceinline__ RowRef row_ref(const Layout& L, int64_t i) {
    RowRef r;
    if (L.row_info == nullptr) {
        r.base = L.rec + (size_t)i * ((size_t)L.stride16 * 16u);
        r.len = (int)L.uniform_len;
    } else {
        const uint2 info = __ldg(L.row_info + i);
        r.base = L.rec + (size_t)info.x * 16u;
        r.len = (int)info.y;
    }
    return r;
}

template <class V>
__device__ __forceinline__ const V* rec_vals(const RowRef& r) {
    return reinterpret_cast<const V*>(r.base + 16);
}
template <class V>
__device__ __forceinline__ const int32_t* rec_cols(const RowRef& r) {
    return reinterpret_cast<const int32_t*>(r.base + 16 + (size_t)r.len * sizeof(V));
}
__device__ __forceinline__ double rec_b(const RowRef& r) { return __ldg(reinterpret_cast<const double*>(r.base)); }
__device__ __forceinline__ double rec_inv(const RowRef& r) {
    return __ldg(reinterpret_cast<const double*>(r.base + 8));
}

// Host/device: record size in 16-byte units for a row of `len` nonzeros.
__host__ __device__ inline uint32_t rec_size16(uint32_t len, int vbytes) {
    const uint64_t bytes = 16ull + (uint64_t)len * (uint64_t)(vbytes + 4);
    return (uint32_t)((bytes + 15ull) / 16ull);
}

// Coordinator state shared by the worker, monitor and finalize kernels of one
// solve. Kernels of a chunk read it at entry; only finalize writes it.
struct DevState {
    long long epoch;        // epochs completed (ref parallel.cpp:465-484 "boundary")
    long long updates;      // row projections applied
    long long nrec;         // trace records written
    long long epochs_cap;   // RunConfig::epochs / RkConfig::max_epochs
    long long interval;     // snapshot_interval
    double target;          // target_r_sq (absolute, as in the reference)
    unsigned long long t0_ns;
    int stop;               // no further work
    int status;             // 0 or ASYRK_E_NonFinite
    long long increments;   // instrument: component increments applied
    // overlapped async solves: the worker launch runs iff go (decided on the
    // worker stream before it, so every block of a launch agrees); snapshots
    // of x at epoch boundaries feed the monitor stream
    int go;
    int snap_valid[2];
    long long snap_epoch[2], snap_updates[2];
    // the snapshot whose record decided the stop (-1: none / in-stream): the
    // solve returns that snapshot, not the epochs that ran past it
    int stop_slot;
    long long stop_epoch, stop_updates;
    // last-block tickets of the fused snapshot+advance and columns+finalize kernels
    unsigned snap_ticket, mon_ticket;
    // decoupled snapshots (the reference coordinator's "latest boundary"): slot
    // states 0 free, 1 filling, 2 filled, 3 being monitored; the snapshot kernel's
    // first block picks a free slot (or none), the monitor claims the oldest filled
    int slot_state[2];
    unsigned snap_arrive, snap_seq, snap_decided;
    int snap_target, mon_slot;
};

// Pinned, device-mapped copy of the latest record's decision inputs, written
// by the record kernel (__threadfence_system): the host-driven monitor
// schedule reads it after the record's event without a copy.
struct HostMirror {
    long long epoch;        // epoch of the latest record
    long long nrec;         // records written so far
    double r_sq;            // its r_sq (the all-reduced one for multi-RHS shards)
    int stop;               // stop decided (target, epoch cap or NonFinite)
    int status;             // 0 or ASYRK_E_NonFinite
    long long seq;          // commits seen (multi-RHS: index of the latest commit + 1)
    long long pad[2];
};

struct DevRecord {
    long long epoch;
    long long updates;
    double r_sq, grad_sq, dist_sq;
    unsigned long long t_ns;
};

__device__ __forceinline__ unsigned long long globaltimer_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__device__ __forceinline__ long long chunk_span(const DevState* st) {
    const long long left = st->epochs_cap - st->epoch;
    return st->interval < left ? st->interval : left;
}

// ---- counter-based RNG: Philox4x32-10 (Salmon, Moraes, Dror, Shaw, SC'11)
struct U4 {
    uint32_t x, y, z, w;
};
__device__ __forceinline__ U4 philox4x32(U4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const uint32_t lo0 = 0xD2511F53u * c.x, hi0 = __umulhi(0xD2511F53u, c.x);
        const uint32_t lo1 = 0xCD9E8D57u * c.z, hi1 = __umulhi(0xCD9E8D57u, c.z);
        c = U4{hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0};
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    return c;
}

// Uniform integer in [0, n) from 64 random bits (multiply-high; bias < n/2^64).
__device__ __forceinline__ uint64_t bounded64(uint64_t r, uint64_t n) { return __umul64hi(r, n); }

// ---- keyed bijection on [0, L): 4-round Feistel network on 2h bits with
// cycle walking (domain < 4L, so < 4 walks expected). Used for the
// slice_shuffle passes (ref parallel.cpp:355-363 reshuffles each slice per pass).
__device__ __forceinline__ uint32_t feistel_round(uint32_t r, uint32_t k) {
    uint32_t h = r * 0x9E3779B1u ^ k;
    h ^= h >> 15;
    h *= 0x2C1B3C6Du;
    h ^= h >> 12;
    h *= 0x297A2D39u;
    h ^= h >> 15;
    return h;
}
__device__ __forceinline__ uint32_t permute_index(uint32_t x, uint32_t L, uint32_t half_bits, uint32_t k0,
                                                  uint32_t k1) {
    const uint32_t mask = (half_bits >= 32) ? 0xffffffffu : ((1u << half_bits) - 1u);
    do {
        uint32_t l = x >> half_bits, r = x & mask;
#pragma unroll
        for (int round = 0; round < 4; ++round) {
            const uint32_t f = feistel_round(r, (round & 1) ? k1 + round : k0 + round) & mask;
            const uint32_t nl = r;
            r = l ^ f;
            l = nl;
        }
        x = (l << half_bits) | r;
    } while (x >= L);
    return x;
}
__host__ __device__ inline uint32_t feistel_half_bits(uint32_t L) {
    uint32_t b = 0;
    while ((1ull << b) < (unsigned long long)L) ++b;
    return (b + 1) / 2;
}

// ---- increment audit of the async workers (instrumented solves): K signed
// checksums of every increment applied, sum_c s_k(c) * d, with s_k(c) = +-1
// from bit k of a hash of the component; the audit compares them with
// sum_j s_k(j) (x_j - x0_j) (pack.cu). A lost or repeated increment d on
// component c moves every checksum by +-d.
constexpr int kAuditK = 4;
__host__ __device__ __forceinline__ uint32_t audit_hash(uint32_t c) {
    c ^= c >> 16;
    c *= 0x7feb352du;
    c ^= c >> 15;
    c *= 0x846ca68bu;
    c ^= c >> 16;
    return c;
}
__device__ __forceinline__ void audit_add(double (&cs)[kAuditK], int c, double d) {
    const uint32_t h = audit_hash((uint32_t)c);
#pragma unroll
    for (int k = 0; k < kAuditK; ++k) cs[k] += ((h >> k) & 1u) ? d : -d;
}

// x reads bypass L1 (it is not coherent with other SMs' red.global adds);
// A is immutable and read through the non-coherent path.
__device__ __forceinline__ double ld_x(const double* p) { return __ldcg(p); }
__device__ __forceinline__ float ld_x(const float* p) { return __ldcg(p); }

template <class T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
    return v;
}

}  // namespace ak
