// K0 — CSR upload and device layout packing (replaces the storage of
// CsrMatrix, ref/include/asyrk/csr.hpp:69-75, as seen by the hot path).
// The reference's int64 row_ptr/col_idx and fp64 values arrive in HBM as
// uploaded; these kernels pack them into the row-record layout (layout.cuh)
// and build the CSC copy the residual monitor reads.
#include <cub/cub.cuh>

#include "kernels.h"

namespace ak {

// one warp per row: header {b, 1/nrm^2}, values (converted), int32 columns
template <class V>
__global__ void pack_records_kernel(const long long* __restrict__ row_ptr, const int32_t* __restrict__ col,
                                    const double* __restrict__ val, const double* __restrict__ row_norm,
                                    const double* __restrict__ b, long long m, const uint2* __restrict__ row_info,
                                    uint32_t stride16, unsigned char* __restrict__ rec) {
    const long long warp = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (warp >= m) return;
    const long long k0 = row_ptr[warp], len = row_ptr[warp + 1] - k0;
    unsigned char* base = rec + (row_info ? (size_t)row_info[warp].x * 16u : (size_t)warp * stride16 * 16u);
    if (lane == 0) {
        const double nrm = row_norm[warp];
        reinterpret_cast<double*>(base)[0] = b ? b[warp] : 0.0;
        reinterpret_cast<double*>(base)[1] = 1.0 / (nrm * nrm);
    }
    V* vals = reinterpret_cast<V*>(base + 16);
    int32_t* cols = reinterpret_cast<int32_t*>(base + 16 + (size_t)len * sizeof(V));
    for (long long k = lane; k < len; k += 32) {
        vals[k] = (V)val[k0 + k];
        cols[k] = (int32_t)col[k0 + k];
    }
    // zero the pad so records are deterministic bytes
    const size_t used = 16 + (size_t)len * (sizeof(V) + 4);
    const size_t total = (size_t)rec_size16((uint32_t)len, (int)sizeof(V)) * 16u;
    for (size_t p = used + lane; p < total; p += 32) base[p] = 0;
}

void launch_pack_records(const long long* row_ptr, const int32_t* col, const double* val, const double* row_norm,
                         const double* b, long long m, const uint2* row_info, uint32_t stride16, uint32_t, int precision,
                         unsigned char* rec, cudaStream_t s) {
    const unsigned blocks = (unsigned)((m * 32 + 255) / 256);
    if (precision == P_F64)
        pack_records_kernel<double><<<blocks, 256, 0, s>>>(row_ptr, col, val, row_norm, b, m, row_info, stride16, rec);
    else
        pack_records_kernel<float><<<blocks, 256, 0, s>>>(row_ptr, col, val, row_norm, b, m, row_info, stride16, rec);
}

__global__ void row_ids_kernel(const long long* __restrict__ row_ptr, long long m, int32_t* __restrict__ row_id) {
    const long long warp = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (warp >= m) return;
    for (long long k = row_ptr[warp] + lane; k < row_ptr[warp + 1]; k += 32) row_id[k] = (int32_t)warp;
}
void launch_row_ids(const long long* row_ptr, long long m, int32_t* row_id, cudaStream_t s) {
    row_ids_kernel<<<(unsigned)((m * 32 + 255) / 256), 256, 0, s>>>(row_ptr, m, row_id);
}

template <class V>
__global__ void gather_csc_kernel(const int32_t* __restrict__ perm, const int32_t* __restrict__ row_id,
                                  const double* __restrict__ val, long long nnz, int32_t* __restrict__ csc_row,
                                  V* __restrict__ csc_val) {
    for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < nnz; e += (long long)gridDim.x * blockDim.x) {
        const int32_t p = perm[e];
        csc_row[e] = row_id[p];
        csc_val[e] = (V)val[p];
    }
}
void launch_gather_csc(const int32_t* perm, const int32_t* row_id, const double* val, long long nnz, int precision,
                       int32_t* csc_row, void* csc_val, cudaStream_t s) {
    if (nnz == 0) return;
    const unsigned blocks = (unsigned)std::min<long long>((nnz + 255) / 256, 148 * 32);
    if (precision == P_F64)
        gather_csc_kernel<double><<<blocks, 256, 0, s>>>(perm, row_id, val, nnz, csc_row, static_cast<double*>(csc_val));
    else
        gather_csc_kernel<float><<<blocks, 256, 0, s>>>(perm, row_id, val, nnz, csc_row, static_cast<float*>(csc_val));
}

// col_ptr[j] = first position of column j in the column-sorted keys
__global__ void col_ptr_kernel(const int32_t* __restrict__ sorted_cols, long long nnz, long long n,
                               long long* __restrict__ col_ptr) {
    for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e <= nnz; e += (long long)gridDim.x * blockDim.x) {
        const long long cur = e < nnz ? sorted_cols[e] : n;
        const long long prev = e > 0 ? sorted_cols[e - 1] : -1;
        for (long long j = prev + 1; j <= cur; ++j) col_ptr[j] = e;
    }
}
void launch_col_hist(const int32_t* sorted_cols, long long nnz, long long n, long long* col_ptr, cudaStream_t s) {
    const unsigned blocks = (unsigned)std::min<long long>((nnz + 256) / 256, 148 * 32);
    col_ptr_kernel<<<blocks, 256, 0, s>>>(sorted_cols, nnz, n, col_ptr);
}

template <class X>
__global__ void x_init_kernel(const double* __restrict__ x0, X* __restrict__ x, long long n) {
    for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (long long)gridDim.x * blockDim.x)
        x[k] = x0 ? (X)x0[k] : X(0);
}
template <class X>
__global__ void x_export_kernel(const X* __restrict__ x, double* __restrict__ out, long long n) {
    for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (long long)gridDim.x * blockDim.x)
        out[k] = (double)x[k];
}
void launch_x_init(const double* x0, void* x, long long n, int precision, cudaStream_t s) {
    const unsigned blocks = (unsigned)std::min<long long>((n + 255) / 256, 148 * 8);
    if (precision == P_F32)
        x_init_kernel<float><<<blocks, 256, 0, s>>>(x0, static_cast<float*>(x), n);
    else
        x_init_kernel<double><<<blocks, 256, 0, s>>>(x0, static_cast<double*>(x), n);
}
void launch_x_export(const void* x, double* out, long long n, int precision, cudaStream_t s) {
    const unsigned blocks = (unsigned)std::min<long long>((n + 255) / 256, 148 * 8);
    if (precision == P_F32)
        x_export_kernel<float><<<blocks, 256, 0, s>>>(static_cast<const float*>(x), out, n);
    else
        x_export_kernel<double><<<blocks, 256, 0, s>>>(static_cast<const double*>(x), out, n);
}

__global__ void state_init_kernel(DevState* st, long long epochs_cap, long long interval, double target, int go) {
    st->epoch = 0;
    st->updates = 0;
    st->nrec = 0;
    st->epochs_cap = epochs_cap;
    st->interval = interval;
    st->target = target;
    st->stop = 0;
    st->status = 0;
    st->increments = 0;
    st->go = go;  // 0: set by the initial record's commit
    st->snap_valid[0] = st->snap_valid[1] = 0;
    st->stop_slot = -1;
    st->snap_ticket = st->mon_ticket = 0;
    st->slot_state[0] = st->slot_state[1] = 0;
    st->snap_arrive = st->snap_seq = st->snap_decided = 0;
    st->snap_target = st->mon_slot = -1;
    st->t0_ns = globaltimer_ns();
}
void launch_state_init(DevState* st, long long epochs_cap, long long interval, double target, cudaStream_t s, int go) {
    state_init_kernel<<<1, 1, 0, s>>>(st, epochs_cap, interval, target, go);
}

// max_t |x_t - x0_t - shadow_t|  (finish_instrument, parallel.cpp:94-106)
template <class X>
__global__ void instrument_check_kernel(const X* __restrict__ x, const double* __restrict__ x0,
                                        const X* __restrict__ shadow, long long n, unsigned long long* out) {
    double mx = 0.0;
    for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (long long)gridDim.x * blockDim.x) {
        const double d = fabs((double)x[k] - x0[k] - (double)shadow[k]);
        mx = d > mx ? d : mx;
    }
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(FULL, mx, o));
    if ((threadIdx.x & 31) == 0) atomicMax(out, __double_as_longlong(mx));
}
void launch_instrument_check(const void* x, const double* x0, const void* shadow, long long n, int precision,
                             double* out_max, cudaStream_t s) {
    cudaMemsetAsync(out_max, 0, sizeof(double), s);
    const unsigned blocks = (unsigned)std::min<long long>((n + 255) / 256, 148 * 8);
    auto* o = reinterpret_cast<unsigned long long*>(out_max);
    if (precision == P_F32)
        instrument_check_kernel<float><<<blocks, 256, 0, s>>>(static_cast<const float*>(x), x0,
                                                              static_cast<const float*>(shadow), n, o);
    else
        instrument_check_kernel<double><<<blocks, 256, 0, s>>>(static_cast<const double*>(x), x0,
                                                               static_cast<const double*>(shadow), n, o);
}

// Async audit: lhs_k = sum_j s_k(j) (x_j - x0_j) beside the workers'
// per-warp checksums of the increments they applied; out_max = max_k
// |lhs_k - sum_w part[w][k]| (the partials summed in a fixed order).
template <class X>
__global__ void audit_lhs_kernel(const X* __restrict__ x, const double* __restrict__ x0, long long n, double* lhs) {
    double cs[kAuditK] = {};
    for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (long long)gridDim.x * blockDim.x)
        audit_add(cs, (int)k, (double)x[k] - x0[k]);
#pragma unroll
    for (int q = 0; q < kAuditK; ++q) {
        const double v = warp_sum(cs[q]);
        if ((threadIdx.x & 31) == 0) atomicAdd(lhs + q, v);
    }
}
__global__ void __launch_bounds__(256) audit_final_kernel(const double* part, const unsigned long long* incr,
                                                          long long W, const double* lhs, double* out_max,
                                                          unsigned long long* out_incr) {
    __shared__ double red[kAuditK][256];
    __shared__ unsigned long long ired[256];
    double s[kAuditK] = {};
    unsigned long long ic = 0;
    for (long long w = threadIdx.x; w < W; w += 256) {
#pragma unroll
        for (int q = 0; q < kAuditK; ++q) s[q] += part[w * kAuditK + q];
        ic += incr[w];
    }
#pragma unroll
    for (int q = 0; q < kAuditK; ++q) red[q][threadIdx.x] = s[q];
    ired[threadIdx.x] = ic;
    __syncthreads();
    for (int o = 128; o > 0; o >>= 1) {
        if (threadIdx.x < o) {
#pragma unroll
            for (int q = 0; q < kAuditK; ++q) red[q][threadIdx.x] += red[q][threadIdx.x + o];
            ired[threadIdx.x] += ired[threadIdx.x + o];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        double mx = 0.0;
        for (int q = 0; q < kAuditK; ++q) mx = fmax(mx, fabs(lhs[q] - red[q][0]));
        *out_max = mx;
        *out_incr = ired[0];
    }
}
void launch_audit_check(const void* x, const double* x0, long long n, int precision, const double* part,
                        const unsigned long long* incr, long long W, double* lhs, double* out_max,
                        unsigned long long* out_incr, cudaStream_t s) {
    cudaMemsetAsync(lhs, 0, kAuditK * sizeof(double), s);
    const unsigned blocks = (unsigned)std::min<long long>((n + 255) / 256, 148 * 8);
    if (precision == P_F32)
        audit_lhs_kernel<float><<<blocks, 256, 0, s>>>(static_cast<const float*>(x), x0, n, lhs);
    else
        audit_lhs_kernel<double><<<blocks, 256, 0, s>>>(static_cast<const double*>(x), x0, n, lhs);
    audit_final_kernel<<<1, 256, 0, s>>>(part, incr, W, lhs, out_max, out_incr);
}

// CUB radix sort wrapper: stable sort of (col, nnz-index) pairs by column, so
// each column lists its rows ascending (the order multiply_transpose adds in).
size_t csc_sort_temp_bytes(long long nnz) {
    size_t bytes = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, bytes, (const int32_t*)nullptr, (int32_t*)nullptr,
                                    (const int32_t*)nullptr, (int32_t*)nullptr, (int)nnz);
    return bytes;
}
void csc_sort(void* temp, size_t temp_bytes, const int32_t* keys_in, int32_t* keys_out, const int32_t* vals_in,
              int32_t* vals_out, long long nnz, int end_bit, cudaStream_t s) {
    cub::DeviceRadixSort::SortPairs(temp, temp_bytes, keys_in, keys_out, vals_in, vals_out, (int)nnz, 0, end_bit, s);
}

__global__ void iota_cols_kernel(const int32_t* __restrict__ col, long long nnz, int32_t* __restrict__ keys,
                                 int32_t* __restrict__ idx) {
    for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < nnz; e += (long long)gridDim.x * blockDim.x) {
        keys[e] = (int32_t)col[e];
        idx[e] = (int32_t)e;
    }
}
void launch_iota_cols(const int32_t* col, long long nnz, int32_t* keys, int32_t* idx, cudaStream_t s) {
    if (nnz == 0) return;
    const unsigned blocks = (unsigned)std::min<long long>((nnz + 255) / 256, 148 * 32);
    iota_cols_kernel<<<blocks, 256, 0, s>>>(col, nnz, keys, idx);
}

// ---- SELL-32 column layout (see CscDev): one warp per group of 32 positions;
// position p holds column perm[p] (perm == nullptr: column p)
__global__ void sell_len_kernel(const long long* __restrict__ col_ptr, long long n, const int32_t* __restrict__ perm,
                                int32_t* __restrict__ col_len, long long* __restrict__ grp_size) {
    const long long g = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    const long long groups = (n + 31) / 32;
    if (g >= groups) return;
    const long long p = g * 32 + lane;
    const long long j = p < n ? (perm ? (long long)perm[p] : p) : 0;
    const int len = p < n ? (int)(col_ptr[j + 1] - col_ptr[j]) : 0;
    if (p < n) col_len[p] = len;
    int mx = len;
    for (int o = 16; o > 0; o >>= 1) mx = max(mx, __shfl_xor_sync(FULL, mx, o));
    if (lane == 0) grp_size[g] = 32ll * mx;
}
void launch_sell_len(const long long* col_ptr, long long n, int32_t* col_len, long long* grp_size, cudaStream_t s,
                     const int32_t* perm) {
    const long long groups = (n + 31) / 32;
    sell_len_kernel<<<(unsigned)((groups * 32 + 255) / 256), 256, 0, s>>>(col_ptr, n, perm, col_len, grp_size);
}

// sigma-sorting of the columns (SELL-C-sigma with sigma = n): positions in
// order of decreasing length, ties in column order (a stable radix sort), so
// the 32 columns of a group have nearly equal lengths and the padding of the
// column copy (each group padded to its longest column) all but disappears
__global__ void col_len_iota_kernel(const long long* __restrict__ col_ptr, long long n, int32_t* __restrict__ len,
                                    int32_t* __restrict__ iota) {
    for (long long j = (long long)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (long long)gridDim.x * blockDim.x) {
        len[j] = (int32_t)(col_ptr[j + 1] - col_ptr[j]);
        iota[j] = (int32_t)j;
    }
}
size_t sigma_sort_temp_bytes(long long n) {
    size_t bytes = 0;
    cub::DeviceRadixSort::SortPairsDescending(nullptr, bytes, (const int32_t*)nullptr, (int32_t*)nullptr,
                                              (const int32_t*)nullptr, (int32_t*)nullptr, (int)n);
    return bytes;
}
void launch_sigma_sort(const long long* col_ptr, long long n, void* temp, size_t temp_bytes, int32_t* len_tmp,
                       int32_t* len_sorted, int32_t* iota_tmp, int32_t* perm, cudaStream_t s) {
    if (n == 0) return;
    const unsigned blocks = (unsigned)std::min<long long>((n + 255) / 256, 148 * 8);
    col_len_iota_kernel<<<blocks, 256, 0, s>>>(col_ptr, n, len_tmp, iota_tmp);
    cub::DeviceRadixSort::SortPairsDescending(temp, temp_bytes, len_tmp, len_sorted, iota_tmp, perm, (int)n, 0, 32, s);
}

template <class V>
__global__ void sell_scatter_kernel(const long long* __restrict__ ptr, const int32_t* __restrict__ src_idx,
                                    const double* __restrict__ src_val, const int32_t* __restrict__ len_arr,
                                    const long long* __restrict__ grp_off, long long n, const int32_t* __restrict__ perm,
                                    int32_t* __restrict__ dst_idx, V* __restrict__ dst_val) {
    const long long g = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    const long long p = g * 32 + lane;
    if (g >= (n + 31) / 32 || p >= n) return;
    const long long src = ptr[perm ? (long long)perm[p] : p], dst = grp_off[g] + lane;
    const int len = len_arr[p];
    for (int t = 0; t < len; ++t) {
        dst_idx[dst + 32ll * t] = src_idx[src + t];
        dst_val[dst + 32ll * t] = (V)src_val[src + t];
    }
}
// src_val is fp64 (the reference's values); dst_val gets the device precision
void launch_sell_scatter(const long long* ptr, const int32_t* src_idx, const void* src_val, const int32_t* len_arr,
                         const long long* grp_off, long long n, int precision, int32_t* dst_idx, void* dst_val,
                         cudaStream_t s, const int32_t* perm) {
    const long long groups = (n + 31) / 32;
    const unsigned blocks = (unsigned)((groups * 32 + 255) / 256);
    const double* sv = static_cast<const double*>(src_val);
    if (precision == P_F64)
        sell_scatter_kernel<double><<<blocks, 256, 0, s>>>(ptr, src_idx, sv, len_arr, grp_off, n, perm, dst_idx,
                                                           static_cast<double*>(dst_val));
    else
        sell_scatter_kernel<float><<<blocks, 256, 0, s>>>(ptr, src_idx, sv, len_arr, grp_off, n, perm, dst_idx,
                                                          static_cast<float*>(dst_val));
}

size_t scan_temp_bytes(long long count) {
    size_t bytes = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, bytes, (const long long*)nullptr, (long long*)nullptr, (int)count);
    return bytes;
}
void exclusive_scan(void* temp, size_t temp_bytes, const long long* in, long long* out, long long count,
                    cudaStream_t s) {
    cub::DeviceScan::ExclusiveSum(temp, temp_bytes, in, out, (int)count, s);
}

__global__ void set_rhs_kernel(Layout L, const double* __restrict__ b) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < L.m; i += (long long)gridDim.x * blockDim.x) {
        const RowRef r = row_ref(L, i);
        *reinterpret_cast<double*>(const_cast<unsigned char*>(r.base)) = b[i];
    }
}
void launch_set_rhs(const Layout& L, const double* b, cudaStream_t s) {
    const unsigned blocks = (unsigned)std::min<long long>((L.m + 255) / 256, 148 * 8);
    set_rhs_kernel<<<blocks, 256, 0, s>>>(L, b);
}

}  // namespace ak

namespace ak {

// ---- overlapped async solve: epoch-boundary snapshot of x for the monitor
// stream, then (last block to finish) the coordinator state advance. Every
// block reads `go` before taking its ticket and only the last block changes
// it, so a whole epoch is either run and counted or skipped.
template <class X>
__global__ void snapshot_kernel(DevState* st, const X* __restrict__ x, X* __restrict__ xs, long long n, int slot,
                                long long m, int advance) {
    __shared__ int copy;
    __shared__ bool last;
    // advance = 0: boundary 0 (x0), before any worker ran (go is not set yet)
    if (threadIdx.x == 0) copy = (advance ? st->go : 1) && !st->stop;  // after a stop the deciding snapshot must survive
    __syncthreads();
    if (copy)
        for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < n;
             k += (long long)gridDim.x * blockDim.x)
            xs[k] = __ldcg(x + k);
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) last = atomicAdd(&st->snap_ticket, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!last || threadIdx.x != 0) return;
    st->snap_ticket = 0;
    if (st->stop) {  // stopped: the slots are frozen, no further epochs
        st->go = 0;
        return;
    }
    if (advance ? st->go : 1) {
        if (advance) {
            const long long sp = chunk_span(st);
            st->epoch += sp;
            st->updates += sp * m;
        }
        st->snap_epoch[slot] = st->epoch;
        st->snap_updates[slot] = st->updates;
        st->snap_valid[slot] = 1;
    } else {
        st->snap_valid[slot] = 0;
    }
    st->go = (!st->stop && st->epoch < st->epochs_cap) ? 1 : 0;
}

// Decoupled snapshot (no back-pressure from the monitor): the first block to
// arrive takes a free slot if there is one and publishes the choice; the
// epoch is counted either way, and a skipped boundary gets no record — the
// reference's coordinator likewise reports only the latest boundary it
// catches (parallel.cpp:388-399).
template <class X>
__global__ void snapshot_dyn_kernel(DevState* st, const X* __restrict__ x, X* __restrict__ xs0, X* __restrict__ xs1,
                                    long long n, long long m, int advance) {
    __shared__ int target;
    __shared__ bool last;
    if (threadIdx.x == 0) {
        const unsigned seq = *reinterpret_cast<volatile unsigned*>(&st->snap_seq);
        if (atomicAdd(&st->snap_arrive, 1u) == 0) {
            int t = -1;
            if ((advance ? st->go : 1) && !st->stop)
                for (int q = 0; q < 2 && t < 0; ++q)
                    if (atomicCAS(&st->slot_state[q], 0, 1) == 0) t = q;
            st->snap_target = t;
            __threadfence();
            atomicExch(&st->snap_decided, seq + 1u);
        } else {
            while (*reinterpret_cast<volatile unsigned*>(&st->snap_decided) != seq + 1u) __nanosleep(64);
            __threadfence();
        }
        target = *reinterpret_cast<volatile int*>(&st->snap_target);
    }
    __syncthreads();
    if (target >= 0) {
        X* xs = target == 0 ? xs0 : xs1;
        for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < n;
             k += (long long)gridDim.x * blockDim.x)
            xs[k] = __ldcg(x + k);
    }
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) last = atomicAdd(&st->snap_ticket, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!last || threadIdx.x != 0) return;
    st->snap_ticket = 0;
    st->snap_arrive = 0;
    st->snap_seq += 1u;
    if ((advance ? st->go : 1) && !st->stop) {
        if (advance) {
            const long long sp = chunk_span(st);
            st->epoch += sp;
            st->updates += sp * m;
        }
        if (target >= 0) {
            st->snap_epoch[target] = st->epoch;
            st->snap_updates[target] = st->updates;
            st->snap_valid[target] = 1;
            __threadfence();
            atomicExch(&st->slot_state[target], 2);
        }
    } else if (target >= 0) {
        atomicExch(&st->slot_state[target], 0);
    }
    st->go = (!st->stop && st->epoch < st->epochs_cap) ? 1 : 0;
}

// monitor stream: claim the oldest filled snapshot (or none) for the passes that follow
__global__ void claim_kernel(DevState* st) {
    int best = -1;
    long long be = 0;
    for (int q = 0; q < 2; ++q)
        if (atomicAdd(&st->slot_state[q], 0) == 2 && (best < 0 || st->snap_epoch[q] < be)) {
            best = q;
            be = st->snap_epoch[q];
        }
    if (best >= 0) atomicExch(&st->slot_state[best], 3);
    st->mon_slot = st->stop ? -1 : best;
}

void launch_snapshot_dyn(DevState* st, const void* x, void* xs0, void* xs1, long long n, int precision, long long m,
                         cudaStream_t s, int advance) {
    const unsigned blocks = (unsigned)std::min<long long>((n + 255) / 256, 148 * 4);
    if (precision == P_F32)
        snapshot_dyn_kernel<float><<<blocks, 256, 0, s>>>(st, static_cast<const float*>(x), static_cast<float*>(xs0),
                                                          static_cast<float*>(xs1), n, m, advance);
    else
        snapshot_dyn_kernel<double><<<blocks, 256, 0, s>>>(st, static_cast<const double*>(x),
                                                           static_cast<double*>(xs0), static_cast<double*>(xs1), n, m,
                                                           advance);
}

void launch_claim(DevState* st, cudaStream_t s) { claim_kernel<<<1, 1, 0, s>>>(st); }

// end of an overlapped solve: return the snapshot that decided the stop
template <class X>
__global__ void restore_kernel(DevState* st, X* __restrict__ x, const X* __restrict__ xs0, const X* __restrict__ xs1,
                               long long n) {
    const int slot = st->stop_slot;
    if (slot < 0) return;
    const X* src = slot == 0 ? xs0 : xs1;
    for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (long long)gridDim.x * blockDim.x)
        x[k] = src[k];
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        st->epoch = st->stop_epoch;
        st->updates = st->stop_updates;
    }
}

void launch_restore(DevState* st, void* x, const void* xs0, const void* xs1, long long n, int precision,
                    cudaStream_t s) {
    const unsigned blocks = (unsigned)std::min<long long>((n + 255) / 256, 148 * 4);
    if (precision == P_F32)
        restore_kernel<float><<<blocks, 256, 0, s>>>(st, static_cast<float*>(x), static_cast<const float*>(xs0),
                                                     static_cast<const float*>(xs1), n);
    else
        restore_kernel<double><<<blocks, 256, 0, s>>>(st, static_cast<double*>(x), static_cast<const double*>(xs0),
                                                      static_cast<const double*>(xs1), n);
}

void launch_snapshot(const DevState* st, const void* x, void* xs, long long n, int precision, int slot, DevState* stw,
                     long long m, cudaStream_t s, int advance) {
    (void)st;
    const unsigned blocks = (unsigned)std::min<long long>((n + 255) / 256, 148 * 4);
    if (precision == P_F32)
        snapshot_kernel<float><<<blocks, 256, 0, s>>>(stw, static_cast<const float*>(x), static_cast<float*>(xs), n,
                                                      slot, m, advance);
    else
        snapshot_kernel<double><<<blocks, 256, 0, s>>>(stw, static_cast<const double*>(x), static_cast<double*>(xs),
                                                       n, slot, m, advance);
}

}  // namespace ak
