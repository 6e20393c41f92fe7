// Launch wrappers of the sm_100a kernels (host-callable, no CUDA types
// beyond cudaStream_t). Implemented in worker.cu, det.cu, monitor.cu, pack.cu.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "layout.cuh"

namespace ak {

// SM count of the calling thread's current device, cached per device ordinal
// (runtime.cu); a process may drive several GPUs.
int current_sm_count();


enum Precision { P_F64 = 0, P_F32 = 1, P_F32X64 = 2 };
enum Sampling { S_UNIFORM = 0, S_SLICE = 1, S_ALIAS = 2 };

struct AliasEntry {
    float prob;
    int32_t alias;
};

// ---- K2: asynchronous Hogwild worker (one warp = one AsyRK worker)
struct WorkerArgs {
    Layout L;
    void* x;                      // X[n]
    double* audit;                // instrumented run: per-warp checksums [W][kAuditK], or nullptr
    const AliasEntry* alias;      // m entries (S_ALIAS)
    DevState* st;
    unsigned long long* increments;  // instrumented run: per-warp increment counts [W]
    long long W;                  // worker warps
    double gamma;
    uint32_t key0, key1;          // seed
    int sampling;
    int full_row;
    long long epoch0, span0;      // span0 > 0: this launch runs epochs [epoch0, epoch0 + span0) (host-scheduled
                                  // solves); span0 = 0: the epoch / span come from st (chunk_span)
};
int worker_elems_per_lane(uint32_t max_len);  // 1, 2, 4 or 0 (looped)
// the workers' row draws for positions [0, per_warp) of every warp (tests)
void launch_sample_rows(const WorkerArgs& a, long long epoch, long long per_warp, int32_t* out, cudaStream_t s);
void launch_worker(const WorkerArgs& a, int precision, int E, cudaStream_t s);
int worker_max_resident_warps(int precision, int E, int full_row);

// ---- K1: deterministic single worker consuming a host-generated sequence
struct DetArgs {
    Layout L;
    const double* row_norm;       // reference row norms (coefficient exactness)
    double* x;
    double* shadow;               // or nullptr
    const int32_t* seq;           // rows of this chunk, in order
    const int32_t* picks;         // single_component picks, or nullptr
    long long count;              // rows in this chunk (0 = take span*m from st)
    DevState* st;
    double gamma;
    int full_row;
    int x_in_smem;
    const int32_t* need;          // per (event, nonzero): earlier events of the chunk on that column
    const long long* flat_off;    // per event: offset of its nonzeros in need (nullptr: q * uniform_len)
    const int32_t* ev_col;        // per (event, nonzero): column, in event order (prepass)
    double* ev_val;               // per (event, nonzero): value, in event order (prepass)
    double* ev_b;                 // per event: b_i
    double* ev_nn;                // per event: row_norm_i^2 (rounded, as the reference forms it)
    double* ev_rcp;               // per event: RN(1 / ev_nn), the division's reciprocal
    long long* dbg;               // optional per-event phase timestamps (diagnostics)
    int poll_ns;                  // dataflow polling back-off (0: spin)
    uint32_t max_len;             // longest row (picks the dataflow kernel's elements per lane)
    // deterministic multi-RHS (asyrk_system_rk_solve_multi): ncols > 1 runs one
    // CTA per right-hand side over the same event sequence / prepass; column c's
    // iterate is x + c * n and its b is b_cols + c * m (b_cols null: one column,
    // b from the records)
    int ncols;
    const double* b_cols;
    int reassoc;                  // 1: warp-tree dot, reciprocal coefficient, fused update (tolerance mode)
};
void launch_det(const DetArgs& a, int n_smem_x, cudaStream_t s);
bool det_fits_smem(long long n);
struct DetPrep {
    int32_t *keys, *vals, *keys_s, *vals_s, *start;
    double *ev_val, *ev_b, *ev_nn, *ev_rcp;
    void* temp;
    size_t temp_bytes;
};
size_t det_prepare_temp_bytes(long long total);
// fills a.need for the chunk (total = number of (event, nonzero) pairs)
void launch_det_prepare(const DetArgs& a, const DetPrep& p, long long total, cudaStream_t s);

// ---- K3: residual monitor r = Ax - b, g = A^T r, dist = ||x - x*||^2
// Columns of A in SELL-32 order: the 32 positions of group g interleave their
// entries, entry t of position 32g+l at grp_off[g] + 32t + l (rows ascending
// within each column); slots past a column's length are padding. Position p
// holds column perm[p]: the column copy is sigma-sorted (decreasing length,
// so a group pads to almost nothing); perm == nullptr (the row copy) is the
// identity. Consumers walk positions and write per-column results at perm[p].
struct CscDev {
    const long long* grp_off;     // ceil(n/32)+1
    const int32_t* col_len;       // n, by position
    const int32_t* row;           // padded
    const void* val;              // padded (V)
    const int32_t* perm = nullptr;  // position -> column, or nullptr
    __device__ __forceinline__ long long col(long long p) const { return perm ? (long long)__ldg(perm + p) : p; }
};
struct MonitorArgs {
    Layout L;
    CscDev csc;
    const void* x;                // X[n]
    const double* x_star;         // or nullptr
    double* r;                    // m
    double* g;                    // n
    double* part;                 // per-block partials [3][nblocks]
    DevRecord* rec;               // trace records
    long long rec_cap;
    DevState* st;
    int* host_flag;               // mapped pinned: stop seen by the host
    int exact;                    // 1: reference summation order (bitwise)
    CscDev rows;                  // SELL-32 rows of A (pass 1)
    const double* b;              // m
    int slot;                     // >= 0: record the epoch-boundary snapshot in this slot (overlapped solve);
                                  // kDynSlot: the slot the monitor stream claimed (st->mon_slot), x / x_alt
    const void* x_alt;            // kDynSlot: the snapshot buffer of slot 1 (x is slot 0's)
    int force;                    // 1: run even after stop (the final exact record); replaces a same-epoch record
    int advance;                  // 0: initial record, 1: after a chunk
    long long m_rows;
    long long set_epoch;          // >= 0: the boundary this record is taken at (host-scheduled solves:
                                  // st->epoch = set_epoch, st->updates = set_epoch * m_rows); -1: unused
    HostMirror* mirror;           // or nullptr: the record's decision inputs for the host
    double* col_out;              // exact mode: write {r_sq, grad_sq, dist_sq} here instead of recording
};
void launch_monitor(const MonitorArgs& a, int precision, cudaStream_t s);
// deterministic multi-RHS record: sums the per-column exact sums colres[c][3]
// in column order, then records / decides like the single-RHS finalize
void launch_multi_commit(const MonitorArgs& a, const double* colres, int ncols, cudaStream_t s);
// overlapped solves: copy x into snapshot slot xs (if the epoch ran) and
// advance the coordinator state (epoch, updates, slot meta, next go);
// advance = 0 takes boundary 0 (x0, before the first workers; sets go)
void launch_snapshot(const DevState* st, const void* x, void* xs, long long n, int precision, int slot, DevState* stw,
                     long long m, cudaStream_t s, int advance = 1);
// decoupled variant: a free slot or none (no record for that boundary); then the
// monitor stream claims the oldest filled slot (MonitorArgs::slot = kDynSlot)
void launch_snapshot_dyn(DevState* st, const void* x, void* xs0, void* xs1, long long n, int precision, long long m,
                         cudaStream_t s, int advance = 1);
void launch_claim(DevState* st, cudaStream_t s);
constexpr int kDynSlot = 2;
// end of an overlapped solve: x, epoch and updates back to the snapshot whose
// record decided the stop (no-op when the stop came from the epoch cap in-stream)
void launch_restore(DevState* st, void* x, const void* xs0, const void* xs1, long long n, int precision,
                    cudaStream_t s);

// ---- K2b/K3b: multi-right-hand-side worker and monitor (mrhs.cu)
struct MrhsArgs {
    Layout L;                     // fp32 row records (b unused)
    float* X;                     // n x KL row-major
    const float* B;               // m x KL row-major
    float* R;                     // m x KL residual scratch (CSC monitor)
    float* G;                     // n x KL: G = A^T R scattered by the rows pass (scatter monitor), or nullptr
    const double* Xstar;          // n x KL or nullptr
    const long long* col_ptr;     // plain CSC for G = A^T R
    const int32_t* csc_row;
    const double* csc_val;
    double* part;                 // block partials
    double* norms;                // {r_sq, g_sq, d_sq} of this shard (all-reduce target)
    DevRecord* rec;
    long long rec_cap;
    DevState* st;
    int* host_flag;
    long long W;
    double gamma;
    uint32_t key0, key1;
    int KL;
    int sampling;                 // S_UNIFORM (with replacement) or S_SLICE
    long long epoch0, span0;      // this worker launch runs epochs [epoch0, epoch0 + span0)
    HostMirror* mirror;           // latest record for the host-driven schedule
    uint32_t max_len;             // longest row (> 32: the looped worker)
};
bool mrhs_supported_kl(long long kl);
int32_t xside_mrhs_on_buffer(float* X, int64_t n, int32_t theta, int32_t kl, int32_t warps, int64_t proj_per_warp,
                                  cudaStream_t stream, double* proj_per_s, double* kernel_ms);  // an asyrk_status
bool mrhs_rowpar(int kl);  // the row-parallel worker runs at this width (KL 8 / 16 / 32 by default)
int mrhs_max_resident_warps(int kl, uint32_t max_len);  // co-resident worker warps of the worker used
int mrhs_row_blocks(long long m);
int mrhs_col_blocks(long long n);
void launch_mrhs_worker(const MrhsArgs& a, cudaStream_t s);
void launch_mrhs_monitor(const MrhsArgs& a, cudaStream_t s);
// record at boundary set_epoch (-1: the initial state) + stop decision
void launch_mrhs_commit(const MrhsArgs& a, long long set_epoch, cudaStream_t s);

// ---- K4: power iteration building blocks (stats.cpp:15-50)
void launch_spmv_rows(const CscDev& R, int precision, long long m, const double* v, double* out, cudaStream_t s);
// SELL-32 columns from a column-sorted CSC: lengths + group sizes, then scatter
// (perm: position -> column, or nullptr for the identity)
void launch_sell_len(const long long* col_ptr, long long n, int32_t* col_len, long long* grp_size, cudaStream_t s,
                     const int32_t* perm = nullptr);
void launch_sell_scatter(const long long* col_ptr, const int32_t* src_row, const void* src_val, const int32_t* col_len,
                         const long long* grp_off, long long n, int precision, int32_t* dst_row, void* dst_val,
                         cudaStream_t s, const int32_t* perm = nullptr);
// perm = the columns by decreasing length (stable); len_tmp / len_sorted / iota_tmp: n-long scratch
size_t sigma_sort_temp_bytes(long long n);
void launch_sigma_sort(const long long* col_ptr, long long n, void* temp, size_t temp_bytes, int32_t* len_tmp,
                       int32_t* len_sorted, int32_t* iota_tmp, int32_t* perm, cudaStream_t s);
size_t scan_temp_bytes(long long count);
void exclusive_scan(void* temp, size_t temp_bytes, const long long* in, long long* out, long long count, cudaStream_t s);
void launch_spmv_cols(const CscDev& C, int precision, long long n, const double* r, double* out,
                      cudaStream_t s);
// dot/norm with a fixed-order tree; result in *out (device)
void launch_dot(const double* a, const double* b, long long n, double* scratch, double* out, cudaStream_t s);
void launch_power_update(double* v, const double* w, const double* wn_dot, long long n, cudaStream_t s);

// ---- K5: compute_stats (stats.cu)
struct StatsDev {
    long long zero_col;                 // first empty column (LLONG_MAX: none)
    long long nu;                       // max column count
    long long max_w;                    // max over columns of the sum of its rows' lengths
    unsigned long long l_max_bits, alpha_bits, l_res_bits;  // non-negative doubles as bits
    double frob_sq;
};
void launch_stats_cols(const CscDev& C, long long n, const int32_t* row_len, double* col_sq, double* col_norm,
                       StatsDev* out, cudaStream_t s);
// alpha, frob_sq, l_res; scratch: global hash tables when a table exceeds shared memory
void launch_stats_rest(const CscDev& C, const CscDev& R, long long m, long long n, const double* col_sq,
                       const double* col_norm, long long max_w, unsigned char* scratch, size_t scratch_bytes,
                       StatsDev* out, cudaStream_t s);
int stats_table_cap(long long max_w, long long n);

// ---- K6: batched bounded-delay simulator (delay.cu)
struct SimEventDev {
    long long j, i, t, k;
    double step;
};
struct SimArgs {
    Layout L;                      // fp64 row records (lane 0's contiguous row walks)
    CscDev R;                      // SELL-32 rows (fp64; the residual passes)
    CscDev C;                      // SELL-32 columns (fp64, rows ascending; the residual passes)
    const long long* col_ptr;      // plain CSC (rows ascending): lane 0's LiveResidual bumps
    const int32_t* csc_row;
    const double* csc_val;
    const double* row_norm;        // m
    const double* b;               // m
    const double* x0;              // n
    long long m, n;
    double gamma;
    long long tau;
    int delay_kind;                // 0 fixed, 1 uniform_random, 2 max_staleness
    int variant;                   // 0 single_component, 1 full_row
    long long iterations;
    unsigned long long seed0;      // run r uses seed0 + r
    long long probe_every;
    int probe_r_sq;
    const double* xdist;           // n: the projector's solution point (dist_sq records / probes), or nullptr
    double* probe_d;               // runs x probe_stride dist probes, or nullptr
    long long max_events;
    long long runs;
    double* work;                  // runs x work_stride doubles (sim_work_doubles)
    long long work_stride;
    double* probe;                 // runs x probe_stride, or nullptr
    long long probe_stride;
    DevRecord* rec;                // run 0's epoch records, or nullptr
    long long rec_cap;
    long long *nrec, *nev, *nprobe;  // run 0 counts, or nullptr
    SimEventDev* ev;               // run 0's events, or nullptr
    int* status;                   // per run: 0 or ASYRK_E_NonFinite
    long long* fail_updates;       // per run
    long long hot;                 // set by launch_sim: doubles of x | ring | LiveResidual r
    int smem_state;                // set by launch_sim: hot state in shared memory
};
size_t sim_work_doubles(long long m, long long n, long long tau);
void launch_sim(const SimArgs& a, bool cta_per_run, cudaStream_t s);
void launch_sim_mean(const double* probe, long long probe_stride, long long runs, long long K, double* mean,
                     double* ratios, cudaStream_t s);

// ---- K0: packing
void launch_pack_records(const long long* row_ptr, const int32_t* col, const double* val,
                         const double* row_norm, const double* b, long long m, const uint2* row_info,
                         uint32_t stride16, uint32_t uniform_len, int precision, unsigned char* rec,
                         cudaStream_t s);
void launch_row_ids(const long long* row_ptr, long long m, int32_t* row_id, cudaStream_t s);
void launch_gather_csc(const int32_t* perm, const int32_t* row_id, const double* val, long long nnz,
                       int precision, int32_t* csc_row, void* csc_val, cudaStream_t s);
void launch_col_hist(const int32_t* sorted_cols, long long nnz, long long n, long long* col_ptr,
                     cudaStream_t s);
void launch_x_init(const double* x0, void* x, long long n, int precision, cudaStream_t s);
void launch_x_export(const void* x, double* out, long long n, int precision, cudaStream_t s);
void launch_state_init(DevState* st, long long epochs_cap, long long interval, double target,
                       cudaStream_t s, int go = 0);
// async audit (layout.cuh kAuditK checksums): part = the workers' per-warp
// checksums [W][kAuditK], incr = their per-warp increment counts [W]; lhs =
// kAuditK scratch doubles; writes max_k |lhs_k - sum_w part[w][k]| to out_max
// and sum_w incr[w] to out_incr
void launch_audit_check(const void* x, const double* x0, long long n, int precision, const double* part,
                        const unsigned long long* incr, long long W, double* lhs, double* out_max,
                        unsigned long long* out_incr, cudaStream_t s);
void launch_instrument_check(const void* x, const double* x0, const void* shadow, long long n,
                             int precision, double* out_max, cudaStream_t s);

}  // namespace ak

namespace ak {
size_t csc_sort_temp_bytes(long long nnz);
void csc_sort(void* temp, size_t temp_bytes, const int32_t* keys_in, int32_t* keys_out, const int32_t* vals_in,
              int32_t* vals_out, long long nnz, int end_bit, cudaStream_t s);
void launch_iota_cols(const int32_t* col, long long nnz, int32_t* keys, int32_t* idx, cudaStream_t s);
int monitor_row_blocks(long long m);
int monitor_col_blocks(long long n);
void launch_set_rhs(const Layout& L, const double* b, cudaStream_t s);
}  // namespace ak
