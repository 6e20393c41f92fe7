// Dense thin SVD on the device — replaces the Eigen BDCSVD of the reference's
// desk-scale oracle (ref/src/dense.cpp:27-50: decompose, spectrum_of), which
// feeds compute_stats(exact_spectral) (stats.cpp:136-140), lsq_solve's sigma_r
// (lsq.cpp:118-129) and SolutionProjector (dense.cpp:70-117).
//
// One-sided (Hestenes) Jacobi on G = A (m >= n) or G = A^T (m < n): G is
// L x k column-major, k = min(m, n). A sweep visits every column pair once in
// k-1 round-robin steps of k/2 disjoint pairs (circle method); one CTA owns a
// pair, forms a = |g_p|^2, b = |g_q|^2, c = g_p.g_q in one pass and applies the
// rotation that makes g_p, g_q orthogonal (Rutishauser's formulas), also to
// the k x k accumulator W when singular vectors are wanted. Sweeps repeat
// until no pair needs a rotation (|c| <= tol sqrt(ab), tol = sqrt(L) eps as
// in LAPACK dgesvj). Then sigma_j = |g_j|, U_G = g_j / sigma_j, and
//   m >= n: A = U_G S W^T      m < n: A = W S U_G^T.
// One-sided Jacobi computes small singular values to high relative accuracy,
// so the rank cutoff 1e-10 sigma_max (dense.cpp:12,36-40) separates the
// numerical null space the same way.
//
// HBM/L2: for k <= 2048 columns of a 4M-cell matrix, G (32 MB) and W stay
// resident in the 126 MB L2 across a sweep's steps; each step streams G once.
#include <algorithm>
#include <cmath>
#include <numeric>
#include <vector>

#include "../../include/asyrk_dense.h"
#include "capi_common.h"
#include "kernels.h"

namespace ak {

constexpr int kJT = 256;

__device__ __forceinline__ int circle_elem(int pos, int step, int K) {
    return pos == 0 ? 0 : 1 + (pos - 1 + step) % (K - 1);
}

__device__ __forceinline__ void block_sum3(double& a, double& b, double& c, double* sh) {
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        a += __shfl_xor_sync(FULL, a, o);
        b += __shfl_xor_sync(FULL, b, o);
        c += __shfl_xor_sync(FULL, c, o);
    }
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0) {
        sh[3 * w] = a;
        sh[3 * w + 1] = b;
        sh[3 * w + 2] = c;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double s0 = 0, s1 = 0, s2 = 0;
        for (int k = 0; k < kJT / 32; ++k) {
            s0 += sh[3 * k];
            s1 += sh[3 * k + 1];
            s2 += sh[3 * k + 2];
        }
        sh[0] = s0;
        sh[1] = s1;
        sh[2] = s2;
    }
    __syncthreads();
    a = sh[0];
    b = sh[1];
    c = sh[2];
}

__global__ void __launch_bounds__(kJT) jacobi_step_kernel(double* __restrict__ G, long long L, double* __restrict__ W,
                                                          int k, int K, int step, double tol,
                                                          unsigned long long* rotations) {
    __shared__ double sh[3 * (kJT / 32)];
    __shared__ double cs[2];
    int p = circle_elem(blockIdx.x, step, K), q = circle_elem(K - 1 - blockIdx.x, step, K);
    if (p >= k || q >= k) return;
    if (p > q) {
        const int t = p;
        p = q;
        q = t;
    }
    double* gp = G + (long long)p * L;
    double* gq = G + (long long)q * L;
    double a = 0.0, b = 0.0, c = 0.0;
    for (long long r = threadIdx.x; r < L; r += kJT) {
        const double x = gp[r], y = gq[r];
        a = fma(x, x, a);
        b = fma(y, y, b);
        c = fma(x, y, c);
    }
    block_sum3(a, b, c, sh);
    if (!(fabs(c) > tol * sqrt(a) * sqrt(b))) return;  // already orthogonal (or a zero column)
    if (threadIdx.x == 0) {
        const double zeta = (b - a) / (2.0 * c);
        const double t = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + hypot(1.0, zeta));
        const double cc = 1.0 / sqrt(fma(t, t, 1.0));
        cs[0] = cc;
        cs[1] = cc * t;
        atomicAdd(rotations, 1ull);
    }
    __syncthreads();
    const double cc = cs[0], sn = cs[1];
    for (long long r = threadIdx.x; r < L; r += kJT) {
        const double x = gp[r], y = gq[r];
        gp[r] = fma(cc, x, -sn * y);
        gq[r] = fma(sn, x, cc * y);
    }
    if (W) {
        double* wp = W + (long long)p * k;
        double* wq = W + (long long)q * k;
        for (int r = threadIdx.x; r < k; r += kJT) {
            const double x = wp[r], y = wq[r];
            wp[r] = fma(cc, x, -sn * y);
            wq[r] = fma(sn, x, cc * y);
        }
    }
}

__global__ void __launch_bounds__(kJT) column_norm_kernel(const double* __restrict__ G, long long L,
                                                          double* __restrict__ sigma) {
    __shared__ double sh[3 * (kJT / 32)];
    const double* g = G + (long long)blockIdx.x * L;
    double a = 0.0, z0 = 0.0, z1 = 0.0;
    for (long long r = threadIdx.x; r < L; r += kJT) a = fma(g[r], g[r], a);
    block_sum3(a, z0, z1, sh);
    if (threadIdx.x == 0) sigma[blockIdx.x] = sqrt(a);
}

__global__ void identity_kernel(double* W, int k) {
    const long long total = (long long)k * k;
    for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (long long)gridDim.x * blockDim.x)
        W[e] = (e / k == e % k) ? 1.0 : 0.0;
}

namespace {

constexpr int kMaxSweeps = 60;

asyrk_status svd_impl(const asyrk_csr_view* A, int64_t max_cells, double* sigma_out, double* U, double* V,
                      int32_t* rank_out, int32_t* sweeps_out) {
    if (!A || !A->row_ptr || !A->col_idx || !A->values || !sigma_out)
        return fail(ASYRK_E_InvalidArgument, "dense_svd: null argument");
    const int64_t m = A->m, n = A->n;
    if (m < 1 || n < 1) return fail(ASYRK_E_InvalidArgument, "dense_svd: empty matrix");
    if (max_cells <= 0) max_cells = ASYRK_DENSE_DEVICE_CAP;
    if ((double)m * (double)n > (double)max_cells)
        return fail(ASYRK_E_TooLarge, "dense SVD capped at " + std::to_string(max_cells) + " elements (m*n = " +
                                          std::to_string((double)m * (double)n) + ")");
    const bool tall = m >= n;
    const long long L = tall ? m : n;
    const int k = (int)(tall ? n : m);
    const bool want_vec = U || V;

    // dense G on the host (to_dense order, dense.cpp:121-128), one upload
    std::vector<double> Gh((size_t)L * k, 0.0);
    for (int64_t i = 0; i < m; ++i)
        for (int64_t e = A->row_ptr[i]; e < A->row_ptr[i + 1]; ++e) {
            const int64_t j = A->col_idx[e];
            if (j < 0 || j >= n) return fail(ASYRK_E_IndexOutOfRange, "dense_svd: column index out of range");
            Gh[tall ? (size_t)(i + j * m) : (size_t)(j + i * n)] = A->values[e];
        }

    cudaStream_t s;
    CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    struct StreamGuard {
        cudaStream_t s;
        ~StreamGuard() { cudaStreamDestroy(s); }
    } sg{s};
    AllocStream as(s);
    double* G = dalloc<double>((size_t)L * k);
    double* W = want_vec ? dalloc<double>((size_t)k * k) : nullptr;
    double* sig = dalloc<double>((size_t)k);
    unsigned long long* rot = dalloc<unsigned long long>(1);
    struct Free {
        cudaStream_t s;
        std::vector<void*> p;
        ~Free() {
            for (void* q : p) pool_free(q, s);
        }
    } fr{s, {G, W, sig, rot}};
    CK(cudaMemcpyAsync(G, Gh.data(), Gh.size() * 8, cudaMemcpyHostToDevice, s));
    if (W) identity_kernel<<<std::min<long long>(((long long)k * k + 255) / 256, 148 * 8), 256, 0, s>>>(W, k);

    const int K = k + (k & 1);
    const double tol = std::sqrt((double)L) * 2.220446049250313e-16;
    int sweeps = 0;
    unsigned long long rh = 1;
    while (K >= 2 && rh && sweeps < kMaxSweeps) {
        CK(cudaMemsetAsync(rot, 0, 8, s));
        for (int st = 0; st < K - 1; ++st)
            jacobi_step_kernel<<<K / 2, kJT, 0, s>>>(G, L, W, k, K, st, tol, rot);
        CK(cudaGetLastError());
        CK(cudaMemcpyAsync(&rh, rot, 8, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        ++sweeps;
    }
    column_norm_kernel<<<k, kJT, 0, s>>>(G, L, sig);
    CK(cudaGetLastError());
    std::vector<double> sh((size_t)k);
    CK(cudaMemcpyAsync(sh.data(), sig, (size_t)k * 8, cudaMemcpyDeviceToHost, s));
    std::vector<double> Wh;
    if (want_vec) {
        Wh.resize((size_t)k * k);
        CK(cudaMemcpyAsync(Gh.data(), G, Gh.size() * 8, cudaMemcpyDeviceToHost, s));
        CK(cudaMemcpyAsync(Wh.data(), W, Wh.size() * 8, cudaMemcpyDeviceToHost, s));
    }
    CK(cudaStreamSynchronize(s));

    std::vector<int> ord((size_t)k);
    std::iota(ord.begin(), ord.end(), 0);
    std::stable_sort(ord.begin(), ord.end(), [&](int x, int y) { return sh[(size_t)x] > sh[(size_t)y]; });
    for (int j = 0; j < k; ++j) sigma_out[j] = sh[(size_t)ord[(size_t)j]];
    const double cutoff = k > 0 ? 1e-10 * sigma_out[0] : 0.0;
    int rank = 0;
    for (int j = 0; j < k; ++j)
        if (sigma_out[j] > cutoff) ++rank;
    if (rank_out) *rank_out = rank;
    if (sweeps_out) *sweeps_out = sweeps;
    if (want_vec) {
        // U_G columns = g_j / sigma_j (zero for a zero singular value)
        double* UG = tall ? U : V;      // L x k
        double* WW = tall ? V : U;      // k x k
        for (int j = 0; j < k; ++j) {
            const int src = ord[(size_t)j];
            const double sj = sh[(size_t)src];
            if (UG) {
                const double* g = Gh.data() + (size_t)src * L;
                double* d = UG + (size_t)j * L;
                for (long long r = 0; r < L; ++r) d[r] = sj > 0.0 ? g[r] / sj : 0.0;
            }
            if (WW) std::copy(Wh.begin() + (size_t)src * k, Wh.begin() + (size_t)(src + 1) * k, WW + (size_t)j * k);
        }
    }
    return ASYRK_OK;
}

}  // namespace
}  // namespace ak

extern "C" asyrk_status asyrk_dense_svd(const asyrk_csr_view* A, int64_t max_cells, double* sigma, double* U,
                                        double* V, int32_t* rank, int32_t* sweeps) {
    return ak::guarded([&] { return ak::svd_impl(A, max_cells, sigma, U, V, rank, sweeps); });
}
