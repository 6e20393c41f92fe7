// Dev: host CSR assembly timing of the drop-in path (triplets -> CsrMatrix -> normalize_rows), 6M entries.
// g++ -O2 -std=c++20 -Iinclude scripts/cpp/csr_host_timing.cpp -Lpaper_1401_4780_b200 -lasyrk_b200 -Wl,-rpath,$PWD/paper_1401_4780_b200
#include <chrono>
#include <cstdio>
#include <random>
#include <vector>
#include "asyrk/csr.hpp"
#include "../../paper_1401_4780_b200/csrc/host/csr_coo.hpp"
using namespace asyrk;
int main() {
    const index_t m = 200000, n = 100000, th = 30;
    std::vector<Triplet> t;
    t.reserve(m * th);
    std::mt19937_64 g(1);
    std::vector<double> b(m, 1.0);
    for (index_t i = 0; i < m; ++i) {
        index_t c = g() % 3000;
        for (int k = 0; k < th; ++k) { t.push_back(Triplet{i, c, 1.0 + (double)(g() % 100)}); c += 1 + g() % 3000; if (c >= n) c = n - 1 - k; }
    }
    for (int rep = 0; rep < 3; ++rep) {
        auto t0 = std::chrono::steady_clock::now();
        std::vector<Triplet> tc = t;
        auto t1 = std::chrono::steady_clock::now();
        CsrMatrix A = CsrMatrix::from_triplets(tc, m, n);
        auto t2 = std::chrono::steady_clock::now();
        auto pr = normalize_rows(A, b);
        auto t3 = std::chrono::steady_clock::now();
        auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
        printf("copy %.1f ms, from_triplets %.1f ms, normalize %.1f ms (nnz %lld)\n", ms(t0, t1), ms(t1, t2), ms(t2, t3), (long long)A.nnz());
        std::vector<index_t> rr(t.size()), cc(t.size());
        std::vector<double> vv(t.size());
        for (size_t k = 0; k < t.size(); ++k) rr[k] = t[k].row, cc[k] = t[k].col, vv[k] = t[k].value;
        auto t4 = std::chrono::steady_clock::now();
        CsrMatrix B = csr_from_coo(m, n, rr.data(), cc.data(), vv.data(), rr.size());
        auto t5 = std::chrono::steady_clock::now();
        printf("csr_from_coo %.1f ms (same arrays: %d)\n", ms(t4, t5), (int)(B.col_idx() == A.col_idx() && B.values() == A.values() && B.row_ptr() == A.row_ptr()));
    }
}
