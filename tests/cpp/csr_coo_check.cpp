// csr_from_coo (the pybind drop-in path's CSR assembly, host/csr_coo.hpp)
// against CsrMatrix::from_triplets on the same entries: identical arrays and
// row norms, or the same error code and message. Cases: sorted / unsorted,
// zero values (one row emptied by them), out-of-range indices, duplicates,
// sizes that split into several parallel chunks. Also csr_from_coo_normalized
// against normalize_rows(from_triplets(...), b): the same matrix and scaled b
// (unit and non-unit rows, a wrong-length b). Prints "ok" or the case.
#include <cstdio>
#include <random>
#include <string>
#include <vector>

#include "../../paper_1401_4780_b200/csrc/host/csr_coo.hpp"

using namespace asyrk;

struct Out {
    bool err = false;
    std::string what;
    int code = -1;
    std::vector<index_t> rp, ci;
    std::vector<double> v, nrm, b;
    bool normalized = false;
};

template <class F>
Out run_n(F&& f) {
    Out o;
    try {
        auto pr = f();
        const CsrMatrix& A = pr.first;
        o.rp.assign(A.row_ptr().begin(), A.row_ptr().end());
        o.ci.assign(A.col_idx().begin(), A.col_idx().end());
        o.v.assign(A.values().begin(), A.values().end());
        o.nrm.assign(A.row_norm().begin(), A.row_norm().end());
        o.b = pr.second;
        o.normalized = A.is_normalized();
    } catch (const Error& e) {
        o.err = true;
        o.what = e.what();
        o.code = static_cast<int>(e.code());
    }
    return o;
}

template <class F>
Out run(F&& f) {
    Out o;
    try {
        CsrMatrix A = f();
        o.rp.assign(A.row_ptr().begin(), A.row_ptr().end());
        o.ci.assign(A.col_idx().begin(), A.col_idx().end());
        o.v.assign(A.values().begin(), A.values().end());
        o.nrm.assign(A.row_norm().begin(), A.row_norm().end());
    } catch (const Error& e) {
        o.err = true;
        o.what = e.what();
        o.code = static_cast<int>(e.code());
    }
    return o;
}

static bool same(const Out& a, const Out& b) {
    if (a.err || b.err) return a.err == b.err && a.code == b.code && a.what == b.what;
    return a.rp == b.rp && a.ci == b.ci && a.v == b.v && a.nrm == b.nrm && a.b == b.b && a.normalized == b.normalized;
}

int main() {
    std::mt19937_64 g(7);
    int cases = 0;
    for (int c = 0; c < 24; ++c) {
        const index_t m = c < 12 ? 300 : 40000, n = c < 12 ? 200 : 30000;
        std::vector<index_t> rows, cols;
        std::vector<double> vals;
        for (index_t i = 0; i < m; ++i) {
            const int len = 1 + (int)(g() % 12);
            index_t col = (index_t)(g() % 50);
            for (int k = 0; k < len && col < n; ++k) {
                rows.push_back(i);
                cols.push_back(col);
                vals.push_back(((g() % 7) == 0 && (c % 3) == 1) ? 0.0 : 1.0 + (double)(g() % 1000) / 7.0);
                col += 1 + (index_t)(g() % 40);
            }
        }
        const int kind = c % 6;
        if (kind == 2) std::swap(rows[5], rows[rows.size() - 3]), std::swap(cols[5], cols[cols.size() - 3]);  // unsorted
        if (kind == 3) cols[rows.size() / 2] = n + 4;                                                            // out of range
        if (kind == 4) {  // a duplicate (unsorted path)
            rows.push_back(rows[10]);
            cols.push_back(cols[10]);
            vals.push_back(2.0);
        }
        if (kind == 5) {  // a row whose only entries are zero
            for (std::size_t k = 0; k < rows.size(); ++k)
                if (rows[k] == 7) vals[k] = 0.0;
        }
        std::vector<Triplet> t(rows.size());
        for (std::size_t k = 0; k < rows.size(); ++k) t[k] = Triplet{rows[k], cols[k], vals[k]};
        const Out a = run([&] { return CsrMatrix::from_triplets(t, m, n); });
        const Out b = run([&] { return csr_from_coo(m, n, rows.data(), cols.data(), vals.data(), rows.size()); });
        if (!same(a, b)) {
            std::printf("mismatch case %d (kind %d): ref err %d '%s', coo err %d '%s'\n", c, kind, a.err, a.what.c_str(),
                        b.err, b.what.c_str());
            return 1;
        }
        ++cases;
        // normalized: rows scaled so that some are unit already; b of the right / wrong length
        std::vector<double> vals2 = vals;
        for (std::size_t k = 0; k < vals2.size(); ++k)
            if (rows[k] % 5 == 0) vals2[k] = 0.5;  // rows of 0.5 entries: unit when 4 entries
        for (std::size_t k = 0; k < t.size(); ++k) t[k].value = vals2[k];
        std::vector<double> rhs(c == 7 ? m - 1 : m);
        for (auto& x : rhs) x = (double)(g() % 1000) / 3.0;
        const Out an = run_n([&] { return normalize_rows(CsrMatrix::from_triplets(t, m, n), rhs); });
        const Out bn = run_n(
            [&] { return csr_from_coo_normalized(m, n, rows.data(), cols.data(), vals2.data(), rows.size(), rhs); });
        if (!same(an, bn)) {
            std::printf("normalized mismatch case %d (kind %d): ref err %d '%s', coo err %d '%s'\n", c, kind, an.err,
                        an.what.c_str(), bn.err, bn.what.c_str());
            return 1;
        }
        ++cases;
    }
    std::printf("ok %d\n", cases);
    return 0;
}
