// Instance I/O (replaces ref/src/io.cpp:41-183) + the binary CSR cache.
//
// Same bytes as the reference: entries "%lld %lld %.17g\n" (std::to_chars
// with general format and precision 17 is specified to print exactly what
// printf("%.17g") prints), vectors "%.17g\n", meta.json in nlohmann's
// dump(2) layout (sorted keys, shortest round-trip doubles). Reading parses
// the whitespace-separated token stream the reference reads with
// `in >> i >> j >> v`, correctly rounded (std::from_chars), and reports the
// reference's IoError messages. Both directions are split over host threads:
// the text is cut at whitespace into one chunk per thread, tokens are
// counted, then parsed straight into their global slots.
#include "asyrk/io.hpp"

#include <algorithm>
#include <cerrno>
#include <cmath>
#include <memory>
#include <mutex>
#include <charconv>
#include <cstdio>
#include <cstring>
#include <filesystem>
#include <limits>
#include <thread>

#include "../capi_common.h"
#include "asyrk/error.hpp"
#include "asyrk_io.h"
#include "common.hpp"
#include "json.hpp"

namespace asyrk {

namespace {

[[noreturn]] void io_fail(const std::string& path, const std::string& what) {
    fail(ErrorCode::IoError, path + ": " + what);
}

int io_threads(std::size_t work_bytes) {
    if (work_bytes < (1u << 20)) return 1;
    const unsigned hc = std::thread::hardware_concurrency();
    return (int)std::max(1u, std::min(16u, hc ? hc : 1u));
}

template <class F>
void parallel_for(int T, F&& f) {
    if (T <= 1) {
        f(0);
        return;
    }
    std::vector<std::thread> th;
    th.reserve((size_t)T - 1);
    for (int t = 1; t < T; ++t) th.emplace_back([&f, t] { f(t); });
    f(0);
    for (auto& x : th) x.join();
}

inline bool is_space(char c) { return c == ' ' || c == '\t' || c == '\n' || c == '\r' || c == '\v' || c == '\f'; }

std::string slurp(const std::string& path) {
    std::FILE* f = std::fopen(path.c_str(), "rb");
    if (!f) io_fail(path, "cannot open");
    std::string s;
    if (std::fseek(f, 0, SEEK_END) == 0) {
        const long sz = std::ftell(f);
        if (sz > 0) {
            s.resize((size_t)sz);
            std::fseek(f, 0, SEEK_SET);
            const size_t got = std::fread(s.data(), 1, s.size(), f);
            s.resize(got);
        }
    }
    std::fclose(f);
    return s;
}

// Whitespace-separated tokens of [b, e), in parallel: fn(token_index, p, q)
// for every token (global index in stream order). Returns the token count.
template <class F>
long long for_each_token(const char* b, const char* e, int T, F&& fn) {
    T = std::max(1, std::min<int>(T, (int)((e - b) / 4096) + 1));
    std::vector<const char*> cut((size_t)T + 1);
    cut[0] = b;
    cut[(size_t)T] = e;
    for (int t = 1; t < T; ++t) {
        const char* p = b + (e - b) * t / T;
        if (p < cut[(size_t)t - 1]) p = cut[(size_t)t - 1];
        while (p < e && !is_space(*p)) ++p;  // never split a token
        cut[(size_t)t] = p;
    }
    std::vector<long long> cnt((size_t)T + 1, 0);
    parallel_for(T, [&](int t) {
        long long c = 0;
        for (const char* p = cut[(size_t)t]; p < cut[(size_t)t + 1];) {
            while (p < cut[(size_t)t + 1] && is_space(*p)) ++p;
            if (p == cut[(size_t)t + 1]) break;
            ++c;
            while (p < cut[(size_t)t + 1] && !is_space(*p)) ++p;
        }
        cnt[(size_t)t + 1] = c;
    });
    for (int t = 0; t < T; ++t) cnt[(size_t)t + 1] += cnt[(size_t)t];
    parallel_for(T, [&](int t) {
        long long k = cnt[(size_t)t];
        for (const char* p = cut[(size_t)t]; p < cut[(size_t)t + 1];) {
            while (p < cut[(size_t)t + 1] && is_space(*p)) ++p;
            if (p == cut[(size_t)t + 1]) break;
            const char* q = p;
            while (q < cut[(size_t)t + 1] && !is_space(*q)) ++q;
            fn(k++, p, q);
            p = q;
        }
    });
    return cnt[(size_t)T];
}

// istream-style numbers: optional sign, the whole token must be the number
bool parse_i64(const char* p, const char* q, long long& v) {
    if (p < q && *p == '+') ++p;
    auto r = std::from_chars(p, q, v);
    return r.ec == std::errc() && r.ptr == q;
}

bool parse_f64(const char* p, const char* q, double& v) {
    const char* s = p;
    if (s < q && *s == '+') ++s;
    const char* d = (s < q && *s == '-') ? s + 1 : s;
    if (d < q && (*d == 'i' || *d == 'I' || *d == 'n' || *d == 'N')) return false;  // num_get: no inf/nan
    auto r = std::from_chars(s, q, v, std::chars_format::general);
    return r.ec == std::errc() && r.ptr == q;
}

// printf("%.17g") via std::to_chars (same output by specification)
inline char* put_g17(char* o, char* end, double v) { return std::to_chars(o, end, v, std::chars_format::general, 17).ptr; }
inline char* put_i64(char* o, char* end, long long v) { return std::to_chars(o, end, v).ptr; }

struct FileOut {
    std::FILE* f;
    std::string path;
    FileOut(const std::string& p) : f(std::fopen(p.c_str(), "wb")), path(p) {
        if (!f) io_fail(p, std::strerror(errno));
    }
    ~FileOut() {
        if (f) std::fclose(f);
    }
    void put(const std::string& s) {
        if (!s.empty() && std::fwrite(s.data(), 1, s.size(), f) != s.size()) io_fail(path, "write failed");
    }
    void close() {
        if (std::fflush(f) != 0) io_fail(path, "write failed");
        const int rc = std::fclose(f);
        f = nullptr;
        if (rc != 0) io_fail(path, "write failed");
    }
};

// ---- matrices ----------------------------------------------------------
struct CsrArrays {
    index_t m, n;
    const index_t *row_ptr, *col_idx;
    const double* values;
};

void write_mtx(const std::string& path, const CsrArrays& A) {
    FileOut out(path);
    const index_t nnz = A.row_ptr[A.m];
    out.put("%%MatrixMarket matrix coordinate real general\n" + std::to_string(A.m) + " " + std::to_string(A.n) + " " +
            std::to_string(nnz) + "\n");
    const int T = io_threads((size_t)nnz * 40);
    std::vector<std::string> buf((size_t)T);
    constexpr index_t kRowsPerRound = 1 << 16;
    for (index_t r0 = 0; r0 < A.m; r0 += kRowsPerRound * T) {  // bounded buffers, in file order
        parallel_for(T, [&](int t) {
            const index_t a = std::min(A.m, r0 + kRowsPerRound * t), b = std::min(A.m, a + kRowsPerRound);
            std::string& s = buf[(size_t)t];
            s.clear();
            s.resize((size_t)(A.row_ptr[b] - A.row_ptr[a]) * 64 + 64);
            char* w = s.data();
            char* end = s.data() + s.size();
            for (index_t i = a; i < b; ++i)
                for (index_t p = A.row_ptr[i]; p < A.row_ptr[i + 1]; ++p) {
                    w = put_i64(w, end, i + 1);
                    *w++ = ' ';
                    w = put_i64(w, end, A.col_idx[p] + 1);
                    *w++ = ' ';
                    w = put_g17(w, end, A.values[p]);
                    *w++ = '\n';
                }
            s.resize((size_t)(w - s.data()));
        });
        for (int t = 0; t < T; ++t) out.put(buf[(size_t)t]);
    }
    out.close();
}

// the first line (getline semantics), and the offset just past it
std::string line_at(const std::string& s, size_t& pos, bool& ok) {
    if (pos >= s.size()) {
        ok = false;
        return std::string();
    }
    const size_t e = s.find('\n', pos);
    std::string l = s.substr(pos, (e == std::string::npos ? s.size() : e) - pos);
    pos = e == std::string::npos ? s.size() : e + 1;
    ok = true;
    return l;
}

std::vector<std::string> words(const std::string& l) {
    std::vector<std::string> w;
    size_t p = 0;
    while (p < l.size()) {
        while (p < l.size() && is_space(l[p])) ++p;
        if (p == l.size()) break;
        size_t q = p;
        while (q < l.size() && !is_space(l[q])) ++q;
        w.emplace_back(l.substr(p, q - p));
        p = q;
    }
    return w;
}

// CSR from entries in file order: a parallel check for row-major order with
// strictly increasing columns (what write_matrix_market produces) builds the
// arrays directly; anything else goes through from_triplets (sort, duplicate
// and zero handling of ref csr.cpp:9-63).
CsrMatrix entries_to_csr(index_t m, index_t n, std::vector<index_t>& ri, std::vector<index_t>& ci,
                         std::vector<double>& va) {
    const index_t nnz = (index_t)ri.size();
    const int T = io_threads((size_t)nnz * 24);
    std::vector<char> sorted_ok((size_t)T, 1);
    parallel_for(T, [&](int t) {
        const index_t a = nnz * t / T, b = nnz * (t + 1) / T;
        for (index_t k = std::max<index_t>(a, 1); k < b; ++k)
            if (ri[k] < ri[k - 1] || (ri[k] == ri[k - 1] && ci[k] <= ci[k - 1])) {
                sorted_ok[(size_t)t] = 0;
                return;
            }
        if (a > 0 && a < b && (ri[a] < ri[a - 1] || (ri[a] == ri[a - 1] && ci[a] <= ci[a - 1]))) sorted_ok[(size_t)t] = 0;
    });
    const bool sorted = std::all_of(sorted_ok.begin(), sorted_ok.end(), [](char c) { return c != 0; });
    const bool zeros = std::any_of(va.begin(), va.end(), [](double v) { return v == 0.0; });
    if (!sorted || zeros) {
        std::vector<Triplet> t((size_t)nnz);
        for (index_t k = 0; k < nnz; ++k) t[(size_t)k] = Triplet{ri[k], ci[k], va[k]};
        return CsrMatrix::from_triplets(t, m, n);
    }
    std::vector<index_t> rp((size_t)m + 1, 0);
    for (index_t k = 0; k < nnz; ++k) ++rp[(size_t)ri[k] + 1];
    for (index_t i = 0; i < m; ++i) rp[(size_t)i + 1] += rp[(size_t)i];
    return CsrMatrix::from_csr(m, n, std::move(rp), std::move(ci), std::move(va));
}

CsrMatrix read_mtx(const std::string& path) {
    const std::string s = slurp(path);
    size_t pos = 0;
    bool ok = false;
    std::string line = line_at(s, pos, ok);
    if (!ok) io_fail(path, "empty file");
    if (line.rfind("%%MatrixMarket", 0) != 0) io_fail(path, "missing MatrixMarket banner");
    {
        std::vector<std::string> w = words(line);
        w.resize(std::max<size_t>(w.size(), 5));
        if (w[1] != "matrix" || w[2] != "coordinate" || w[3] != "real" || w[4] != "general")
            io_fail(path, "unsupported MatrixMarket type: " + line);
    }
    for (;;) {  // comments and blank lines up to the size line
        line = line_at(s, pos, ok);
        if (!ok) {
            line.clear();
            break;
        }
        if (!line.empty() && line[0] != '%') break;
    }
    long long m = 0, n = 0, nnz = 0;
    {
        const std::vector<std::string> w = words(line);
        if (w.size() < 3 || !parse_i64(w[0].data(), w[0].data() + w[0].size(), m) ||
            !parse_i64(w[1].data(), w[1].data() + w[1].size(), n) ||
            !parse_i64(w[2].data(), w[2].data() + w[2].size(), nnz))
            io_fail(path, "bad size line");
    }
    if (m < 1 || n < 1 || nnz < 0) io_fail(path, "bad dimensions");
    std::vector<index_t> ri((size_t)nnz), ci((size_t)nnz);
    std::vector<double> va((size_t)nnz);
    // first failing entry per kind (the reference stops at the first one)
    const long long need = 3 * nnz;
    const int T = io_threads(s.size() - pos);
    std::mutex mu;
    long long first_parse = std::numeric_limits<long long>::max();
    const long long total = for_each_token(s.data() + pos, s.data() + s.size(), T, [&](long long k, const char* p,
                                                                                    const char* q) {
        if (k >= need) return;
        const long long e = k / 3;
        const int f = (int)(k % 3);
        bool good;
        if (f < 2) {
            long long v = 0;
            good = parse_i64(p, q, v);
            if (good) (f == 0 ? ri : ci)[(size_t)e] = v;
        } else {
            double v = 0.0;
            good = parse_f64(p, q, v);
            if (good) va[(size_t)e] = v;
        }
        if (!good) {
            std::lock_guard<std::mutex> lk(mu);
            first_parse = std::min(first_parse, e);
        }
    });
    if (total < need) first_parse = std::min(first_parse, total / 3);
    // range check of the entries before the first parse failure
    long long first_range = std::numeric_limits<long long>::max();
    const long long upto = std::min<long long>(first_parse, nnz);
    for (long long e = 0; e < upto; ++e)
        if (ri[(size_t)e] < 1 || ri[(size_t)e] > m || ci[(size_t)e] < 1 || ci[(size_t)e] > n) {
            first_range = e;
            break;
        }
    if (first_range < first_parse) io_fail(path, "entry index out of range");
    if (first_parse < nnz) io_fail(path, "truncated entry list");
    for (long long e = 0; e < nnz; ++e) {
        --ri[(size_t)e];
        --ci[(size_t)e];
    }
    return entries_to_csr(m, n, ri, ci, va);
}

// ---- vectors -----------------------------------------------------------
void write_vec(const std::string& path, const double* v, size_t count) {
    FileOut out(path);
    const int T = io_threads(count * 24);
    std::vector<std::string> buf((size_t)T);
    parallel_for(T, [&](int t) {
        const size_t a = count * t / T, b = count * (t + 1) / T;
        std::string& s = buf[(size_t)t];
        s.resize((b - a) * 32 + 8);
        char* w = s.data();
        for (size_t k = a; k < b; ++k) {
            w = put_g17(w, s.data() + s.size(), v[k]);
            *w++ = '\n';
        }
        s.resize((size_t)(w - s.data()));
    });
    for (int t = 0; t < T; ++t) out.put(buf[(size_t)t]);
    out.close();
}

std::vector<double> read_vec(const std::string& path) {
    const std::string s = slurp(path);
    const int T = io_threads(s.size());
    std::mutex mu;
    long long first_bad = std::numeric_limits<long long>::max();
    // a counting pass sizes the output, then every token parses into its slot
    const long long count = for_each_token(s.data(), s.data() + s.size(), T, [](long long, const char*, const char*) {});
    std::vector<double> v((size_t)count);
    for_each_token(s.data(), s.data() + s.size(), T, [&](long long k, const char* p, const char* q) {
        double x = 0.0;
        if (parse_f64(p, q, x)) {
            v[(size_t)k] = x;
        } else {
            std::lock_guard<std::mutex> lk(mu);
            first_bad = std::min(first_bad, k);
        }
    });
    if (first_bad != std::numeric_limits<long long>::max()) io_fail(path, "non-numeric content");
    return v;
}

// ---- meta.json in nlohmann's dump(2) layout ----------------------------
// Shortest round-trip digits placed like nlohmann::detail::dtoa_impl::
// format_buffer (decimal notation for exponents in [-4, 15), else d.ddde+XX).
std::string nl_double(double v) {
    if (v == 0.0) return std::signbit(v) ? "-0.0" : "0.0";
    char buf[64];
    auto r = std::to_chars(buf, buf + sizeof buf, v, std::chars_format::scientific);
    std::string sci(buf, r.ptr);
    std::string out;
    size_t p = 0;
    if (sci[0] == '-') {
        out += '-';
        p = 1;
    }
    const size_t epos = sci.find('e');
    std::string digits;
    for (size_t k = p; k < epos; ++k)
        if (sci[k] != '.') digits += sci[k];
    const int e10 = std::atoi(sci.c_str() + epos + 1);
    const int k = (int)digits.size();
    const int n = e10 + 1;  // value = 0.d1d2... x 10^n
    if (k <= n && n <= 15) {
        out += digits + std::string((size_t)(n - k), '0') + ".0";
    } else if (0 < n && n <= 15) {
        out += digits.substr(0, (size_t)n) + "." + digits.substr((size_t)n);
    } else if (-4 < n && n <= 0) {
        out += "0." + std::string((size_t)(-n), '0') + digits;
    } else {
        out += digits.substr(0, 1);
        if (k > 1) out += "." + digits.substr(1);
        const int x = n - 1;
        out += x < 0 ? "e-" : "e+";
        const int ax = x < 0 ? -x : x;
        if (ax < 10) out += '0';
        out += std::to_string(ax);
    }
    return out;
}

struct MetaField {
    std::string key, text;
};

std::string meta_json(std::vector<MetaField> f) {
    std::sort(f.begin(), f.end(), [](const MetaField& a, const MetaField& b) { return a.key < b.key; });
    std::string s = "{\n";
    for (size_t k = 0; k < f.size(); ++k) {
        s += "  \"" + f[k].key + "\": " + f[k].text;
        s += k + 1 < f.size() ? ",\n" : "\n";
    }
    return s + "}";
}

}  // namespace

void write_matrix_market(const std::string& path, const CsrMatrix& A) {
    write_mtx(path, CsrArrays{A.rows(), A.cols(), A.row_ptr().data(), A.col_idx().data(), A.values().data()});
}

CsrMatrix read_matrix_market(const std::string& path) { return read_mtx(path); }

void write_vector(const std::string& path, std::span<const double> v) { write_vec(path, v.data(), v.size()); }

std::vector<double> read_vector(const std::string& path) { return read_vec(path); }

void write_text(const std::string& path, const std::string& text) {
    FileOut out(path);
    out.put(text);
    out.close();
}

std::string read_text(const std::string& path) { return slurp(path); }

void write_instance(const std::string& dir, const Instance& inst) {
    std::error_code ec;
    std::filesystem::create_directories(dir, ec);
    if (ec) io_fail(dir, ec.message());
    write_matrix_market(dir + "/A.mtx", inst.A);
    write_vector(dir + "/b.txt", inst.b);
    if (inst.x_star) write_vector(dir + "/xstar.txt", *inst.x_star);
    const GenSpec& g = inst.spec;
    write_text(dir + "/meta.json", meta_json({{"schema", "1"},
                                              {"m", std::to_string(g.m)},
                                              {"n", std::to_string(g.n)},
                                              {"delta", nl_double(g.delta)},
                                              {"seed", std::to_string(g.seed)},
                                              {"consistent", g.consistent ? "true" : "false"},
                                              {"noise_level", nl_double(g.noise_level)},
                                              {"nnz", std::to_string(inst.A.nnz())},
                                              {"normalized", inst.A.is_normalized() ? "true" : "false"},
                                              {"has_x_star", inst.x_star ? "true" : "false"}}) +
                                       "\n");
}

Instance read_instance(const std::string& dir) {
    json::Value meta;
    try {
        meta = json::parse(read_text(dir + "/meta.json"));
    } catch (const Error&) {
        throw;
    } catch (const std::exception& e) {
        io_fail(dir + "/meta.json", e.what());
    }
    Instance inst;
    bool normalized = false, has_xs = false;
    try {
        if (!meta.is_object()) throw std::runtime_error("not an object");
        const json::Object& o = meta.object();
        inst.spec.m = o.at("m").integer();
        inst.spec.n = o.at("n").integer();
        inst.spec.delta = o.at("delta").number();
        inst.spec.seed = (std::uint64_t)o.at("seed").integer();
        inst.spec.consistent = std::get<bool>(o.at("consistent").v);
        inst.spec.noise_level = o.at("noise_level").number();
        if (o.count("normalized")) normalized = std::get<bool>(o.at("normalized").v);
        if (o.count("has_x_star")) has_xs = std::get<bool>(o.at("has_x_star").v);
    } catch (const std::exception& e) {
        io_fail(dir + "/meta.json", e.what());
    }
    inst.A = read_matrix_market(dir + "/A.mtx");
    inst.b = read_vector(dir + "/b.txt");
    if (inst.A.rows() != (index_t)inst.b.size()) io_fail(dir, "A and b dimensions disagree");
    if (inst.A.rows() != inst.spec.m || inst.A.cols() != inst.spec.n)
        io_fail(dir, "matrix dimensions disagree with metadata");
    if (normalized) inst.A.flag_normalized();
    if (has_xs) {
        auto xs = read_vector(dir + "/xstar.txt");
        if ((index_t)xs.size() != inst.A.cols()) io_fail(dir + "/xstar.txt", "wrong length");
        inst.x_star = std::move(xs);
    }
    return inst;
}

// ---- binary CSR cache --------------------------------------------------
namespace {
constexpr char kMagic[8] = {'A', 'S', 'Y', 'R', 'K', 'C', 'S', 'R'};

void write_cache(const std::string& path, index_t m, index_t n, const index_t* rp, const index_t* ci, const double* v,
                 const double* rn, bool normalized) {
    FileOut out(path);
    const index_t nnz = rp[m];
    std::string head(kMagic, 8);
    const uint32_t ver = 1, flags = normalized ? 1u : 0u;
    head.append(reinterpret_cast<const char*>(&ver), 4);
    head.append(reinterpret_cast<const char*>(&flags), 4);
    for (index_t x : {m, n, nnz}) head.append(reinterpret_cast<const char*>(&x), 8);
    out.put(head);
    auto blob = [&](const void* p, size_t bytes) {
        if (bytes && std::fwrite(p, 1, bytes, out.f) != bytes) io_fail(path, "write failed");
    };
    blob(rp, ((size_t)m + 1) * 8);
    blob(ci, (size_t)nnz * 8);
    blob(v, (size_t)nnz * 8);
    blob(rn, (size_t)m * 8);
    out.close();
}
}  // namespace

void write_csr_cache(const std::string& path, const CsrMatrix& A) {
    write_cache(path, A.rows(), A.cols(), A.row_ptr().data(), A.col_idx().data(), A.values().data(),
                A.row_norm().data(), A.is_normalized());
}

CsrMatrix read_csr_cache(const std::string& path) {
    const std::string s = slurp(path);
    if (s.size() < 40 || std::memcmp(s.data(), kMagic, 8) != 0) io_fail(path, "not an ASYRKCSR cache");
    uint32_t ver = 0, flags = 0;
    std::memcpy(&ver, s.data() + 8, 4);
    std::memcpy(&flags, s.data() + 12, 4);
    index_t m = 0, n = 0, nnz = 0;
    std::memcpy(&m, s.data() + 16, 8);
    std::memcpy(&n, s.data() + 24, 8);
    std::memcpy(&nnz, s.data() + 32, 8);
    if (ver != 1) io_fail(path, "unsupported cache version");
    if (m < 1 || n < 1 || nnz < 0 ||
        s.size() != 40 + ((size_t)m + 1) * 8 + (size_t)nnz * 16 + (size_t)m * 8)
        io_fail(path, "truncated or inconsistent cache");
    std::vector<index_t> rp((size_t)m + 1), ci((size_t)nnz);
    std::vector<double> v((size_t)nnz);
    const char* p = s.data() + 40;
    std::memcpy(rp.data(), p, rp.size() * 8);
    p += rp.size() * 8;
    std::memcpy(ci.data(), p, ci.size() * 8);
    p += ci.size() * 8;
    std::memcpy(v.data(), p, v.size() * 8);
    if (rp[0] != 0 || rp[(size_t)m] != nnz) io_fail(path, "corrupt row pointers");
    for (index_t i = 0; i < m; ++i) {
        if (rp[(size_t)i + 1] <= rp[(size_t)i]) io_fail(path, "corrupt row pointers");
        for (index_t k = rp[(size_t)i]; k < rp[(size_t)i + 1]; ++k)
            if (ci[(size_t)k] < 0 || ci[(size_t)k] >= n || (k > rp[(size_t)i] && ci[(size_t)k] <= ci[(size_t)k - 1]))
                io_fail(path, "corrupt column indices");
    }
    CsrMatrix A = CsrMatrix::from_csr(m, n, std::move(rp), std::move(ci), std::move(v));
    if (flags & 1u) A.flag_normalized();
    return A;
}

}  // namespace asyrk

// ---- C ABI (include/asyrk_io.h) ------------------------------------------
namespace {

template <class F>
asyrk_status io_guarded(F&& f) {
    try {
        return f();
    } catch (const asyrk::Error& e) {
        return ak::fail((asyrk_status)(static_cast<int>(e.code()) + 1), e.what());
    } catch (const std::bad_alloc&) {
        return ak::fail(ASYRK_E_TooLarge, "host allocation failed");
    } catch (const std::exception& e) {
        return ak::fail(ASYRK_E_IoError, e.what());
    }
}

asyrk::CsrArrays view_arrays(const asyrk_csr_view* A) {
    return asyrk::CsrArrays{A->m, A->n, A->row_ptr, A->col_idx, A->values};
}

void put_info(const asyrk::CsrMatrix& A, asyrk_host_csr_info* info) {
    if (!info) return;
    info->m = A.rows();
    info->n = A.cols();
    info->nnz = A.nnz();
    info->normalized = A.is_normalized() ? 1 : 0;
}

double* copy_out(const std::vector<double>& v) {
    double* p = static_cast<double*>(std::malloc(std::max<size_t>(v.size(), 1) * sizeof(double)));
    if (!p) throw std::bad_alloc();
    if (!v.empty()) std::memcpy(p, v.data(), v.size() * sizeof(double));
    return p;
}

bool bad_view(const asyrk_csr_view* A) { return !A || !A->row_ptr || (A->nnz > 0 && (!A->col_idx || !A->values)); }

}  // namespace

extern "C" {

asyrk_status asyrk_read_matrix_market(const char* path, asyrk_host_csr** out, asyrk_host_csr_info* info) {
    if (!path || !out) return ak::fail(ASYRK_E_InvalidArgument, "null argument");
    return io_guarded([&] {
        auto h = std::make_unique<asyrk_host_csr>();
        h->A = asyrk::read_matrix_market(path);
        put_info(h->A, info);
        *out = h.release();
        return ASYRK_OK;
    });
}

asyrk_status asyrk_write_matrix_market(const char* path, const asyrk_csr_view* A) {
    if (!path || bad_view(A)) return ak::fail(ASYRK_E_InvalidArgument, "null argument");
    return io_guarded([&] {
        asyrk::write_mtx(path, view_arrays(A));
        return ASYRK_OK;
    });
}

asyrk_status asyrk_read_csr_cache(const char* path, asyrk_host_csr** out, asyrk_host_csr_info* info) {
    if (!path || !out) return ak::fail(ASYRK_E_InvalidArgument, "null argument");
    return io_guarded([&] {
        auto h = std::make_unique<asyrk_host_csr>();
        h->A = asyrk::read_csr_cache(path);
        put_info(h->A, info);
        *out = h.release();
        return ASYRK_OK;
    });
}

asyrk_status asyrk_write_csr_cache(const char* path, const asyrk_csr_view* A) {
    if (!path || bad_view(A) || !A->row_norm) return ak::fail(ASYRK_E_InvalidArgument, "null argument");
    return io_guarded([&] {
        asyrk::write_cache(path, A->m, A->n, A->row_ptr, A->col_idx, A->values, A->row_norm, A->normalized != 0);
        return ASYRK_OK;
    });
}

asyrk_status asyrk_host_csr_copy(const asyrk_host_csr* h, int64_t* row_ptr, int64_t* col_idx, double* values,
                                 double* row_norm) {
    if (!h || !row_ptr || !col_idx || !values) return ak::fail(ASYRK_E_InvalidArgument, "null argument");
    const asyrk::CsrMatrix& A = h->A;
    std::memcpy(row_ptr, A.row_ptr().data(), A.row_ptr().size() * 8);
    if (A.nnz()) {
        std::memcpy(col_idx, A.col_idx().data(), (size_t)A.nnz() * 8);
        std::memcpy(values, A.values().data(), (size_t)A.nnz() * 8);
    }
    if (row_norm) std::memcpy(row_norm, A.row_norm().data(), (size_t)A.rows() * 8);
    return ASYRK_OK;
}

asyrk_status asyrk_host_csr_get_info(const asyrk_host_csr* h, asyrk_host_csr_info* info) {
    if (!h || !info) return ak::fail(ASYRK_E_InvalidArgument, "null argument");
    put_info(h->A, info);
    return ASYRK_OK;
}

void asyrk_host_csr_free(asyrk_host_csr* h) { delete h; }

asyrk_status asyrk_read_vector(const char* path, double** out, int64_t* count) {
    if (!path || !out || !count) return ak::fail(ASYRK_E_InvalidArgument, "null argument");
    return io_guarded([&] {
        const std::vector<double> v = asyrk::read_vector(path);
        *out = copy_out(v);
        *count = (int64_t)v.size();
        return ASYRK_OK;
    });
}

asyrk_status asyrk_write_vector(const char* path, const double* v, int64_t count) {
    if (!path || (count > 0 && !v) || count < 0) return ak::fail(ASYRK_E_InvalidArgument, "bad argument");
    return io_guarded([&] {
        asyrk::write_vec(path, v, (size_t)count);
        return ASYRK_OK;
    });
}

void asyrk_free(void* p) { std::free(p); }

asyrk_status asyrk_write_instance(const char* dir, const asyrk_csr_view* A, const double* b, const double* x_star,
                                  const asyrk_instance_meta* spec) {
    if (!dir || bad_view(A) || !b || !spec) return ak::fail(ASYRK_E_InvalidArgument, "null argument");
    return io_guarded([&] {
        asyrk::Instance inst;
        inst.A = asyrk::CsrMatrix::from_csr(
            A->m, A->n, std::vector<int64_t>(A->row_ptr, A->row_ptr + A->m + 1),
            std::vector<int64_t>(A->col_idx, A->col_idx + A->nnz), std::vector<double>(A->values, A->values + A->nnz));
        if (A->normalized) inst.A.flag_normalized();
        inst.b.assign(b, b + A->m);
        if (x_star) inst.x_star = std::vector<double>(x_star, x_star + A->n);
        inst.spec = asyrk::GenSpec{spec->m, spec->n, spec->delta, spec->seed, spec->consistent != 0, spec->noise_level};
        asyrk::write_instance(dir, inst);
        return ASYRK_OK;
    });
}

asyrk_status asyrk_read_instance(const char* dir, asyrk_host_csr** A, double** b, double** x_star,
                                 asyrk_instance_meta* meta) {
    if (!dir || !A || !b || !x_star) return ak::fail(ASYRK_E_InvalidArgument, "null argument");
    return io_guarded([&] {
        asyrk::Instance inst = asyrk::read_instance(dir);
        auto h = std::make_unique<asyrk_host_csr>();
        h->A = std::move(inst.A);
        double* bb = copy_out(inst.b);
        double* xs = inst.x_star ? copy_out(*inst.x_star) : nullptr;
        if (meta) {
            meta->m = inst.spec.m;
            meta->n = inst.spec.n;
            meta->delta = inst.spec.delta;
            meta->seed = inst.spec.seed;
            meta->consistent = inst.spec.consistent ? 1 : 0;
            meta->noise_level = inst.spec.noise_level;
            meta->has_x_star = xs ? 1 : 0;
        }
        *A = h.release();
        *b = bb;
        *x_star = xs;
        return ASYRK_OK;
    });
}

}  // extern "C"
