// Double -> text as the reference's JSON library writes it (nlohmann/json
// 3.11, the trace contract's serializer, ref/src/trace.cpp:33-63): Grisu2 of
// F. Loitsch, "Printing Floating-Point Numbers Quickly and Accurately with
// Integers" (PLDI 2010) — the published algorithm, restated here — followed
// by the library's layout rules (fixed notation for decimal exponents in
// (-4, 15], otherwise d.ddde±XX; "x.0" for integral values). Grisu2 is
// accurate (the output parses back to the same double) but not always
// shortest, so a shortest-digits formatter (std::to_chars) differs from it on
// a small fraction of doubles; matching it makes Trace::to_jsonl byte-identical
// (tests/test_gpu_parity2.py, tests/test_host.py).
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

namespace asyrk::grisu2 {

struct DiyFp {
    uint64_t f;
    int e;
};

inline DiyFp sub(DiyFp x, DiyFp y) { return {x.f - y.f, x.e}; }

// x * y rounded to 64 bits (the upper half of the 128-bit product, rounded)
inline DiyFp mul(DiyFp x, DiyFp y) {
    const uint64_t a = x.f >> 32, b = x.f & 0xFFFFFFFFu, c = y.f >> 32, d = y.f & 0xFFFFFFFFu;
    const uint64_t ac = a * c, bc = b * c, ad = a * d, bd = b * d;
    uint64_t tmp = (bd >> 32) + (ad & 0xFFFFFFFFu) + (bc & 0xFFFFFFFFu);
    tmp += uint64_t{1} << 31;  // round
    return {ac + (ad >> 32) + (bc >> 32) + (tmp >> 32), x.e + y.e + 64};
}

inline DiyFp normalize(DiyFp x) {
    while ((x.f >> 63) == 0) {
        x.f <<= 1;
        x.e--;
    }
    return x;
}

inline DiyFp normalize_to(DiyFp x, int e) {
    const int delta = x.e - e;
    return {x.f << delta, e};
}

struct CachedPower {
    uint64_t f;
    int e;
    int k;
};

// 10^k for k = -300, -292, ..., 324 as normalized 64-bit significands
// (round to nearest) and binary exponents, computed once with exact big
// integer arithmetic.
class PowerTable {
  public:
    static const PowerTable& get() {
        static const PowerTable t;
        return t;
    }
    static constexpr int kMinDecExp = -300, kStep = 8, kCount = 79;
    CachedPower at(int i) const { return p_[i]; }

  private:
    using Big = std::vector<uint32_t>;  // little-endian base 2^32
    static void mul_small(Big& a, uint32_t m) {
        uint64_t carry = 0;
        for (auto& w : a) {
            const uint64_t v = uint64_t{w} * m + carry;
            w = (uint32_t)v;
            carry = v >> 32;
        }
        if (carry) a.push_back((uint32_t)carry);
    }
    static int bitlen(const Big& a) {
        int n = (int)a.size();
        while (n > 0 && a[n - 1] == 0) --n;
        if (!n) return 0;
        int b = 32;
        while (!((a[n - 1] >> (b - 1)) & 1)) --b;
        return (n - 1) * 32 + b;
    }
    static bool bit(const Big& a, int i) { return (i / 32 < (int)a.size()) && ((a[i / 32] >> (i % 32)) & 1); }
    static int cmp(const Big& a, const Big& b) {
        const size_t n = std::max(a.size(), b.size());
        for (size_t i = n; i-- > 0;) {
            const uint32_t x = i < a.size() ? a[i] : 0, y = i < b.size() ? b[i] : 0;
            if (x != y) return x < y ? -1 : 1;
        }
        return 0;
    }
    static void sub_in(Big& a, const Big& b) {  // a -= b (a >= b)
        int64_t borrow = 0;
        for (size_t i = 0; i < a.size(); ++i) {
            int64_t v = (int64_t)a[i] - (i < b.size() ? (int64_t)b[i] : 0) - borrow;
            borrow = v < 0;
            a[i] = (uint32_t)(v + (borrow ? (int64_t{1} << 32) : 0));
        }
    }
    static void shl1_add(Big& a, bool b) {  // a = 2a + b
        uint32_t carry = b ? 1u : 0u;
        for (auto& w : a) {
            const uint32_t nc = w >> 31;
            w = (w << 1) | carry;
            carry = nc;
        }
        if (carry) a.push_back(carry);
    }
    PowerTable() {
        for (int i = 0; i < kCount; ++i) {
            const int k = kMinDecExp + i * kStep;
            Big ten{1};
            for (int j = 0; j < (k < 0 ? -k : k); ++j) mul_small(ten, 10);
            uint64_t f = 0;
            int e = 0;
            if (k >= 0) {  // 10^k: the top 64 bits, rounded on the next bit
                const int L = bitlen(ten);
                const int shift = L - 64;
                if (shift <= 0) {
                    f = 0;
                    for (int b = L - 1; b >= 0; --b) f = (f << 1) | (bit(ten, b) ? 1 : 0);
                    f <<= -shift;
                    e = shift;
                } else {
                    for (int b = L - 1; b >= shift; --b) f = (f << 1) | (bit(ten, b) ? 1 : 0);
                    e = shift;
                    if (bit(ten, shift - 1)) {
                        ++f;
                        if (f == 0) {
                            f = uint64_t{1} << 63;
                            ++e;
                        }
                    }
                }
            } else {  // 10^k = 1 / 10^|k|: long division of 2^N by 10^|k|, 64 quotient bits + rounding
                const int L = bitlen(ten);
                // quotient of 2^(L + 63) / ten has 64 bits (2^(L-1) <= ten < 2^L)
                const int N = L + 63;
                Big rem{0};
                uint64_t q = 0;
                for (int b = N; b >= 0; --b) {
                    shl1_add(rem, b == N);
                    q <<= 1;
                    if (cmp(rem, ten) >= 0) {
                        sub_in(rem, ten);
                        q |= 1;
                    }
                }
                // q = floor(2^N / ten) in [2^63, 2^64); round on the remainder
                Big twice = rem;
                shl1_add(twice, false);
                f = q;
                e = -N;
                if (cmp(twice, ten) >= 0) {
                    ++f;
                    if (f == 0) {
                        f = uint64_t{1} << 63;
                        ++e;
                    }
                }
            }
            p_[i] = {f, e, k};
        }
    }
    CachedPower p_[kCount];
};

constexpr int kAlpha = -60, kGamma = -32;

inline CachedPower cached_power_for(int e) {
    const int f = kAlpha - e - 1;
    const int k = (f * 78913) / (1 << 18) + static_cast<int>(f > 0);  // ceil(f * log10(2))
    const int index = (-PowerTable::kMinDecExp + k + (PowerTable::kStep - 1)) / PowerTable::kStep;
    return PowerTable::get().at(index);
}

inline int largest_pow10(uint32_t n, uint32_t& pow10) {
    static const uint32_t p[] = {1u, 10u, 100u, 1000u, 10000u, 100000u, 1000000u, 10000000u, 100000000u, 1000000000u};
    int k = 10;
    while (k > 1 && n < p[k - 1]) --k;
    pow10 = p[k - 1];
    return k;
}

inline void round_weed(char* buf, int len, uint64_t dist, uint64_t delta, uint64_t rest, uint64_t ten_k) {
    while (rest < dist && delta - rest >= ten_k && (rest + ten_k < dist || dist - rest > rest + ten_k - dist)) {
        buf[len - 1]--;
        rest += ten_k;
    }
}

inline void digit_gen(char* buf, int& len, int& dec_exp, DiyFp M_minus, DiyFp w, DiyFp M_plus) {
    uint64_t delta = sub(M_plus, M_minus).f;
    uint64_t dist = sub(M_plus, w).f;
    const DiyFp one{uint64_t{1} << -M_plus.e, M_plus.e};
    uint32_t p1 = static_cast<uint32_t>(M_plus.f >> -one.e);
    uint64_t p2 = M_plus.f & (one.f - 1);
    uint32_t pow10 = 0;
    int n = largest_pow10(p1, pow10);
    while (n > 0) {
        const uint32_t d = p1 / pow10, r = p1 % pow10;
        buf[len++] = static_cast<char>('0' + d);
        p1 = r;
        n--;
        const uint64_t rest = (uint64_t{p1} << -one.e) + p2;
        if (rest <= delta) {
            dec_exp += n;
            round_weed(buf, len, dist, delta, rest, uint64_t{pow10} << -one.e);
            return;
        }
        pow10 /= 10;
    }
    int m = 0;
    for (;;) {
        p2 *= 10;
        const uint64_t d = p2 >> -one.e, r = p2 & (one.f - 1);
        buf[len++] = static_cast<char>('0' + d);
        p2 = r;
        m++;
        delta *= 10;
        dist *= 10;
        if (p2 <= delta) break;
    }
    dec_exp -= m;
    round_weed(buf, len, dist, delta, p2, one.f);
}

// digits of v > 0 into buf (no sign), len digits, value = digits * 10^dec_exp
inline void grisu2(char* buf, int& len, int& dec_exp, double value) {
    uint64_t bits;
    std::memcpy(&bits, &value, sizeof(bits));
    const uint64_t F = bits & ((uint64_t{1} << 52) - 1);
    const int E = static_cast<int>(bits >> 52) & 0x7FF;
    constexpr int kBias = 1075, kMinExp = 1 - kBias;
    const DiyFp v = E == 0 ? DiyFp{F, kMinExp} : DiyFp{F + (uint64_t{1} << 52), E - kBias};
    const bool lower_closer = F == 0 && E > 1;
    const DiyFp m_plus{2 * v.f + 1, v.e - 1};
    const DiyFp m_minus = lower_closer ? DiyFp{4 * v.f - 1, v.e - 2} : DiyFp{2 * v.f - 1, v.e - 1};
    const DiyFp w_plus = normalize(m_plus);
    const DiyFp w_minus = normalize_to(m_minus, w_plus.e);
    const DiyFp w = normalize(v);
    const CachedPower cp = cached_power_for(w_plus.e);
    const DiyFp c{cp.f, cp.e};
    const DiyFp W = mul(w, c), Wm = mul(w_minus, c), Wp = mul(w_plus, c);
    const DiyFp M_minus{Wm.f + 1, Wm.e}, M_plus{Wp.f - 1, Wp.e};
    len = 0;
    dec_exp = -cp.k;
    digit_gen(buf, len, dec_exp, M_minus, W, M_plus);
}

inline void append_exponent(std::string& out, int e) {
    out += e < 0 ? '-' : '+';
    const unsigned k = static_cast<unsigned>(e < 0 ? -e : e);
    if (k < 10) {
        out += '0';
        out += static_cast<char>('0' + k);
    } else if (k < 100) {
        out += static_cast<char>('0' + k / 10);
        out += static_cast<char>('0' + k % 10);
    } else {
        out += static_cast<char>('0' + k / 100);
        out += static_cast<char>('0' + (k / 10) % 10);
        out += static_cast<char>('0' + k % 10);
    }
}

// finite doubles only
inline void to_string(double value, std::string& out) {
    if (std::signbit(value)) {
        out += '-';
        value = -value;
    }
    if (value == 0.0) {
        out += "0.0";
        return;
    }
    char buf[32];
    int k = 0, dec_exp = 0;
    grisu2(buf, k, dec_exp, value);
    const int n = k + dec_exp;  // decimal point position
    constexpr int kMin = -4, kMax = 15;
    if (k <= n && n <= kMax) {  // digits, zeros, ".0"
        out.append(buf, k);
        out.append(n - k, '0');
        out += ".0";
    } else if (0 < n && n <= kMax) {  // dig.its
        out.append(buf, n);
        out += '.';
        out.append(buf + n, k - n);
    } else if (kMin < n && n <= 0) {  // 0.000digits
        out += "0.";
        out.append(-n, '0');
        out.append(buf, k);
    } else {  // d[.igits]e+-XX
        out += buf[0];
        if (k > 1) {
            out += '.';
            out.append(buf + 1, k - 1);
        }
        out += 'e';
        append_exponent(out, n - 1);
    }
}

}  // namespace asyrk::grisu2
