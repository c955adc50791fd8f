#pragma once
// Decimal -> binary64 conversion, correctly rounded (round half to even), for JSON number
// tokens: the value nlohmann::json's lexer obtains with std::strtod (serde.hpp record_from_json
// -> get<double>, via json::parse). Host + device: the JSONL ingest kernels (jsonl.cu) run it
// per feature value, and the CPU unit test (tests/test_decimal_cpu.py) compiles the same code
// against the C library's strtod.
//
//   1. <= 19 significant digits: w * 10^q exactly with the 128-bit normalised power-of-five
//      table (Eisel-Lemire; the 128-bit product always decides the rounding, Mushtak & Lemire);
//   2. more digits: w = the first 19 digits; if w and w + 1 round to the same double, done;
//   3. otherwise an exact big-integer comparison of the full digit string with the halfway
//      point between the two candidates (rare: inputs within 1e-19 relative of a tie).
#include <stdint.h>

#if defined(__CUDACC__)
#define LAT_HD __host__ __device__ __forceinline__
#define LAT_HDN __host__ __device__ __noinline__
#else
#define LAT_HD inline
#define LAT_HDN inline
#endif

namespace lat {
namespace dec {

#if defined(__CUDACC__)
__device__ const uint64_t d_pow5[] = {
#include "pow5_128.inc"
};
#endif
static const uint64_t h_pow5[] = {
#include "pow5_128.inc"
};

LAT_HD const uint64_t* pow5_table() {
#if defined(__CUDA_ARCH__)
    return d_pow5;
#else
    return h_pow5;
#endif
}

LAT_HD int clz64(uint64_t x) {
#if defined(__CUDA_ARCH__)
    return __clzll((long long)x);
#else
    return __builtin_clzll(x);
#endif
}

LAT_HD void mul128(uint64_t a, uint64_t b, uint64_t& hi, uint64_t& lo) {
#if defined(__CUDA_ARCH__)
    lo = a * b;
    hi = __umul64hi(a, b);
#else
    const unsigned __int128 p = (unsigned __int128)a * b;
    lo = (uint64_t)p;
    hi = (uint64_t)(p >> 64);
#endif
}

// Binary exponent (biased, 0 = zero/subnormal, 0x7FF = infinity) and 52-bit stored mantissa.
struct Fp {
    uint64_t mant;
    int32_t exp2;
};

// w * 10^q, w != 0, rounded to nearest even (fast_float's compute_float, restated).
LAT_HD Fp eisel_lemire(uint64_t w, int64_t q) {
    Fp r;
    if (w == 0 || q < -342) return Fp{0, 0};
    if (q > 308) return Fp{0, 0x7FF};
    const int lz = clz64(w);
    w <<= lz;
    const uint64_t* T = pow5_table() + 2 * (q + 342);
    uint64_t hi, lo;
    mul128(w, T[0], hi, lo);
    if ((hi & 0x1FF) == 0x1FF) {  // the low bits could carry: add the second product
        uint64_t h2, l2;
        mul128(w, T[1], h2, l2);
        lo += h2;
        if (h2 > lo) ++hi;
    }
    const int upper = (int)(hi >> 63);
    const int shift = upper + 9;
    r.mant = hi >> shift;
    // floor(log2(10^q)) + 63 = ((217706 * q) >> 16) + 63; minimum exponent -1023
    r.exp2 = (int32_t)((((152170 + 65536) * q) >> 16) + 63 + upper - lz + 1023);
    if (r.exp2 <= 0) {  // subnormal
        if (-r.exp2 + 1 >= 64) return Fp{0, 0};
        r.mant >>= -r.exp2 + 1;
        r.mant += r.mant & 1;
        r.mant >>= 1;
        r.exp2 = r.mant < (1ull << 52) ? 0 : 1;
        r.mant &= ~(1ull << 52);
        return r;
    }
    // exactly halfway (only possible for small |q|): round down to even
    if (lo <= 1 && q >= -4 && q <= 23 && (r.mant & 3) == 1 && (r.mant << shift) == hi) r.mant &= ~1ull;
    r.mant += r.mant & 1;
    r.mant >>= 1;
    if (r.mant >= (2ull << 52)) {
        r.mant = 1ull << 52;
        ++r.exp2;
    }
    r.mant &= ~(1ull << 52);
    if (r.exp2 >= 0x7FF) return Fp{0, 0x7FF};
    return r;
}

// ---- exact fallback: fixed-capacity unsigned big integers (32-bit limbs, little endian) ----
constexpr int kLimbs = 136;        // 4352 bits: 780 digits * 10^-1130 .. 10^310 fit
constexpr int kMaxExactDigits = 780;  // later digits only matter as "nonzero" (sticky)

struct Big {
    uint32_t l[kLimbs];
    int n;  // used limbs
};

LAT_HD void big_set(Big& b, uint64_t v) {
    b.l[0] = (uint32_t)v;
    b.l[1] = (uint32_t)(v >> 32);
    b.n = b.l[1] ? 2 : (b.l[0] ? 1 : 0);
}
LAT_HD void big_muladd(Big& b, uint32_t m, uint32_t a) {
    uint64_t carry = a;
    for (int i = 0; i < b.n; ++i) {
        const uint64_t t = (uint64_t)b.l[i] * m + carry;
        b.l[i] = (uint32_t)t;
        carry = t >> 32;
    }
    if (carry && b.n < kLimbs) b.l[b.n++] = (uint32_t)carry;
}
LAT_HD void big_mul_pow5(Big& b, int e) {
    while (e >= 13) {
        big_muladd(b, 1220703125u, 0);  // 5^13
        e -= 13;
    }
    uint32_t m = 1;
    while (e-- > 0) m *= 5;
    if (m > 1) big_muladd(b, m, 0);
}
LAT_HD void big_shl(Big& b, int s) {
    if (b.n == 0 || s <= 0) return;
    const int w = s >> 5, bits = s & 31;
    int n = b.n + w + 1;
    if (n > kLimbs) n = kLimbs;
    for (int i = n - 1; i >= 0; --i) {
        const int src = i - w;
        uint32_t v = 0;
        if (src >= 0 && src < b.n) v = bits ? b.l[src] << bits : b.l[src];
        if (bits && src - 1 >= 0 && src - 1 < b.n) v |= b.l[src - 1] >> (32 - bits);
        b.l[i] = v;
    }
    b.n = n;
    while (b.n > 0 && b.l[b.n - 1] == 0) --b.n;
}
LAT_HD int big_cmp(const Big& a, const Big& b) {
    if (a.n != b.n) return a.n < b.n ? -1 : 1;
    for (int i = a.n - 1; i >= 0; --i)
        if (a.l[i] != b.l[i]) return a.l[i] < b.l[i] ? -1 : 1;
    return 0;
}

LAT_HD uint64_t fp_bits(Fp f) { return ((uint64_t)f.exp2 << 52) | f.mant; }

LAT_HD Fp fp_next(Fp f) {
    if (f.exp2 >= 0x7FF) return f;
    ++f.mant;
    if (f.mant == (1ull << 52)) {
        f.mant = 0;
        ++f.exp2;
    }
    if (f.exp2 >= 0x7FF) return Fp{0, 0x7FF};
    return f;
}

// Exact decision between `lo` and its successor for the value digits * 10^e_last of the token
// [p, e) (the first kMaxExactDigits significant digits, the rest as a sticky bit).
LAT_HDN Fp exact_round(const uint8_t* p, const uint8_t* e, int64_t exp19, Fp lo) {
    Big A, B;
    big_set(A, 0);
    A.n = 0;
    int64_t taken = 0;
    bool sticky = false, started = false;
    uint32_t chunk = 0, cmul = 1;
    for (const uint8_t* q = p; q < e; ++q) {
        const uint8_t c = *q;
        if (c == '.') continue;
        if (c < '0' || c > '9') break;  // exponent part
        const uint32_t d = c - '0';
        if (!started && d == 0) continue;
        started = true;
        if (taken < kMaxExactDigits) {
            chunk = chunk * 10 + d;
            cmul *= 10;
            ++taken;
            if (cmul == 1000000000u) {
                big_muladd(A, cmul, chunk);
                if (A.n == 0 && chunk) big_set(A, chunk);
                chunk = 0;
                cmul = 1;
            }
        } else if (d) {
            sticky = true;
        }
    }
    if (cmul > 1) {
        big_muladd(A, cmul, chunk);
        if (A.n == 0 && chunk) big_set(A, chunk);
    }
    const int64_t eM = exp19 - (taken - 19);  // exponent of the last digit taken
    uint64_t M;
    int64_t E;
    if (lo.exp2 == 0) {
        M = lo.mant;
        E = -1074;
    } else {
        M = lo.mant | (1ull << 52);
        E = (int64_t)lo.exp2 - 1075;
    }
    big_set(B, 2 * M + 1);  // halfway point (2M + 1) * 2^(E - 1)
    int64_t a2 = 0, b2 = E - 1;
    if (eM >= 0) {
        big_mul_pow5(A, (int)eM);
        a2 = eM;
    } else {
        big_mul_pow5(B, (int)-eM);
        b2 += -eM;
    }
    if (a2 > b2)
        big_shl(A, (int)(a2 - b2));
    else
        big_shl(B, (int)(b2 - a2));
    int c = big_cmp(A, B);
    if (c == 0 && sticky) c = 1;
    if (c < 0) return lo;
    if (c > 0) return fp_next(lo);
    return (M & 1) ? fp_next(lo) : lo;
}

// Value of the validated JSON number token [p, e) (grammar -?(0|[1-9]\d*)(\.\d+)?([eE][+-]?\d+)?),
// as strtod rounds it.
LAT_HDN double parse_double(const uint8_t* p, const uint8_t* e) {
    const bool neg = p < e && *p == '-';
    if (neg) ++p;
    uint64_t w = 0;
    int nd = 0;
    int64_t exp10 = 0;
    bool trunc = false, started = false;
    const uint8_t* q = p;
    for (; q < e && *q >= '0' && *q <= '9'; ++q) {
        const int d = *q - '0';
        if (!started && d == 0) continue;
        started = true;
        if (nd < 19) {
            w = w * 10 + d;
            ++nd;
        } else {
            ++exp10;
            trunc |= d != 0;
        }
    }
    if (q < e && *q == '.') {
        for (++q; q < e && *q >= '0' && *q <= '9'; ++q) {
            const int d = *q - '0';
            if (!started && d == 0) {
                --exp10;
                continue;
            }
            started = true;
            if (nd < 19) {
                w = w * 10 + d;
                ++nd;
                --exp10;
            } else {
                trunc |= d != 0;
            }
        }
    }
    if (q < e && (*q == 'e' || *q == 'E')) {
        ++q;
        bool eneg = false;
        if (q < e && (*q == '+' || *q == '-')) eneg = *q++ == '-';
        int64_t ex = 0;
        for (; q < e && *q >= '0' && *q <= '9'; ++q)
            if (ex < 1000000) ex = ex * 10 + (*q - '0');
        exp10 += eneg ? -ex : ex;
    }
    double v;
    if (w == 0) {
        v = 0.0;
    } else if (!trunc && w <= (1ull << 53) && exp10 >= -22 && exp10 <= 22) {
        // Clinger's fast path: both operands exact, one IEEE rounding
        const double pw[23] = {1e0,  1e1,  1e2,  1e3,  1e4,  1e5,  1e6,  1e7,  1e8,  1e9,  1e10, 1e11,
                               1e12, 1e13, 1e14, 1e15, 1e16, 1e17, 1e18, 1e19, 1e20, 1e21, 1e22};
        v = exp10 >= 0 ? (double)w * pw[exp10] : (double)w / pw[-exp10];
    } else {
        Fp f = eisel_lemire(w, exp10);
        if (trunc) {
            const Fp g = eisel_lemire(w + 1, exp10);
            if (g.mant != f.mant || g.exp2 != f.exp2) f = exact_round(p, e, exp10, f);
        }
        const uint64_t bits = fp_bits(f);
#if defined(__CUDA_ARCH__)
        v = __longlong_as_double((long long)bits);
#else
        __builtin_memcpy(&v, &bits, 8);
#endif
    }
    return neg ? -v : v;
}

}  // namespace dec
}  // namespace lat
