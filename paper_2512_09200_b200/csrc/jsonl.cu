// jsonl.cu -- JSON-lines impression ingest ("JSONL impression ingest to
// columnar", the wire format in front of the Zipper). Replaces parse_jsonl_records +
// record_from_json (serde.hpp:129-194) for a whole file on the GPU:
//
//   lines    newline positions (cub select) -> [start, end) per line; getline semantics, a last
//            line without '\n' counts, blank lines (only " \t\r\n", serde.hpp detail::trim) are
//            skipped but keep their number for error context
//   pass 1   thread per line: full RFC 8259 validation as nlohmann::json::parse does it (UTF-8 BOM
//            skipped, well-formed UTF-8 and escapes incl. surrogate pairs, number grammar,
//            literals, nothing after the value), and the offset/type of the LAST occurrence of
//            each top-level field (duplicate keys: the last one wins, as in nlohmann's parser)
//   pass 2   thread per record: record_from_json's checks in its order (at() on a non-object,
//            missing key, get<string> / get<number> type errors) and the output sizes;
//            impression_time_ms converted (get<int64_t> of unsigned / integer / float / boolean)
//   pass 3   thread per record: unescaped UTF-8 strings, feature (key, double) and conversion
//            (key, int64) entries into caller-sized columns
//
// "features" / "conversions" follow nlohmann's items() for every value type: object members
// (a key repeated inside the object keeps its last value), array elements keyed "0", "1", ...,
// a primitive as one entry with the empty key, null as no entries. The first bad line (lowest
// number) is the error, as the reference's line loop throws there; messages carry the
// reference's "<source>:<line>: " context and nlohmann's exception texts for the record-level
// errors (parse errors are reported with their byte column, not nlohmann's full text --
// the reference's tests assert exception types only).
#include <cub/cub.cuh>
#include <thrust/iterator/counting_iterator.h>

#include <string>
#include <vector>

#include "common.cuh"
#include "decimal.cuh"

namespace lat {
namespace {

// value types (nlohmann type_name order is irrelevant; names below)
enum : uint8_t { T_NULL = 0, T_OBJ, T_ARR, T_STR, T_BOOL, T_UINT, T_INT, T_FLT, T_NONE = 255 };
enum { F_DOMAIN = 0, F_USER, F_AD, F_TS, F_FEAT, F_CONV, NFIELD };
// error codes (per line)
enum : int32_t {
    E_OK = 0,
    E_PARSE = 1,     // arg: reason
    E_NOT_OBJ = 2,   // at() on a non-object; arg: type
    E_MISSING = 3,   // arg: field
    E_TYPE = 4,      // arg: expected (0 string, 1 number) * 256 + actual type
    E_OVERFLOW = 5,  // col: token offset in the line, arg: token length
};
enum : int32_t {
    P_END = 1,      // unexpected end of input
    P_CHAR,         // unexpected character
    P_STRING,       // invalid string (control character, escape, UTF-8, unterminated)
    P_NUMBER,       // invalid number
    P_LITERAL,      // invalid literal
    P_DEPTH,        // nesting deeper than kMaxDepth (a limit of this parser, not of JSON)
    P_TRAILING,     // content after the top-level value
    P_OVERFLOW,     // a number literal overflowing binary64 (nlohmann out_of_range.406)
};
constexpr int kMaxDepth = 256;

__device__ __forceinline__ bool is_ws(uint8_t c) { return c == ' ' || c == '\t' || c == '\n' || c == '\r'; }
__device__ __forceinline__ int hexv(uint8_t c) {
    return c >= '0' && c <= '9' ? c - '0' : c >= 'a' && c <= 'f' ? c - 'a' + 10 : c >= 'A' && c <= 'F' ? c - 'A' + 10 : -1;
}
__device__ __forceinline__ int hex4(const uint8_t* s, uint32_t i, uint32_t n) {
    if (i + 4 > n) return -1;
    int v = 0;
    for (int k = 0; k < 4; ++k) {
        const int h = hexv(s[i + k]);
        if (h < 0) return -1;
        v = v * 16 + h;
    }
    return v;
}
__device__ __forceinline__ int utf8_len(uint32_t cp) { return cp < 0x80 ? 1 : cp < 0x800 ? 2 : cp < 0x10000 ? 3 : 4; }

// Validates the string starting at s[i] == '"'; i ends after the closing quote. Returns the
// unescaped UTF-8 length, or -1 (error, i at the offending byte).
__device__ int64_t scan_string(const uint8_t* s, uint32_t n, uint32_t& i) {
    int64_t len = 0;
    ++i;
    while (true) {
        if (i >= n) return -1;
        const uint8_t c = s[i];
        if (c == '"') {
            ++i;
            return len;
        }
        if (c < 0x20) return -1;
        if (c == '\\') {
            if (i + 1 >= n) return -1;
            const uint8_t e = s[i + 1];
            if (e == 'u') {
                int cp = hex4(s, i + 2, n);
                if (cp < 0) return -1;
                i += 6;
                if (cp >= 0xD800 && cp <= 0xDBFF) {
                    if (i + 1 >= n || s[i] != '\\' || s[i + 1] != 'u') return -1;
                    const int lo = hex4(s, i + 2, n);
                    if (lo < 0xDC00 || lo > 0xDFFF) return -1;
                    i += 6;
                    cp = 0x10000 + ((cp - 0xD800) << 10) + (lo - 0xDC00);
                } else if (cp >= 0xDC00 && cp <= 0xDFFF) {
                    return -1;
                }
                len += utf8_len((uint32_t)cp);
                continue;
            }
            if (e != '"' && e != '\\' && e != '/' && e != 'b' && e != 'f' && e != 'n' && e != 'r' && e != 't')
                return -1;
            i += 2;
            ++len;
            continue;
        }
        if (c < 0x80) {
            ++i;
            ++len;
            continue;
        }
        // well-formed UTF-8 (RFC 3629 table, as nlohmann's lexer checks it)
        int extra;
        uint8_t lo = 0x80, hi = 0xBF;
        if (c >= 0xC2 && c <= 0xDF) {
            extra = 1;
        } else if (c == 0xE0) {
            extra = 2;
            lo = 0xA0;
        } else if ((c >= 0xE1 && c <= 0xEC) || c == 0xEE || c == 0xEF) {
            extra = 2;
        } else if (c == 0xED) {
            extra = 2;
            hi = 0x9F;
        } else if (c == 0xF0) {
            extra = 3;
            lo = 0x90;
        } else if (c >= 0xF1 && c <= 0xF3) {
            extra = 3;
        } else if (c == 0xF4) {
            extra = 3;
            hi = 0x8F;
        } else {
            return -1;
        }
        if (i + extra >= n) return -1;
        for (int k = 1; k <= extra; ++k) {
            const uint8_t b = s[i + k];
            if (k == 1 ? (b < lo || b > hi) : (b < 0x80 || b > 0xBF)) return -1;
        }
        i += 1 + extra;
        len += 1 + extra;
    }
}

// Bytes of a validated string (s[i] == '"') with the escapes decoded, one at a time.
struct UIter {
    const uint8_t* s;
    uint32_t i;
    uint8_t buf[4];
    int nb, bi;
    __device__ UIter(const uint8_t* s_, uint32_t open_quote) : s(s_), i(open_quote + 1), nb(0), bi(0) {}
    __device__ int next() {
        if (bi < nb) return buf[bi++];
        const uint8_t c = s[i];
        if (c == '"') return -1;
        if (c != '\\') {
            ++i;
            return c;
        }
        const uint8_t e = s[i + 1];
        i += 2;
        switch (e) {
            case 'b': return 8;
            case 'f': return 12;
            case 'n': return 10;
            case 'r': return 13;
            case 't': return 9;
            case 'u': break;
            default: return e;  // " \ /
        }
        uint32_t cp = (uint32_t)hex4(s, i, 0xffffffffu);
        i += 4;
        if (cp >= 0xD800 && cp <= 0xDBFF) {
            const uint32_t lo = (uint32_t)hex4(s, i + 2, 0xffffffffu);
            i += 6;
            cp = 0x10000 + ((cp - 0xD800) << 10) + (lo - 0xDC00);
        }
        if (cp < 0x80) return (int)cp;
        if (cp < 0x800) {
            buf[0] = (uint8_t)(0xC0 | (cp >> 6));
            buf[1] = (uint8_t)(0x80 | (cp & 0x3F));
            nb = 2;
        } else if (cp < 0x10000) {
            buf[0] = (uint8_t)(0xE0 | (cp >> 12));
            buf[1] = (uint8_t)(0x80 | ((cp >> 6) & 0x3F));
            buf[2] = (uint8_t)(0x80 | (cp & 0x3F));
            nb = 3;
        } else {
            buf[0] = (uint8_t)(0xF0 | (cp >> 18));
            buf[1] = (uint8_t)(0x80 | ((cp >> 12) & 0x3F));
            buf[2] = (uint8_t)(0x80 | ((cp >> 6) & 0x3F));
            buf[3] = (uint8_t)(0x80 | (cp & 0x3F));
            nb = 4;
        }
        bi = 1;
        return buf[0];
    }
};

// Byte-wise comparison of two validated strings' decoded values (std::string ordering).
__device__ int str_cmp(const uint8_t* s, uint32_t a, uint32_t b) {
    UIter x(s, a), y(s, b);
    while (true) {
        const int p = x.next(), q = y.next();
        if (p != q) return p < q ? -1 : 1;
        if (p < 0) return 0;
    }
}
__device__ bool str_eq_lit(const uint8_t* s, uint32_t a, const char* lit) {
    UIter x(s, a);
    for (int k = 0;; ++k) {
        const int p = x.next();
        const int q = lit[k] ? (uint8_t)lit[k] : -1;
        if (p != q) return false;
        if (p < 0) return true;
    }
}

// JSON number grammar from s[i]; type T_UINT / T_INT (fits uint64 / int64) or T_FLT.
__device__ bool scan_number(const uint8_t* s, uint32_t n, uint32_t& i, uint8_t& type) {
    const uint32_t st = i;
    bool neg = false, flt = false;
    if (s[i] == '-') {
        neg = true;
        ++i;
    }
    if (i >= n) return false;
    if (s[i] == '0') {
        ++i;
    } else if (s[i] >= '1' && s[i] <= '9') {
        while (i < n && s[i] >= '0' && s[i] <= '9') ++i;
    } else {
        return false;
    }
    const uint32_t int_end = i;
    if (i < n && s[i] == '.') {
        flt = true;
        ++i;
        if (i >= n || s[i] < '0' || s[i] > '9') return false;
        while (i < n && s[i] >= '0' && s[i] <= '9') ++i;
    }
    if (i < n && (s[i] == 'e' || s[i] == 'E')) {
        flt = true;
        ++i;
        if (i < n && (s[i] == '+' || s[i] == '-')) ++i;
        if (i >= n || s[i] < '0' || s[i] > '9') return false;
        while (i < n && s[i] >= '0' && s[i] <= '9') ++i;
    }
    if (flt) {
        type = T_FLT;
        return true;
    }
    // integer: in range of int64 (negative) / uint64 (non-negative), else a float
    const uint32_t d0 = st + (neg ? 1 : 0), nd = int_end - d0;
    const char* lim = neg ? "9223372036854775808" : "18446744073709551615";
    const uint32_t ln = neg ? 19 : 20;
    bool fits = nd < ln;
    if (nd == ln) {
        fits = true;
        for (uint32_t k = 0; k < ln; ++k) {
            if (s[d0 + k] != (uint8_t)lim[k]) {
                fits = s[d0 + k] < (uint8_t)lim[k];
                break;
            }
        }
    }
    type = !fits ? T_FLT : neg ? T_INT : T_UINT;
    return true;
}

__device__ bool scan_literal(const uint8_t* s, uint32_t n, uint32_t& i, uint8_t& type) {
    const char* lit = s[i] == 't' ? "true" : s[i] == 'f' ? "false" : "null";
    type = s[i] == 'n' ? T_NULL : T_BOOL;
    for (int k = 0; lit[k]; ++k, ++i)
        if (i >= n || s[i] != (uint8_t)lit[k]) return false;
    return true;
}

// Validates one value from s[i] (after whitespace); i ends after it. Returns 0 or a P_* reason.
// OVF: also reject float literals that overflow (pass 1; later passes walk validated lines).
template <bool OVF = true>
__device__ int skip_value(const uint8_t* s, uint32_t n, uint32_t& i, uint8_t& type) {
    uint32_t stk[kMaxDepth / 32];  // bit per level: 1 = object
    int depth = 0;
    bool first = true;
    while (true) {
        // ---- expect a value
        while (i < n && is_ws(s[i])) ++i;
        if (i >= n) return P_END;
        uint8_t c = s[i], t;
        bool opened = false;
        if (c == '{' || c == '[') {
            if (depth >= kMaxDepth) return P_DEPTH;
            const bool obj = c == '{';
            if (obj)
                stk[depth >> 5] |= 1u << (depth & 31);
            else
                stk[depth >> 5] &= ~(1u << (depth & 31));
            ++depth;
            ++i;
            t = obj ? T_OBJ : T_ARR;
            opened = true;
        } else if (c == '"') {
            if (scan_string(s, n, i) < 0) return P_STRING;
            t = T_STR;
        } else if (c == '-' || (c >= '0' && c <= '9')) {
            const uint32_t tok = i;
            if (!scan_number(s, n, i, t)) return P_NUMBER;
            // nlohmann's parser rejects a float literal that overflows (the SAX number_float
            // callback, before anything after the token is looked at); i is left at the token
            if (OVF && t == T_FLT && isinf(dec::parse_double(s + tok, s + i))) {
                i = tok;
                return P_OVERFLOW;
            }
        } else if (c == 't' || c == 'f' || c == 'n') {
            if (!scan_literal(s, n, i, t)) return P_LITERAL;
        } else {
            return P_CHAR;
        }
        if (first) {
            type = t;
            first = false;
        }
        bool need_value = false;
        if (opened) {
            while (i < n && is_ws(s[i])) ++i;
            if (i >= n) return P_END;
            const bool obj = (stk[(depth - 1) >> 5] >> ((depth - 1) & 31)) & 1u;
            if (s[i] == (obj ? '}' : ']')) {
                ++i;
                --depth;
            } else if (obj) {
                if (s[i] != '"') return P_CHAR;
                if (scan_string(s, n, i) < 0) return P_STRING;
                while (i < n && is_ws(s[i])) ++i;
                if (i >= n) return P_END;
                if (s[i] != ':') return P_CHAR;
                ++i;
                need_value = true;
            } else {
                need_value = true;
            }
        }
        // ---- after a value: close containers / continue lists
        while (!need_value) {
            if (depth == 0) return 0;
            while (i < n && is_ws(s[i])) ++i;
            if (i >= n) return P_END;
            const bool obj = (stk[(depth - 1) >> 5] >> ((depth - 1) & 31)) & 1u;
            c = s[i];
            if (c == ',') {
                ++i;
                if (obj) {
                    while (i < n && is_ws(s[i])) ++i;
                    if (i >= n) return P_END;
                    if (s[i] != '"') return P_CHAR;
                    if (scan_string(s, n, i) < 0) return P_STRING;
                    while (i < n && is_ws(s[i])) ++i;
                    if (i >= n) return P_END;
                    if (s[i] != ':') return P_CHAR;
                    ++i;
                }
                need_value = true;
            } else if (c == (obj ? '}' : ']')) {
                ++i;
                --depth;
            } else {
                return P_CHAR;
            }
        }
    }
}

struct Lines {
    const uint8_t* content;
    const int64_t* start;  // [L]
    const int64_t* end;    // [L]
};

__device__ __forceinline__ void fail(int32_t* code, int32_t* col, int32_t* arg, unsigned long long* first, int64_t ln,
                                     int32_t c, int32_t column, int32_t a) {
    code[ln] = c;
    col[ln] = column;
    arg[ln] = a;
    atomicMin(first, (unsigned long long)ln);
}

__device__ uint32_t number_end(const uint8_t* s, uint32_t n, uint32_t i);

// a skip_value failure: a syntax error at i, or the overflowing number literal starting at i
__device__ void fail_value(const uint8_t* s, uint32_t n, uint32_t i, int r, int32_t* code, int32_t* col, int32_t* arg,
                           unsigned long long* first, int64_t ln) {
    if (r == P_OVERFLOW) return fail(code, col, arg, first, ln, E_OVERFLOW, (int)i, (int)(number_end(s, n, i) - i));
    fail(code, col, arg, first, ln, E_PARSE, (int)i + 1, r);
}

// ---- pass 1 ---------------------------------------------------------------------------
__global__ void pass1_kernel(Lines L, int64_t nlines, uint32_t* loc_off, uint8_t* loc_type, uint8_t* top_type,
                             int32_t* is_rec, int32_t* code, int32_t* col, int32_t* arg, unsigned long long* first) {
    const int64_t ln = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (ln >= nlines) return;
    const uint8_t* s = L.content + L.start[ln];
    const uint32_t n = (uint32_t)(L.end[ln] - L.start[ln]);
    code[ln] = E_OK;
    is_rec[ln] = 0;
    bool blank = true;  // detail::trim: only " \t\r\n"
    for (uint32_t k = 0; k < n && blank; ++k) blank = is_ws(s[k]);
    if (blank) return;
    uint32_t i = 0;
    if (n >= 3 && s[0] == 0xEF && s[1] == 0xBB && s[2] == 0xBF) i = 3;  // nlohmann skips a UTF-8 BOM
    for (int f = 0; f < NFIELD; ++f) loc_type[ln * NFIELD + f] = T_NONE;
    while (i < n && is_ws(s[i])) ++i;
    if (i >= n) return fail(code, col, arg, first, ln, E_PARSE, (int)i + 1, P_END);
    uint8_t top;
    if (s[i] == '{') {
        top = T_OBJ;
        ++i;
        while (i < n && is_ws(s[i])) ++i;
        if (i >= n) return fail(code, col, arg, first, ln, E_PARSE, (int)i + 1, P_END);
        if (s[i] == '}') {
            ++i;
        } else {
            while (true) {
                if (s[i] != '"') return fail(code, col, arg, first, ln, E_PARSE, (int)i + 1, P_CHAR);
                const uint32_t kq = i;
                if (scan_string(s, n, i) < 0) return fail(code, col, arg, first, ln, E_PARSE, (int)i + 1, P_STRING);
                int fid = -1;
                if (str_eq_lit(s, kq, "domain")) fid = F_DOMAIN;
                else if (str_eq_lit(s, kq, "user_id")) fid = F_USER;
                else if (str_eq_lit(s, kq, "ad_id")) fid = F_AD;
                else if (str_eq_lit(s, kq, "impression_time_ms")) fid = F_TS;
                else if (str_eq_lit(s, kq, "features")) fid = F_FEAT;
                else if (str_eq_lit(s, kq, "conversions")) fid = F_CONV;
                while (i < n && is_ws(s[i])) ++i;
                if (i >= n) return fail(code, col, arg, first, ln, E_PARSE, (int)i + 1, P_END);
                if (s[i] != ':') return fail(code, col, arg, first, ln, E_PARSE, (int)i + 1, P_CHAR);
                ++i;
                while (i < n && is_ws(s[i])) ++i;
                const uint32_t vs = i;
                uint8_t vt = T_NONE;
                const int r = skip_value(s, n, i, vt);
                if (r) return fail_value(s, n, i, r, code, col, arg, first, ln);
                if (fid >= 0) {  // the last occurrence wins
                    loc_off[ln * NFIELD + fid] = vs;
                    loc_type[ln * NFIELD + fid] = vt;
                }
                while (i < n && is_ws(s[i])) ++i;
                if (i >= n) return fail(code, col, arg, first, ln, E_PARSE, (int)i + 1, P_END);
                if (s[i] == '}') {
                    ++i;
                    break;
                }
                if (s[i] != ',') return fail(code, col, arg, first, ln, E_PARSE, (int)i + 1, P_CHAR);
                ++i;
                while (i < n && is_ws(s[i])) ++i;
                if (i >= n) return fail(code, col, arg, first, ln, E_PARSE, (int)i + 1, P_END);
            }
        }
    } else {
        const int r = skip_value(s, n, i, top);
        if (r) return fail_value(s, n, i, r, code, col, arg, first, ln);
    }
    while (i < n && is_ws(s[i])) ++i;
    if (i < n) return fail(code, col, arg, first, ln, E_PARSE, (int)i + 1, P_TRAILING);
    top_type[ln] = top;
    is_rec[ln] = 1;
}

// ---- value conversions (nlohmann get<T> of a number / boolean) --------------------------------
__device__ uint64_t parse_u64(const uint8_t* s, uint32_t i) {
    uint64_t v = 0;
    while (s[i] >= '0' && s[i] <= '9') v = v * 10 + (s[i++] - '0');
    return v;
}
__device__ uint32_t number_end(const uint8_t* s, uint32_t n, uint32_t i) {
    uint8_t t;
    scan_number(s, n, i, t);
    return i;
}
// get<int64_t>: unsigned -> two's complement cast, float -> static_cast (x86 cvttsd2si: out of
// range -> INT64_MIN)
__device__ int64_t value_i64(const uint8_t* s, uint32_t n, uint32_t i, uint8_t t) {
    switch (t) {
        case T_UINT: return (int64_t)parse_u64(s, i);
        case T_INT: return (int64_t)(0ull - parse_u64(s, i + 1));
        default: {
            const double d = dec::parse_double(s + i, s + number_end(s, n, i));
            if (!(d >= -9223372036854775808.0 && d < 9223372036854775808.0)) return INT64_MIN;
            return (int64_t)d;
        }
    }
}
__device__ double value_f64(const uint8_t* s, uint32_t n, uint32_t i, uint8_t t) {
    switch (t) {
        case T_UINT: return __ull2double_rn(parse_u64(s, i));
        case T_INT: return __ll2double_rn((long long)(0ull - parse_u64(s, i + 1)));
        default: return dec::parse_double(s + i, s + number_end(s, n, i));
    }
}
// get<double> / get<int64_t> accept the three number kinds only (a boolean is a type_error.302)
__device__ __forceinline__ bool is_number(uint8_t t) { return t == T_UINT || t == T_INT || t == T_FLT; }

__device__ __forceinline__ uint8_t peek_type(const uint8_t* s, uint32_t i) {
    const uint8_t c = s[i];
    if (c == '{') return T_OBJ;
    if (c == '[') return T_ARR;
    if (c == '"') return T_STR;
    if (c == 't' || c == 'f') return T_BOOL;
    if (c == 'n') return T_NULL;
    return T_FLT;  // number (exact kind from scan_number when needed)
}

// Entries of a features / conversions value (nlohmann items()). Visits entries in document
// order, skipping object members whose key repeats later in the object; fn(key_kind, key_pos,
// index, value_pos) with key_kind 0 = object member (key string at key_pos), 1 = array element
// (key = decimal index), 2 = primitive (empty key).
template <typename Fn>
__device__ void for_entries(const uint8_t* s, uint32_t n, uint32_t vpos, Fn&& fn) {
    const uint8_t t = peek_type(s, vpos);
    if (t == T_NULL) return;
    if (t != T_OBJ && t != T_ARR) {
        fn(2, 0u, 0ll, vpos);
        return;
    }
    uint32_t i = vpos + 1;
    int64_t idx = 0;
    while (i < n && is_ws(s[i])) ++i;
    if (s[i] == (t == T_OBJ ? '}' : ']')) return;
    while (true) {
        uint32_t kq = 0;
        if (t == T_OBJ) {
            kq = i;
            scan_string(s, n, i);
            while (is_ws(s[i])) ++i;
            ++i;  // ':'
            while (is_ws(s[i])) ++i;
        }
        const uint32_t vs = i;
        uint8_t vt;
        skip_value<false>(s, n, i, vt);
        bool last = true;
        if (t == T_OBJ) {  // a later member with the same key replaces this one
            uint32_t j = i;
            while (true) {
                while (is_ws(s[j])) ++j;
                if (s[j] != ',') break;
                ++j;
                while (is_ws(s[j])) ++j;
                const uint32_t kq2 = j;
                scan_string(s, n, j);
                if (str_cmp(s, kq, kq2) == 0) {
                    last = false;
                    break;
                }
                while (is_ws(s[j])) ++j;
                ++j;
                uint8_t t2;
                skip_value<false>(s, n, j, t2);
            }
        }
        if (last) fn(t == T_OBJ ? 0 : 1, kq, idx, vs);
        ++idx;
        while (is_ws(s[i])) ++i;
        if (s[i] != ',') return;
        ++i;
        while (is_ws(s[i])) ++i;
    }
}

__device__ __forceinline__ int dec_len(int64_t v) {
    int l = 1;
    while (v >= 10) {
        v /= 10;
        ++l;
    }
    return l;
}

// value type of a validated value at s[i] (numbers classified exactly)
__device__ uint8_t value_type(const uint8_t* s, uint32_t n, uint32_t i) {
    uint8_t t = peek_type(s, i);
    if (t == T_FLT) scan_number(s, n, i, t);
    return t;
}

struct RecSizes {
    int64_t* len[3];   // domain / user / ad unescaped bytes
    int64_t* fcnt;     // feature entries
    int64_t* fkey;     // feature key bytes
    int64_t* ccnt;
    int64_t* ckey;
};

// ---- pass 2 ---------------------------------------------------------------------------
__global__ void pass2_kernel(Lines L, int64_t nlines, const int32_t* is_rec, const int32_t* rec_of_line,
                             const uint32_t* loc_off, const uint8_t* loc_type, const uint8_t* top_type,
                             RecSizes sz, int64_t* ts, int64_t* rec_line, int32_t* code, int32_t* col, int32_t* arg,
                             unsigned long long* first) {
    const int64_t ln = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (ln >= nlines || !is_rec[ln]) return;
    const int64_t r = rec_of_line[ln];
    rec_line[r] = ln + 1;
    const uint8_t* s = L.content + L.start[ln];
    const uint32_t n = (uint32_t)(L.end[ln] - L.start[ln]);
    for (int k = 0; k < 3; ++k) sz.len[k][r] = 0;
    sz.fcnt[r] = sz.fkey[r] = sz.ccnt[r] = sz.ckey[r] = 0;
    ts[r] = 0;
    if (top_type[ln] != T_OBJ) return fail(code, col, arg, first, ln, E_NOT_OBJ, 0, top_type[ln]);
    const uint32_t* off = loc_off + ln * NFIELD;
    const uint8_t* typ = loc_type + ln * NFIELD;
    for (int f = F_DOMAIN; f <= F_AD; ++f) {  // at(...).get<std::string>() in record_from_json order
        if (typ[f] == T_NONE) return fail(code, col, arg, first, ln, E_MISSING, 0, f);
        if (typ[f] != T_STR) return fail(code, col, arg, first, ln, E_TYPE, 0, 0 * 256 + typ[f]);
        uint32_t i = off[f];
        sz.len[f][r] = scan_string(s, n, i);
    }
    if (typ[F_TS] == T_NONE) return fail(code, col, arg, first, ln, E_MISSING, 0, F_TS);
    if (!is_number(typ[F_TS])) return fail(code, col, arg, first, ln, E_TYPE, 0, 1 * 256 + typ[F_TS]);
    ts[r] = value_i64(s, n, off[F_TS], typ[F_TS]);
    for (int f = F_FEAT; f <= F_CONV; ++f) {
        if (typ[f] == T_NONE) continue;  // contains() false
        int64_t cnt = 0, kb = 0;
        // the first bad value in items() order: object members in key order, arrays by index
        int bad_type = -1;
        uint32_t bad_key = 0;
        for_entries(s, n, off[f], [&](int kk, uint32_t kq, int64_t idx, uint32_t vs) {
            const uint8_t vt = value_type(s, n, vs);
            if (!is_number(vt)) {
                if (bad_type < 0 || (kk == 0 && str_cmp(s, kq, bad_key) < 0)) {
                    bad_type = vt;
                    bad_key = kq;
                }
                return;
            }
            ++cnt;
            if (kk == 0) {
                uint32_t q = kq;
                kb += scan_string(s, n, q);
            } else if (kk == 1) {
                kb += dec_len(idx);
            }
        });
        if (bad_type >= 0) return fail(code, col, arg, first, ln, E_TYPE, 0, 1 * 256 + bad_type);
        if (f == F_FEAT) {
            sz.fcnt[r] = cnt;
            sz.fkey[r] = kb;
        } else {
            sz.ccnt[r] = cnt;
            sz.ckey[r] = kb;
        }
    }
}

struct RecOut {
    uint8_t* str[3];
    const int64_t* str_off[3];
    const int64_t* f_off;  // entry offsets [N+1]
    const int64_t* fk_off; // per-record key byte offsets [N+1]
    uint8_t* f_key;
    int64_t* f_key_off;    // [E+1] (per entry)
    double* f_val;
    const int64_t* c_off;
    const int64_t* ck_off;
    uint8_t* c_key;
    int64_t* c_key_off;
    int64_t* c_val;
};

__device__ int64_t write_key(const uint8_t* s, int kk, uint32_t kq, int64_t idx, uint8_t* dst) {
    if (kk == 2) return 0;
    if (kk == 1) {
        const int l = dec_len(idx);
        for (int k = l - 1; k >= 0; --k) {
            dst[k] = (uint8_t)('0' + idx % 10);
            idx /= 10;
        }
        return l;
    }
    UIter it(s, kq);
    int64_t l = 0;
    for (int c = it.next(); c >= 0; c = it.next()) dst[l++] = (uint8_t)c;
    return l;
}

// ---- pass 3 ---------------------------------------------------------------------------
__global__ void pass3_kernel(Lines L, int64_t nlines, const int32_t* is_rec, const int32_t* rec_of_line,
                             const uint32_t* loc_off, const uint8_t* loc_type, RecOut o) {
    const int64_t ln = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (ln >= nlines || !is_rec[ln]) return;
    const int64_t r = rec_of_line[ln];
    const uint8_t* s = L.content + L.start[ln];
    const uint32_t n = (uint32_t)(L.end[ln] - L.start[ln]);
    const uint32_t* off = loc_off + ln * NFIELD;
    const uint8_t* typ = loc_type + ln * NFIELD;
    for (int f = F_DOMAIN; f <= F_AD; ++f) {
        if (!o.str[f]) continue;
        uint8_t* d = o.str[f] + o.str_off[f][r];
        UIter it(s, off[f]);
        for (int c = it.next(); c >= 0; c = it.next()) *d++ = (uint8_t)c;
    }
    for (int f = F_FEAT; f <= F_CONV; ++f) {
        if (typ[f] == T_NONE) continue;
        const bool feat = f == F_FEAT;
        if (feat ? !o.f_key : !o.c_key) continue;
        int64_t e = feat ? o.f_off[r] : o.c_off[r];
        int64_t kb = feat ? o.fk_off[r] : o.ck_off[r];
        for_entries(s, n, off[f], [&](int kk, uint32_t kq, int64_t idx, uint32_t vs) {
            const uint8_t vt = value_type(s, n, vs);
            const int64_t l = write_key(s, kk, kq, idx, (feat ? o.f_key : o.c_key) + kb);
            if (feat) {
                o.f_key_off[e] = kb;
                o.f_val[e] = value_f64(s, n, vs, vt);
            } else {
                o.c_key_off[e] = kb;
                o.c_val[e] = value_i64(s, n, vs, vt);
            }
            kb += l;
            ++e;
        });
    }
}

__global__ void lines_kernel(const int64_t* nl, int64_t n_nl, int64_t bytes, int64_t nlines, int64_t* start, int64_t* end) {
    const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k >= nlines) return;
    start[k] = k == 0 ? 0 : nl[k - 1] + 1;
    end[k] = k < n_nl ? nl[k] : bytes;
}

__global__ void tail_kernel(int64_t* off, int64_t n, const int64_t* total_src) {
    // off[n] = total (exclusive scan + last element)
    if (threadIdx.x == 0 && blockIdx.x == 0) off[n] = *total_src;
}

struct IsNewline {
    const uint8_t* c;
    __host__ __device__ bool operator()(int64_t i) const { return c[i] == '\n'; }
};

// task-column kernel: conv[r][t] / present[r][t] from the record's conversion entries
__global__ void task_kernel(int64_t n, const int64_t* c_off, const uint8_t* c_key, const int64_t* c_key_off,
                            const int64_t* c_val, int32_t T, const uint8_t* task_bytes, const int64_t* task_off,
                            int64_t* conv, uint8_t* present) {
    const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (r >= n) return;
    for (int t = 0; t < T; ++t) {
        const int64_t tl = task_off[t + 1] - task_off[t];
        const uint8_t* tb = task_bytes + task_off[t];
        int64_t v = 0;
        uint8_t p = 0;
        for (int64_t e = c_off[r]; e < c_off[r + 1]; ++e) {
            const int64_t kl = c_key_off[e + 1] - c_key_off[e];
            if (kl != tl) continue;
            const uint8_t* kb = c_key + c_key_off[e];
            bool eq = true;
            for (int64_t q = 0; q < kl && eq; ++q) eq = kb[q] == tb[q];
            if (eq) {  // keys are unique per record (duplicates were resolved at parse time)
                v = c_val[e];
                p = 1;
            }
        }
        conv[r * T + t] = v;
        present[r * T + t] = p;
    }
}

}  // namespace
}  // namespace lat

struct lattice_jsonl {
    const uint8_t* content = nullptr;
    int64_t bytes = 0, lines = 0, records = 0;
    int64_t *start = nullptr, *end = nullptr;
    uint32_t* loc_off = nullptr;
    uint8_t *loc_type = nullptr, *top_type = nullptr;
    int32_t *is_rec = nullptr, *rec_of_line = nullptr;
    int64_t* rec_line = nullptr;
    int64_t* ts = nullptr;
    int64_t* off[7] = {};  // exclusive-scan offsets [records + 1]: domain, user, ad, fcnt, fkey, ccnt, ckey
    cudaStream_t stream = nullptr;  // the open call's stream: allocations are ordered on it
    std::vector<void*> allocs;
};

namespace {

using lat::set_error;

// stream-ordered pool allocations: an ingest call allocates ~30 arrays, and plain cudaMalloc /
// cudaFree (which synchronises the device) cost more than the kernels themselves
template <typename T>
lattice_status jl_alloc(lattice_jsonl* h, T** p, int64_t count) {
    void* q = nullptr;
    LAT_CUDA(cudaMallocAsync(&q, (size_t)(count > 0 ? count : 1) * sizeof(T), h->stream));
    h->allocs.push_back(q);
    *p = static_cast<T*>(q);
    return LATTICE_OK;
}

const char* type_name(int t) {
    switch (t) {
        case lat::T_NULL: return "null";
        case lat::T_OBJ: return "object";
        case lat::T_ARR: return "array";
        case lat::T_STR: return "string";
        case lat::T_BOOL: return "boolean";
        default: return "number";
    }
}

std::string error_text(int32_t code, int32_t col, int32_t arg) {
    static const char* fields[] = {"domain", "user_id", "ad_id", "impression_time_ms", "features", "conversions"};
    switch (code) {
        case lat::E_PARSE: {
            static const char* why[] = {"", "unexpected end of input", "unexpected character",
                                        "invalid string", "invalid number", "invalid literal",
                                        "nesting too deep for the GPU parser", "unexpected content after the value"};
            return "[json.exception.parse_error.101] parse error at line 1, column " + std::to_string(col) +
                   ": syntax error while parsing value - " + why[arg >= 1 && arg <= 7 ? arg : 0];
        }
        case lat::E_NOT_OBJ: return std::string("[json.exception.type_error.304] cannot use at() with ") + type_name(arg);
        case lat::E_MISSING:
            return std::string("[json.exception.out_of_range.403] key '") + fields[arg] + "' not found";
        case lat::E_TYPE:
            return std::string("[json.exception.type_error.302] type must be ") + ((arg >> 8) ? "number" : "string") +
                   ", but is " + type_name(arg & 0xff);
        default: return "unknown error";
    }
}

template <typename Fn>
lattice_status with_temp(size_t bytes, cudaStream_t st, Fn&& fn) {
    void* tmp = nullptr;
    LAT_CUDA(cudaMallocAsync(&tmp, bytes ? bytes : 16, st));
    lattice_status s = fn(tmp);
    cudaFreeAsync(tmp, st);
    return s;
}

lattice_status exclusive_offsets(const int64_t* in, int64_t* out, int64_t n, cudaStream_t st) {
    // out[0] = 0, out[k + 1] = sum in[0..k]
    LAT_CUDA(cudaMemsetAsync(out, 0, sizeof(int64_t), st));
    if (n == 0) return LATTICE_OK;
    size_t tb = 0;
    LAT_CUDA(cub::DeviceScan::InclusiveSum(nullptr, tb, in, out + 1, (int)n, st));
    return with_temp(tb, st, [&](void* tmp) -> lattice_status {
        LAT_CUDA(cub::DeviceScan::InclusiveSum(tmp, tb, in, out + 1, (int)n, st));
        return LATTICE_OK;
    });
}

}  // namespace

extern "C" {

lattice_status lattice_jsonl_open(const uint8_t* content, int64_t bytes, const char* source, lattice_jsonl** out,
                                  lattice_jsonl_info* info, lattice_stream stream) {
    using namespace lat;
    LAT_REQUIRE(out != nullptr && info != nullptr, "lattice_jsonl_open: null argument");
    LAT_REQUIRE(bytes >= 0 && (bytes == 0 || content != nullptr), "lattice_jsonl_open: bad content");
    LAT_REQUIRE(bytes < (1ll << 31), "lattice_jsonl_open: content must be < 2 GiB (split the file)");
    *out = nullptr;
    *info = lattice_jsonl_info{};
    cudaStream_t st = (cudaStream_t)stream;
    {  // keep freed pool memory for the next call (the default threshold 0 returns it to the
       // driver at every synchronisation, and re-allocating costs like cudaMalloc)
        static bool pool_set = false;
        if (!pool_set) {
            int dev = 0;
            cudaMemPool_t pool;
            if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
                uint64_t keep = 1ull << 32;
                cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
            }
            pool_set = true;
        }
    }
    lattice_jsonl* h = new lattice_jsonl();
    h->stream = st;
    h->content = content;
    h->bytes = bytes;
    auto fail = [&](lattice_status s) {
        lattice_jsonl_close(h);
        return s;
    };
#define JL_TRY(x)                              \
    do {                                       \
        lattice_status _s = (x);               \
        if (_s != LATTICE_OK) return fail(_s); \
    } while (0)
    // newline positions -> lines
    int64_t *nl = nullptr, *n_nl_d = nullptr;
    JL_TRY(jl_alloc(h, &nl, bytes + 1));
    JL_TRY(jl_alloc(h, &n_nl_d, 1));
    int64_t n_nl = 0;
    uint8_t last = '\n';
    if (bytes > 0) {
        size_t tb = 0;
        thrust::counting_iterator<int64_t> it(0);
        if (cudaSuccess != cub::DeviceSelect::If(nullptr, tb, it, nl, n_nl_d, (int)bytes, IsNewline{content}, st))
            return fail(check_cuda(cudaGetLastError(), "jsonl select"));
        JL_TRY(with_temp(tb, st, [&](void* tmp) -> lattice_status {
            LAT_CUDA(cub::DeviceSelect::If(tmp, tb, it, nl, n_nl_d, (int)bytes, IsNewline{content}, st));
            return LATTICE_OK;
        }));
        if (cudaMemcpyAsync(&n_nl, n_nl_d, sizeof(int64_t), cudaMemcpyDeviceToHost, st) != cudaSuccess ||
            cudaMemcpyAsync(&last, content + bytes - 1, 1, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
            cudaStreamSynchronize(st) != cudaSuccess)
            return fail(check_cuda(cudaGetLastError(), "jsonl line count"));
    }
    const int64_t L = n_nl + (bytes > 0 && last != '\n' ? 1 : 0);
    h->lines = L;
    info->lines = L;
    if (L == 0) {
        *out = h;
        return LATTICE_OK;
    }
    JL_TRY(jl_alloc(h, &h->start, L));
    JL_TRY(jl_alloc(h, &h->end, L));
    const unsigned gl = (unsigned)((L + 127) / 128);
    lines_kernel<<<gl, 128, 0, st>>>(nl, n_nl, bytes, L, h->start, h->end);
    // pass 1
    int32_t *code = nullptr, *col = nullptr, *arg = nullptr;
    unsigned long long* first = nullptr;
    JL_TRY(jl_alloc(h, &h->loc_off, L * NFIELD));
    JL_TRY(jl_alloc(h, &h->loc_type, L * NFIELD));
    JL_TRY(jl_alloc(h, &h->top_type, L));
    JL_TRY(jl_alloc(h, &h->is_rec, L));
    JL_TRY(jl_alloc(h, &h->rec_of_line, L));
    JL_TRY(jl_alloc(h, &code, L));
    JL_TRY(jl_alloc(h, &col, L));
    JL_TRY(jl_alloc(h, &arg, L));
    JL_TRY(jl_alloc(h, &first, 1));
    if (cudaMemsetAsync(first, 0xff, sizeof(*first), st) != cudaSuccess) return fail(check_cuda(cudaGetLastError(), "memset"));
    Lines lines{content, h->start, h->end};
    pass1_kernel<<<gl, 128, 0, st>>>(lines, L, h->loc_off, h->loc_type, h->top_type, h->is_rec, code, col, arg, first);
    if (cudaGetLastError() != cudaSuccess) return fail(check_cuda(cudaGetLastError(), "jsonl pass1"));
    // record numbering
    {
        size_t tb = 0;
        if (cudaSuccess != cub::DeviceScan::ExclusiveSum(nullptr, tb, h->is_rec, h->rec_of_line, (int)L, st))
            return fail(check_cuda(cudaGetLastError(), "jsonl scan"));
        JL_TRY(with_temp(tb, st, [&](void* tmp) -> lattice_status {
            LAT_CUDA(cub::DeviceScan::ExclusiveSum(tmp, tb, h->is_rec, h->rec_of_line, (int)L, st));
            return LATTICE_OK;
        }));
        int32_t a = 0, b = 0;
        if (cudaMemcpyAsync(&a, h->rec_of_line + L - 1, 4, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
            cudaMemcpyAsync(&b, h->is_rec + L - 1, 4, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
            cudaStreamSynchronize(st) != cudaSuccess)
            return fail(check_cuda(cudaGetLastError(), "jsonl record count"));
        h->records = (int64_t)a + b;
    }
    const int64_t N = h->records;
    info->records = N;
    // pass 2
    int64_t* sizes[7];
    for (int k = 0; k < 7; ++k) {
        JL_TRY(jl_alloc(h, &sizes[k], N));
        JL_TRY(jl_alloc(h, &h->off[k], N + 1));
    }
    JL_TRY(jl_alloc(h, &h->ts, N));
    JL_TRY(jl_alloc(h, &h->rec_line, N));
    RecSizes sz{{sizes[0], sizes[1], sizes[2]}, sizes[3], sizes[4], sizes[5], sizes[6]};
    pass2_kernel<<<gl, 128, 0, st>>>(lines, L, h->is_rec, h->rec_of_line, h->loc_off, h->loc_type, h->top_type, sz,
                                     h->ts, h->rec_line, code, col, arg, first);
    if (cudaGetLastError() != cudaSuccess) return fail(check_cuda(cudaGetLastError(), "jsonl pass2"));
    unsigned long long bad = ~0ull;
    if (cudaMemcpyAsync(&bad, first, sizeof(bad), cudaMemcpyDeviceToHost, st) != cudaSuccess ||
        cudaStreamSynchronize(st) != cudaSuccess)
        return fail(check_cuda(cudaGetLastError(), "jsonl pass2"));
    if (bad != ~0ull) {
        int32_t c = 0, cl = 0, ar = 0;
        cudaMemcpy(&c, code + bad, 4, cudaMemcpyDeviceToHost);
        cudaMemcpy(&cl, col + bad, 4, cudaMemcpyDeviceToHost);
        cudaMemcpy(&ar, arg + bad, 4, cudaMemcpyDeviceToHost);
        info->error_line = (int64_t)bad + 1;
        info->error_kind = 1;
        std::string msg;
        if (c == E_OVERFLOW) {  // escapes parse_json's parse_error catch: no "<source>:<line>" context
            int64_t ls = 0;
            std::string tok((size_t)ar, '\0');
            cudaMemcpy(&ls, h->start + bad, sizeof(ls), cudaMemcpyDeviceToHost);
            cudaMemcpy(&tok[0], content + ls + cl, (size_t)ar, cudaMemcpyDeviceToHost);
            msg = "[json.exception.out_of_range.406] number overflow parsing '" + tok + "'";
            info->error_kind = 2;
        } else {
            msg = std::string(source ? source : "records") + ":" + std::to_string(bad + 1) + ": " +
                  error_text(c, cl, ar);
        }
        return fail(set_error(LATTICE_DATA, msg, (int64_t)bad + 1));
    }
    for (int k = 0; k < 7; ++k) JL_TRY(exclusive_offsets(sizes[k], h->off[k], N, st));
    int64_t tot[7] = {};
    for (int k = 0; k < 7; ++k)
        if (cudaMemcpyAsync(&tot[k], h->off[k] + N, sizeof(int64_t), cudaMemcpyDeviceToHost, st) != cudaSuccess)
            return fail(check_cuda(cudaGetLastError(), "jsonl sizes"));
    if (cudaStreamSynchronize(st) != cudaSuccess) return fail(check_cuda(cudaGetLastError(), "jsonl sizes"));
    info->domain_bytes = tot[0];
    info->user_bytes = tot[1];
    info->ad_bytes = tot[2];
    info->feature_entries = tot[3];
    info->feature_key_bytes = tot[4];
    info->conversion_entries = tot[5];
    info->conversion_key_bytes = tot[6];
#undef JL_TRY
    *out = h;
    return LATTICE_OK;
}

lattice_status lattice_jsonl_extract(lattice_jsonl* h, const lattice_jsonl_columns* c, lattice_stream stream) {
    using namespace lat;
    LAT_REQUIRE(h != nullptr && c != nullptr, "lattice_jsonl_extract: null argument");
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t N = h->records;
    if (N == 0) {
        int64_t* zs[] = {c->domain_off, c->user_off, c->ad_off, c->feature_off, c->conversion_off,
                         c->feature_key_off, c->conversion_key_off};
        for (int64_t* z : zs)
            if (z) LAT_CUDA(cudaMemsetAsync(z, 0, sizeof(int64_t), st));
        return LATTICE_OK;
    }
    const size_t on = sizeof(int64_t) * (N + 1);
    auto cp = [&](void* dst, const void* src, size_t b) -> lattice_status {
        if (dst) LAT_CUDA(cudaMemcpyAsync(dst, src, b, cudaMemcpyDeviceToDevice, st));
        return LATTICE_OK;
    };
    lattice_status s;
    if ((s = cp(c->domain_off, h->off[0], on)) || (s = cp(c->user_off, h->off[1], on)) ||
        (s = cp(c->ad_off, h->off[2], on)) || (s = cp(c->feature_off, h->off[3], on)) ||
        (s = cp(c->conversion_off, h->off[5], on)) || (s = cp(c->ts, h->ts, sizeof(int64_t) * N)) ||
        (s = cp(c->line, h->rec_line, sizeof(int64_t) * N)))
        return s;
    LAT_REQUIRE(!c->feature_key == !c->feature_key_off && !c->feature_key == !c->feature_val,
                "lattice_jsonl_extract: feature_key, feature_key_off and feature_val go together");
    LAT_REQUIRE(!c->conversion_key == !c->conversion_key_off && !c->conversion_key == !c->conversion_val,
                "lattice_jsonl_extract: conversion_key, conversion_key_off and conversion_val go together");
    RecOut o{};
    o.str[0] = c->domain;
    o.str[1] = c->user;
    o.str[2] = c->ad;
    for (int k = 0; k < 3; ++k) o.str_off[k] = h->off[k];
    o.f_off = h->off[3];
    o.fk_off = h->off[4];
    o.f_key = c->feature_key;
    o.f_key_off = c->feature_key_off;
    o.f_val = c->feature_val;
    o.c_off = h->off[5];
    o.ck_off = h->off[6];
    o.c_key = c->conversion_key;
    o.c_key_off = c->conversion_key_off;
    o.c_val = c->conversion_val;
    Lines lines{h->content, h->start, h->end};
    pass3_kernel<<<(unsigned)((h->lines + 127) / 128), 128, 0, st>>>(lines, h->lines, h->is_rec, h->rec_of_line,
                                                                      h->loc_off, h->loc_type, o);
    LAT_CUDA(cudaGetLastError());
    // entry key offsets end with the total key bytes
    if (c->feature_key_off) {
        int64_t E = 0;
        LAT_CUDA(cudaMemcpyAsync(&E, h->off[3] + N, sizeof(E), cudaMemcpyDeviceToHost, st));
        LAT_CUDA(cudaStreamSynchronize(st));
        tail_kernel<<<1, 1, 0, st>>>(c->feature_key_off, E, h->off[4] + N);
    }
    if (c->conversion_key_off) {
        int64_t E = 0;
        LAT_CUDA(cudaMemcpyAsync(&E, h->off[5] + N, sizeof(E), cudaMemcpyDeviceToHost, st));
        LAT_CUDA(cudaStreamSynchronize(st));
        tail_kernel<<<1, 1, 0, st>>>(c->conversion_key_off, E, h->off[6] + N);
    }
    LAT_CUDA(cudaGetLastError());
    return LATTICE_OK;
}

lattice_status lattice_jsonl_task_columns(int64_t records, const int64_t* conversion_off,
                                          const uint8_t* conversion_key, const int64_t* conversion_key_off,
                                          const int64_t* conversion_val, int32_t tasks, const uint8_t* task_bytes,
                                          const int64_t* task_off, int64_t* conv, uint8_t* present,
                                          lattice_stream stream) {
    LAT_REQUIRE(records >= 0 && tasks >= 0, "lattice_jsonl_task_columns: bad sizes");
    if (records == 0 || tasks == 0) return LATTICE_OK;
    LAT_REQUIRE(conversion_off && conversion_key_off && conversion_val && task_off && conv && present,
                "lattice_jsonl_task_columns: null pointer");
    lat::task_kernel<<<(unsigned)((records + 127) / 128), 128, 0, (cudaStream_t)stream>>>(
        records, conversion_off, conversion_key, conversion_key_off, conversion_val, tasks, task_bytes, task_off, conv,
        present);
    LAT_CUDA(cudaGetLastError());
    return LATTICE_OK;
}

void lattice_jsonl_close(lattice_jsonl* h) {
    if (!h) return;
    for (void* p : h->allocs) cudaFreeAsync(p, h->stream);
    delete h;
}

}  // extern "C"
