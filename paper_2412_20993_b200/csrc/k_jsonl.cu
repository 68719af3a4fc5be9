// k_jsonl.cu — probe-trace JSON-lines ingestion on the device:
// probe::read_trace_jsonl (probe.cpp:126-165) for a whole trace file resident in HBM.
//
//   1. line split: newline positions by a chunked count / one-CTA scan / scatter (std::getline
//      semantics: a trailing newline adds no empty line, a trailing partial line counts);
//   2. one thread per line validates the line as RFC 8259 JSON (explicit container stack)
//      with the rules of the host reader (facade_jsonl.cpp, pinned to the reference by the
//      drop-in test): UTF-8 validated, raw control bytes rejected, \u escapes with surrogate
//      pairs, no leading zeros, trailing bytes rejected, the LAST duplicate of a key wins;
//      lines whose trim() is empty are skipped;
//   3. the five fields are read in the reference's order (program_id, step_index,
//      token_offset, answer, optional hesitant) with nlohmann's get<>() conversions (int
//      accepts numbers and booleans, long only numbers; floats truncate);
//   4. records are compacted in line order, program ids interned exactly (K1 on the
//      sentinel-wrapped bytes, so trimming cannot merge ids) and every record is checked
//      against the previous record of its program (stable radix sort by program): token
//      offsets, then step indices, must strictly increase (probe.cpp:148-155);
//   5. the first failing line (parse, field or order) wins, as the sequential reference
//      stops there: "trace line <n>: invalid JSON" / "missing or mistyped field" /
//      "token_offset does not increase" / "step_index does not increase".
// Decimal fractions/exponents in the two integer fields are converted exactly on the
// Clinger fast path (<= 19 significant digits with value < 2^53, |exp10| <= 22), which is
// the correctly rounded double the reference's strtod yields; a number outside that range
// in those fields is rejected ("unsupported number"), a documented restriction.

#include <algorithm>
#include <cstring>
#include <climits>
#include <string>
#include <vector>

#include "cdx_internal.cuh"
#include "k_scan.cuh"

extern "C" int cdx_canon_intern(cdx_ctx* ctx, const char* bytes, const uint64_t* offsets, uint64_t n,
                                const char* const* markers, uint32_t n_markers, uint32_t* ids, uint8_t* hes,
                                uint64_t* first_index, uint64_t* n_unique);

namespace cdx {
namespace {
using scan::LoadU32;
using scan::SL_TILE;
using scan::scan_excl;

constexpr uint32_t JL_CHUNK = 16384;  // bytes per CTA in the line split
constexpr int JL_DEPTH = 64;          // nesting depth of the line validator

enum LineState : uint8_t { L_RECORD = 0, L_BLANK = 1, L_BADJSON = 2, L_FIELD = 3, L_UNSUPPORTED = 4 };

// ---- 1. line split ----------------------------------------------------------------------
// Thread t of a CTA owns the contiguous 64 bytes [chunk + 64t, +64) (256 x 64 = JL_CHUNK),
// read as four 16-byte loads when the text is 16-byte aligned.
constexpr uint32_t JL_PER_THREAD = 64;

__device__ __forceinline__ uint64_t nl_mask64(const char* __restrict__ t, uint64_t b, uint64_t n) {
    uint64_t m = 0;
    if (b + JL_PER_THREAD <= n && (reinterpret_cast<uintptr_t>(t + b) & 15u) == 0) {
#pragma unroll
        for (int v = 0; v < 4; ++v) {
            const uint4 x = __ldg(reinterpret_cast<const uint4*>(t + b) + v);
            const uint32_t w[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                // bytes equal to '\n' (0x0a): zero-byte test on w ^ 0x0a0a0a0a, per byte exact
                const uint32_t y = w[k] ^ 0x0a0a0a0au;
                uint32_t z = ((y & 0x7f7f7f7fu) + 0x7f7f7f7fu) | y;
                z = ~(z | 0x7f7f7f7fu);  // bit 7 of each byte set iff that byte is '\n'
                const uint32_t bits = ((z >> 7) & 1u) | ((z >> 14) & 2u) | ((z >> 21) & 4u) | ((z >> 28) & 8u);
                m |= static_cast<uint64_t>(bits) << (v * 16 + k * 4);
            }
        }
    } else {
        for (uint32_t i = 0; i < JL_PER_THREAD && b + i < n; ++i)
            if (t[b + i] == '\n') m |= 1ull << i;
    }
    return m;
}

// counts per chunk; each thread's 64-bit newline mask is kept (n/8 bytes) so the scatter
// pass reads the masks instead of the text a second time
__global__ void nl_count(const char* __restrict__ t, uint64_t n, uint32_t* __restrict__ cnt,
                         uint64_t* __restrict__ masks) {
    const uint64_t b = static_cast<uint64_t>(blockIdx.x) * JL_CHUNK + threadIdx.x * JL_PER_THREAD;
    const uint64_t m = b < n ? nl_mask64(t, b, n) : 0ull;
    masks[static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x] = m;
    uint32_t c = __popcll(m);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    __shared__ uint32_t s[32];
    if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = c;
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t tot = 0;
        for (uint32_t w = 0; w < blockDim.x / 32; ++w) tot += s[w];
        cnt[blockIdx.x] = tot;
    }
}


// newline positions in order: each thread's 64-byte mask, a block scan of the counts
__global__ void nl_scatter(const uint64_t* __restrict__ masks, uint64_t n, const uint32_t* __restrict__ base,
                           uint64_t* __restrict__ pos) {
    __shared__ uint32_t s_w[32];
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint64_t b = static_cast<uint64_t>(blockIdx.x) * JL_CHUNK + threadIdx.x * JL_PER_THREAD;
    uint64_t m = b < n ? masks[static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x] : 0ull;
    const uint32_t c = __popcll(m);
    uint32_t inc = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= static_cast<uint32_t>(o)) inc += y;
    }
    if (lane == 31) s_w[warp] = inc;
    __syncthreads();
    uint32_t before = base[blockIdx.x] + inc - c;
    for (uint32_t w = 0; w < warp; ++w) before += s_w[w];
    while (m) {
        pos[before++] = b + static_cast<uint64_t>(__ffsll(static_cast<long long>(m)) - 1);
        m &= m - 1;
    }
}

// ---- 2./3. per-line parse -----------------------------------------------------------------
struct Span {
    uint64_t b = 0, e = 0;  // value token [b, e) (strings: inside the quotes)
    uint8_t kind = 0;       // 0 absent, 1 string, 2 number, 3 true, 4 false, 5 null, 6 array, 7 object
};

__device__ __forceinline__ bool jws(char c) {  // ' ' \t \n \r as one mask test
    const uint32_t u = static_cast<unsigned char>(c);
    return u <= 32u && ((0x100002600ull >> u) & 1ull);
}
__device__ __forceinline__ bool trim_ws(char c) {
    return c == ' ' || c == '\t' || c == '\n' || c == '\r' || c == '\f' || c == '\v';
}
__device__ __forceinline__ int hexv(char c) {
    if (c >= '0' && c <= '9') return c - '0';
    if (c >= 'a' && c <= 'f') return c - 'a' + 10;
    if (c >= 'A' && c <= 'F') return c - 'A' + 10;
    return -1;
}

// Validate (and optionally decode) the string whose opening quote is at t[p]; returns the
// index after the closing quote, or 0 on error.  len: decoded length; esc: a backslash
// escape occurred.  MODE 0 validates only, 1 also packs the first 16 decoded bytes into
// k0/k1 (member keys), 2 also writes the decoded bytes to out[0, out_cap).
// Runs of plain bytes (0x20..0x7F except '"' and '\') are taken 8 at a time: one aligned
// 16-byte window per step (inside the text: nt is its length), the classes found with SWAR
// byte tests whose lowest flagged byte is exact (borrows only travel upward).
template <int MODE>
__device__ __forceinline__ uint64_t scan_str(const char* __restrict__ t, uint64_t p, uint64_t e, uint64_t nt,
                                             uint32_t& len, bool& esc, uint64_t& k0, uint64_t& k1,
                                             char* __restrict__ out, uint32_t out_cap) {
    ++p;
    uint32_t o = 0;
    auto put = [&](uint32_t c) {
        if (MODE == 1) {
            if (o < 8) k0 |= static_cast<uint64_t>(c) << (8 * o);
            else if (o < 16) k1 |= static_cast<uint64_t>(c) << (8 * (o - 8));
        }
        if (MODE == 2 && o < out_cap) out[o] = static_cast<char>(c);
        ++o;
    };
    constexpr uint64_t ONES = 0x0101010101010101ull, HI = 0x8080808080808080ull;
    while (p < e) {
        if (p + 8 <= e && (p & ~7ull) + 16 <= nt) {
            const uint64_t al = p & ~7ull;
            const uint32_t sh = static_cast<uint32_t>(p & 7) * 8;
            const uint64_t w0 = *reinterpret_cast<const uint64_t*>(t + al);
            const uint64_t w1 = *reinterpret_cast<const uint64_t*>(t + al + 8);
            const uint64_t x = sh ? (w0 >> sh) | (w1 << (64 - sh)) : w0;
            const uint64_t q = x ^ (ONES * '"'), b = x ^ (ONES * '\\');
            const uint64_t m = ((x - ONES * 0x20) & ~x) | ((q - ONES) & ~q) | ((b - ONES) & ~b) | x;
            const uint64_t f = m & HI;
            const uint32_t j = f ? static_cast<uint32_t>(__ffsll(static_cast<long long>(f)) - 1) >> 3 : 8u;
            if (MODE == 1) {  // the j plain bytes enter the packed key at byte offset o
                const uint64_t c = j == 8 ? x : x & ((1ull << (8 * j)) - 1ull);
                if (o < 8) {
                    k0 |= c << (8 * o);
                    if (o) k1 |= c >> (64 - 8 * o);
                } else if (o < 16) {
                    k1 |= c << (8 * (o - 8));
                }
                o += j;
            } else if (MODE == 2) {
                for (uint32_t k = 0; k < j; ++k) put(static_cast<uint32_t>(x >> (8 * k)) & 0xffu);
            } else {
                o += j;
            }
            p += j;
            if (j == 8) continue;
        }
        const unsigned char c = static_cast<unsigned char>(t[p]);
        if (c == '"') {
            len = o;
            return p + 1;
        }
        if (c < 0x20) return 0;
        if (c == '\\') {
            esc = true;
            if (p + 1 >= e) return 0;
            const char x = t[p + 1];
            p += 2;
            uint32_t cp;
            switch (x) {
                case '"': put('"'); continue;
                case '\\': put('\\'); continue;
                case '/': put('/'); continue;
                case 'b': put('\b'); continue;
                case 'f': put('\f'); continue;
                case 'n': put('\n'); continue;
                case 'r': put('\r'); continue;
                case 't': put('\t'); continue;
                case 'u': {
                    if (p + 4 > e) return 0;
                    cp = 0;
                    for (int k = 0; k < 4; ++k) {
                        const int h = hexv(t[p + k]);
                        if (h < 0) return 0;
                        cp = (cp << 4) | static_cast<uint32_t>(h);
                    }
                    p += 4;
                    if (cp >= 0xD800 && cp <= 0xDBFF) {
                        if (p + 6 > e || t[p] != '\\' || t[p + 1] != 'u') return 0;
                        uint32_t lo = 0;
                        for (int k = 0; k < 4; ++k) {
                            const int h = hexv(t[p + 2 + k]);
                            if (h < 0) return 0;
                            lo = (lo << 4) | static_cast<uint32_t>(h);
                        }
                        if (lo < 0xDC00 || lo > 0xDFFF) return 0;
                        p += 6;
                        cp = 0x10000 + ((cp - 0xD800) << 10) + (lo - 0xDC00);
                    } else if (cp >= 0xDC00 && cp <= 0xDFFF) {
                        return 0;
                    }
                    if (cp < 0x80) {
                        put(cp);
                    } else if (cp < 0x800) {
                        put(0xC0 | (cp >> 6));
                        put(0x80 | (cp & 0x3F));
                    } else if (cp < 0x10000) {
                        put(0xE0 | (cp >> 12));
                        put(0x80 | ((cp >> 6) & 0x3F));
                        put(0x80 | (cp & 0x3F));
                    } else {
                        put(0xF0 | (cp >> 18));
                        put(0x80 | ((cp >> 12) & 0x3F));
                        put(0x80 | ((cp >> 6) & 0x3F));
                        put(0x80 | (cp & 0x3F));
                    }
                    continue;
                }
                default: return 0;
            }
        }
        int n;
        uint32_t cp;
        if (c < 0x80) n = 1, cp = c;
        else if (c >= 0xC2 && c <= 0xDF) n = 2, cp = c & 0x1F;
        else if (c >= 0xE0 && c <= 0xEF) n = 3, cp = c & 0x0F;
        else if (c >= 0xF0 && c <= 0xF4) n = 4, cp = c & 0x07;
        else return 0;
        if (p + n > e) return 0;
        for (int k = 1; k < n; ++k) {
            const unsigned char cc = static_cast<unsigned char>(t[p + k]);
            if ((cc & 0xC0) != 0x80) return 0;
            cp = (cp << 6) | (cc & 0x3F);
        }
        if ((n == 3 && (cp < 0x800 || (cp >= 0xD800 && cp <= 0xDFFF))) || (n == 4 && (cp < 0x10000 || cp > 0x10FFFF)))
            return 0;
        for (int k = 0; k < n; ++k) put(static_cast<unsigned char>(t[p + k]));
        p += n;
    }
    return 0;
}

// number token at t[p]: returns the end index or 0; big: it has an exponent or is long
// enough (> 300 bytes) that it could overflow a double
__device__ uint64_t scan_number(const char* t, uint64_t p, uint64_t e, bool& big) {
    const uint64_t p0 = p;
    big = false;
    if (p < e && t[p] == '-') ++p;
    if (p >= e || t[p] < '0' || t[p] > '9') return 0;
    if (t[p] == '0') {
        ++p;
        if (p < e && t[p] >= '0' && t[p] <= '9') return 0;
    } else {
        while (p < e && t[p] >= '0' && t[p] <= '9') ++p;
    }
    if (p < e && t[p] == '.') {
        ++p;
        if (p >= e || t[p] < '0' || t[p] > '9') return 0;
        while (p < e && t[p] >= '0' && t[p] <= '9') ++p;
    }
    if (p < e && (t[p] == 'e' || t[p] == 'E')) {
        big = true;
        ++p;
        if (p < e && (t[p] == '+' || t[p] == '-')) ++p;
        if (p >= e || t[p] < '0' || t[p] > '9') return 0;
        while (p < e && t[p] >= '0' && t[p] <= '9') ++p;
    }
    big = big || p - p0 > 300;
    return p;
}

// strtod overflow (nlohmann: out_of_range.406 "number overflow", a parse error of the whole
// line, for a number at any depth): a decimal rounds to infinity iff its value is at least
// 2^1024 - 2^970 (the midpoint above DBL_MAX; ties go to the even, infinite, side).  With
// E10 the decimal exponent of the leading significant digit, E10 > 308 always overflows,
// E10 < 308 never does, and E10 == 308 compares the digit string with the boundary's 309.
__constant__ char kOvfDigits[310] =
    "179769313486231580793728971405303415079934132710037826936173778980444968292764750946649017977587207096330286416692887910946555547851940402630657488671505820681908902000708383676273854845817711531764475730270069855571366959622842914819860834936475292719074168444365510704342711559699508093042880177904174497792";

// number token [b, e) (grammar already validated); exponents saturate far beyond +-308
__device__ bool num_overflows(const char* t, uint64_t b, uint64_t e) {
    uint64_t p = b;
    if (t[p] == '-') ++p;
    long long e10;
    uint64_t first;  // index of the first significant digit
    uint64_t q = p;
    while (q < e && t[q] >= '0' && t[q] <= '9') ++q;
    const uint64_t int_end = q;
    if (!(int_end - p == 1 && t[p] == '0')) {
        first = p;
        e10 = static_cast<long long>(int_end - p) - 1;
    } else {  // 0.000ddd: the first nonzero fraction digit
        if (q >= e || t[q] != '.') return false;  // plain 0 (with or without exponent)
        ++q;
        const uint64_t fb = q;
        while (q < e && t[q] == '0') ++q;
        if (q >= e || t[q] < '1' || t[q] > '9') return false;  // the value is zero
        first = q;
        e10 = -static_cast<long long>(q - fb) - 1;
    }
    uint64_t x = first;
    while (x < e && t[x] != 'e' && t[x] != 'E') ++x;
    if (x < e) {  // exponent, saturated
        ++x;
        bool en = false;
        if (t[x] == '+' || t[x] == '-') {
            en = t[x] == '-';
            ++x;
        }
        long long v = 0;
        for (; x < e; ++x) v = v < 100000000 ? v * 10 + (t[x] - '0') : v;
        e10 += en ? -v : v;
    }
    if (e10 != 308) return e10 > 308;
    int k = 0;  // digits compared so far
    for (uint64_t y = first; y < e && t[y] != 'e' && t[y] != 'E'; ++y) {
        if (t[y] == '.') continue;
        if (k == 309) return true;  // equal on all 309 digits, more follow: >= the boundary
        const char c = t[y], d = kOvfDigits[k++];
        if (c != d) return c > d;
    }
    return k == 309;  // a shorter equal prefix is below the boundary (its tail is nonzero)
}

// nlohmann number -> (int64 | uint64 | double); returns 0 int64, 1 uint64, 2 double, -1 unsupported
__device__ int number_value(const char* t, uint64_t b, uint64_t e, long long* iv, unsigned long long* uv,
                            double* dv) {
    bool neg = false, is_float = false;
    uint64_t p = b;
    if (t[p] == '-') {
        neg = true;
        ++p;
    }
    for (uint64_t q = p; q < e; ++q)
        if (t[q] == '.' || t[q] == 'e' || t[q] == 'E') is_float = true;
    if (!is_float) {
        unsigned long long v = 0;
        bool ovf = false;
        for (uint64_t q = p; q < e; ++q) {
            const unsigned d = static_cast<unsigned>(t[q] - '0');
            if (v > (ULLONG_MAX - d) / 10ull) ovf = true;
            v = v * 10ull + d;
        }
        if (!ovf) {
            if (!neg) {
                *uv = v;
                return 1;
            }
            if (v <= 0x8000000000000000ull) {  // strtoll range
                *iv = v == 0x8000000000000000ull ? LLONG_MIN : -static_cast<long long>(v);
                return 0;
            }
        }
    }
    // decimal -> double on the Clinger fast path (one correctly rounded IEEE op)
    unsigned long long m = 0;
    int digits = 0, exp10 = 0;
    bool frac = false;
    uint64_t q = p;
    for (; q < e && t[q] != 'e' && t[q] != 'E'; ++q) {
        if (t[q] == '.') {
            frac = true;
            continue;
        }
        const unsigned d = static_cast<unsigned>(t[q] - '0');
        if (m == 0 && d == 0) {
            if (frac) --exp10;
            continue;
        }
        if (digits == 19) {  // more digits than the fast path can hold exactly
            if (d != 0) return -1;
            if (!frac) ++exp10;
            continue;
        }
        m = m * 10ull + d;
        ++digits;
        if (frac) --exp10;
    }
    if (q < e) {  // exponent
        ++q;
        bool en = false;
        if (t[q] == '+' || t[q] == '-') {
            en = t[q] == '-';
            ++q;
        }
        int x = 0;
        for (; q < e; ++q) {
            x = x * 10 + (t[q] - '0');
            if (x > 100000) return -1;
        }
        exp10 += en ? -x : x;
    }
    if (m == 0) {
        *dv = neg ? -0.0 : 0.0;
        return 2;
    }
    if (m >= (1ull << 53) || exp10 < -22 || exp10 > 22) return -1;
    double pw = 1.0;
    for (int k = 0; k < (exp10 < 0 ? -exp10 : exp10); ++k) pw *= 10.0;  // exact for 10^k, k <= 22
    double v = exp10 < 0 ? __ddiv_rn(static_cast<double>(m), pw) : __dmul_rn(static_cast<double>(m), pw);
    *dv = neg ? -v : v;
    return 2;
}

// C++ static_cast<int|long>(double) as x86-64 performs it (out of range -> INT/LONG min)
__device__ __forceinline__ long long trunc_ll(double v) {
    if (!(v > -9223372036854775808.0 && v < 9223372036854775808.0)) return LLONG_MIN;
    return static_cast<long long>(v);
}
__device__ __forceinline__ int trunc_i(double v) {
    if (!(v > -2147483649.0 && v < 2147483648.0)) return INT_MIN;
    return static_cast<int>(v);
}

// key of interest: 0 program_id, 1 step_index, 2 token_offset, 3 answer, 4 hesitant, -1 other
// (decoded key: length n, first 16 bytes packed little-endian in k0/k1)
constexpr uint64_t pack8(const char* s, int from, int n) {
    uint64_t v = 0;
    for (int i = 0; i < 8 && from + i < n; ++i) v |= static_cast<uint64_t>(static_cast<unsigned char>(s[from + i])) << (8 * i);
    return v;
}
__device__ __forceinline__ int key_id(uint64_t k0, uint64_t k1, uint32_t n) {
    if (n == 10 && k0 == pack8("program_id", 0, 10) && k1 == pack8("program_id", 8, 10)) return 0;
    if (n == 10 && k0 == pack8("step_index", 0, 10) && k1 == pack8("step_index", 8, 10)) return 1;
    if (n == 12 && k0 == pack8("token_offset", 0, 12) && k1 == pack8("token_offset", 8, 12)) return 2;
    if (n == 6 && k0 == pack8("answer", 0, 6) && k1 == 0) return 3;
    if (n == 8 && k0 == pack8("hesitant", 0, 8) && k1 == 0) return 4;
    return -1;
}

struct LineOut {
    uint8_t* st;
    uint32_t* pid_len;  // decoded lengths of the program id and the answer
    uint32_t* ans_len;
    uint8_t* esc;       // bit 0: the program id has escapes, bit 1: the answer has
    uint64_t* pid_b;
    uint64_t* pid_e;
    uint64_t* ans_b;
    uint64_t* ans_e;
    int32_t* step;
    int64_t* tok;
    uint8_t* hes;
};

// One thread per line.  The container stack is a bitmask (bit d: the container at depth
// d is an object), the five fields of interest live in registers (written through an
// unrolled select, so no local-memory array), member keys are decoded into two registers
// and compared as packed words, and strings advance 8 plain bytes per step (scan_str).
__global__ void __launch_bounds__(128) parse_lines(const char* __restrict__ t, uint64_t n,
                                                   const uint64_t* __restrict__ nl, uint64_t n_nl, uint64_t n_lines,
                                                   LineOut o, unsigned long long* first_bad) {
    static_assert(JL_DEPTH <= 64, "one bit per nesting level");
    for (uint64_t L = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; L < n_lines;
         L += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint64_t b = L == 0 ? 0 : nl[L - 1] + 1;
        const uint64_t e = L < n_nl ? nl[L] : n;
        uint8_t st = L_RECORD;
        // trim() empty -> skipped (probe.cpp:132)
        uint64_t q = b;
        while (q < e && trim_ws(t[q])) ++q;
        if (q == e) {
            o.st[L] = L_BLANK;
            continue;
        }
        // ---- validate the document (iterative, explicit container stack)
        uint64_t fb[5], fe[5];
        uint32_t fl[5];
        uint8_t fk[5], fx[5];
#pragma unroll
        for (int k = 0; k < 5; ++k) fb[k] = fe[k] = 0, fl[k] = 0, fk[k] = 0, fx[k] = 0;
        auto set_field = [&](int key, uint64_t vb, uint64_t ve, uint8_t kind, uint32_t dl, bool dx) {
#pragma unroll
            for (int k = 0; k < 5; ++k)
                if (k == key) fb[k] = vb, fe[k] = ve, fk[k] = kind, fl[k] = dl, fx[k] = dx;
        };
        uint64_t objmask = 0;  // bit d: container at depth d is an object
        int depth = 0;
        uint64_t p = b;
        bool ok = true;
        int pending_key = -2;  // key id of the member value about to be parsed (-2: none)
        bool top_obj = false;
        // states: 0 expect value, 1 after value, 2 expect key or '}', 3 expect key
        int state = 0;
        uint64_t k0, k1;
        uint32_t slen;
        bool sesc;
        while (ok) {
            char c = 0;  // the next non-whitespace byte (0 at the line end): read once per token
            while (p < e) {
                c = t[p];
                if (!jws(c)) break;
                ++p;
            }
            if (p >= e) c = 0;
            if (state == 0) {
                if (p >= e) {
                    ok = false;
                    break;
                }
                const uint64_t vb = p;
                const bool field = depth == 1 && top_obj && pending_key >= 0;
                if (c == '{' || c == '[') {
                    if (depth == JL_DEPTH) {
                        ok = false;
                        break;
                    }
                    if (depth == 0 && c == '{') top_obj = true;
                    if (field) set_field(pending_key, vb, vb, c == '{' ? uint8_t(7) : uint8_t(6), 0, false);
                    pending_key = -2;
                    objmask = (objmask & ~(1ull << depth)) | (static_cast<uint64_t>(c == '{') << depth);
                    ++depth;
                    ++p;
                    state = c == '{' ? 2 : 0;
                    if (c == '[') {  // empty array?
                        uint64_t r = p;
                        while (r < e && jws(t[r])) ++r;
                        if (r < e && t[r] == ']') {
                            p = r + 1;
                            --depth;
                            state = 1;
                        }
                    }
                    continue;
                }
                if (c == '"') {
                    sesc = false;
                    const uint64_t r = scan_str<0>(t, p, e, n, slen, sesc, k0, k1, nullptr, 0);
                    if (!r) {
                        ok = false;
                        break;
                    }
                    if (field) set_field(pending_key, vb + 1, r - 1, 1, slen, sesc);
                    p = r;
                } else if (c == '-' || (c >= '0' && c <= '9')) {
                    bool big;
                    const uint64_t r = scan_number(t, p, e, big);
                    if (!r || (big && num_overflows(t, p, r))) {
                        ok = false;
                        break;
                    }
                    if (field) set_field(pending_key, vb, r, 2, 0, false);
                    p = r;
                } else {
                    // true / false / null, compared as one packed word
                    const uint32_t ln = c == 'f' ? 5 : 4;
                    const uint64_t want = c == 't' ? 0x65757274ull : (c == 'f' ? 0x65736c6166ull : 0x6c6c756eull);
                    if ((c != 't' && c != 'f' && c != 'n') || p + ln > e) {
                        ok = false;
                        break;
                    }
                    uint64_t got = 0;
                    for (uint32_t k = 0; k < ln; ++k) got |= static_cast<uint64_t>(static_cast<unsigned char>(t[p + k])) << (8 * k);
                    if (got != want) {
                        ok = false;
                        break;
                    }
                    if (field) set_field(pending_key, vb, p + ln, c == 't' ? 3 : (c == 'f' ? 4 : 5), 0, false);
                    p += ln;
                }
                pending_key = -2;
                state = 1;
                if (depth == 0) break;  // the top-level value was a scalar
                continue;
            }
            const bool in_obj = depth > 0 && ((objmask >> (depth - 1)) & 1ull);
            if (state == 1) {  // after a value inside a container
                if (depth == 0) break;
                if (p >= e) {
                    ok = false;
                    break;
                }
                if (c == ',') {
                    ++p;
                    state = in_obj ? 3 : 0;
                } else if ((c == '}' && in_obj) || (c == ']' && !in_obj)) {
                    ++p;
                    --depth;
                    state = 1;
                    if (depth == 0) break;
                } else {
                    ok = false;
                }
                continue;
            }
            // state 2 / 3: a member key
            if (p >= e) {
                ok = false;
                break;
            }
            if (state == 2 && c == '}') {
                ++p;
                --depth;
                state = 1;
                if (depth == 0) break;
                continue;
            }
            if (c != '"') {
                ok = false;
                break;
            }
            k0 = k1 = 0;
            const uint64_t r = scan_str<1>(t, p, e, n, slen, sesc, k0, k1, nullptr, 0);
            if (!r) {
                ok = false;
                break;
            }
            pending_key = (depth == 1 && top_obj) ? key_id(k0, k1, slen) : -1;
            p = r;
            while (p < e && jws(t[p])) ++p;
            if (p >= e || t[p] != ':') {
                ok = false;
                break;
            }
            ++p;
            state = 0;
        }
        if (ok) {  // trailing bytes
            while (p < e && jws(t[p])) ++p;
            ok = p == e;
        }
        if (!ok) {
            st = L_BADJSON;
        } else if (!top_obj) {
            st = L_FIELD;  // at() on a non-object
        } else {
            // ---- fields in the reference's order (probe.cpp:140-145)
            if (fk[0] != 1) st = L_FIELD;
            long long iv = 0;
            unsigned long long uv = 0;
            double dv = 0;
            if (st == L_RECORD) {  // step_index: get<int>() (numbers and booleans)
                if (fk[1] == 3 || fk[1] == 4) {
                    o.step[L] = fk[1] == 3 ? 1 : 0;
                } else if (fk[1] == 2) {
                    const int k = number_value(t, fb[1], fe[1], &iv, &uv, &dv);
                    if (k < 0) st = L_UNSUPPORTED;
                    else o.step[L] = k == 0 ? static_cast<int>(iv) : (k == 1 ? static_cast<int>(uv) : trunc_i(dv));
                } else {
                    st = L_FIELD;
                }
            }
            if (st == L_RECORD) {  // token_offset: get<long>() (numbers only)
                if (fk[2] == 2) {
                    const int k = number_value(t, fb[2], fe[2], &iv, &uv, &dv);
                    if (k < 0) st = L_UNSUPPORTED;
                    else o.tok[L] = k == 0 ? iv : (k == 1 ? static_cast<long long>(uv) : trunc_ll(dv));
                } else {
                    st = L_FIELD;
                }
            }
            if (st == L_RECORD && fk[3] != 1) st = L_FIELD;
            if (st == L_RECORD) {  // hesitant: value("hesitant", false) -> bool or absent
                if (fk[4] == 0) o.hes[L] = 0;
                else if (fk[4] == 3 || fk[4] == 4) o.hes[L] = fk[4] == 3;
                else st = L_FIELD;
            }
            o.pid_b[L] = fb[0];
            o.pid_e[L] = fe[0];
            o.ans_b[L] = fb[3];
            o.ans_e[L] = fe[3];
            o.pid_len[L] = fl[0];
            o.ans_len[L] = fl[3];
            o.esc[L] = static_cast<uint8_t>(fx[0] | (fx[3] << 1));
        }
        o.st[L] = st;
        if (st != L_RECORD) atomicMin(first_bad, static_cast<unsigned long long>(L));
    }
}

// ---- 4. compaction of records + decoded strings -------------------------------------------



// record r <- line L (st == record): fields + decoded string lengths
__global__ void gather_records(const char* __restrict__ t, const uint8_t* __restrict__ st,
                               const uint32_t* __restrict__ pos, uint64_t n_lines, LineOut o,
                               int32_t* __restrict__ r_step, int64_t* __restrict__ r_tok, uint8_t* __restrict__ r_hes,
                               uint64_t* __restrict__ r_line, uint32_t* __restrict__ pid_len,
                               uint32_t* __restrict__ ans_len) {
    for (uint64_t L = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; L < n_lines;
         L += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        if (st[L] != L_RECORD) continue;
        const uint32_t r = pos[L];
        r_step[r] = o.step[L];
        r_tok[r] = o.tok[L];
        r_hes[r] = o.hes[L];
        r_line[r] = L;
        pid_len[r] = o.pid_len[L] + 2;  // wrapped in sentinel bytes for exact interning
        ans_len[r] = o.ans_len[L];
    }
}

// Raw string bytes [b, e) -> dst, 8 source bytes per step through an aligned 16-byte window
// (two loads instead of eight byte loads; the window stays inside the text of length n).
__device__ __forceinline__ void copy_raw(const char* __restrict__ t, uint64_t n, uint64_t b, uint64_t e,
                                         char* __restrict__ dst) {
    uint64_t i = b;
    for (; i + 8 <= e && (i & ~7ull) + 16 <= n; i += 8) {
        const uint64_t al = i & ~7ull;
        const uint32_t sh = static_cast<uint32_t>(i & 7) * 8;
        const uint64_t w0 = *reinterpret_cast<const uint64_t*>(t + al);
        const uint64_t w1 = *reinterpret_cast<const uint64_t*>(t + al + 8);
        const uint64_t x = sh ? (w0 >> sh) | (w1 << (64 - sh)) : w0;
#pragma unroll
        for (int k = 0; k < 8; ++k) dst[i - b + k] = static_cast<char>(x >> (8 * k));
    }
    for (; i < e; ++i) dst[i - b] = t[i];
}

__global__ void write_strings(const char* __restrict__ t, uint64_t n, const uint8_t* __restrict__ st,
                              const uint32_t* __restrict__ pos, uint64_t n_lines, LineOut o,
                              const uint64_t* __restrict__ pid_off, char* __restrict__ pid_arena,
                              const uint64_t* __restrict__ ans_off, char* __restrict__ ans_arena) {
    for (uint64_t L = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; L < n_lines;
         L += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        if (st[L] != L_RECORD) continue;
        const uint32_t r = pos[L];
        char* pp = pid_arena + pid_off[r];
        const uint32_t cap = static_cast<uint32_t>(pid_off[r + 1] - pid_off[r]);
        pp[0] = '\x01';
        const uint8_t x = o.esc[L];
        uint32_t k = 0;
        bool dx = false;
        uint64_t d0 = 0, d1 = 0;
        if (x & 1u)
            scan_str<2>(t, o.pid_b[L] - 1, o.pid_e[L] + 1, n, k, dx, d0, d1, pp + 1, cap - 2);
        else
            copy_raw(t, n, o.pid_b[L], o.pid_e[L], pp + 1);
        pp[cap - 1] = '\x01';
        char* ap = ans_arena + ans_off[r];
        if (x & 2u)
            scan_str<2>(t, o.ans_b[L] - 1, o.ans_e[L] + 1, n, k, dx, d0, d1, ap,
                        static_cast<uint32_t>(ans_off[r + 1] - ans_off[r]));
        else
            copy_raw(t, n, o.ans_b[L], o.ans_e[L], ap);
    }
}

struct LoadRecordFlag {  // 1 for a line that is a record
    const uint8_t* st;
    __device__ uint32_t operator()(uint64_t i) const { return st[i] == L_RECORD ? 1u : 0u; }
};

// ---- 4b. order check per program (probe.cpp:148-155) ------------------------------------
__global__ void order_check(const uint32_t* __restrict__ sorted_rec, const uint64_t* __restrict__ keys,
                            uint64_t n, const int32_t* __restrict__ step, const int64_t* __restrict__ tok,
                            const uint64_t* __restrict__ line, unsigned long long* __restrict__ first_bad,
                            uint8_t* __restrict__ why) {
    for (uint64_t i = 1 + blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        if (keys[i] != keys[i - 1]) continue;  // first record of its program
        const uint32_t cur = sorted_rec[i], prev = sorted_rec[i - 1];
        uint8_t w = 0;
        if (tok[cur] <= tok[prev]) w = 1;
        else if (step[cur] <= step[prev]) w = 2;
        if (w) {
            const unsigned long long L = line[cur];
            atomicMin(first_bad, L);
            why[cur] = w;
        }
    }
}


__global__ void widen_ids(const uint32_t* __restrict__ ids, uint64_t n, uint64_t* __restrict__ k,
                          uint32_t* __restrict__ v) {
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        k[i] = ids[i];
        v[i] = static_cast<uint32_t>(i);
    }
}

// per-record program-id strings without the interning sentinels: record r's bytes start at
// pid_off[r] + 1 in the wrapped arena and at pid_off[r] - 2r unwrapped
__global__ void unwrap_pids(const uint64_t* __restrict__ pid_off, const char* __restrict__ wrapped, uint64_t n,
                            uint64_t* __restrict__ off, char* __restrict__ arena) {
    for (uint64_t r = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; r <= n;
         r += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        off[r] = pid_off[r] - 2 * r;
        if (r == n) continue;
        const uint64_t b = pid_off[r] + 1, e = pid_off[r + 1] - 1;
        for (uint64_t i = b; i < e; ++i) arena[i - 2 * r - 1] = wrapped[i];
    }
}

unsigned gridn(const cdx_ctx* ctx, uint64_t n) {
    const uint64_t want = (n + 255) / 256;
    const uint64_t cap = static_cast<uint64_t>(ctx->sm_count) * 16;
    return static_cast<unsigned>(want < 1 ? 1 : (want < cap ? want : cap));
}

template <typename T>
T* carve(uint8_t*& p, uint64_t n) {
    T* r = reinterpret_cast<T*>(p);
    p += (n * sizeof(T) + 255) / 256 * 256;
    return r;
}

}  // namespace
}  // namespace cdx

extern "C" int cdx_jsonl_parse(cdx_ctx* ctx, const char* text, uint64_t nbytes, uint64_t cap_records,
                               uint32_t* program, int32_t* step_index, int64_t* token_offset, uint8_t* hesitant,
                               uint64_t* answer_off, char* answer_arena, uint64_t* program_off,
                               char* program_arena, uint64_t* program_first, uint64_t* n_records,
                               uint64_t* n_programs) {
    using namespace cdx;
    CDX_NVTX("cdx_jsonl_parse");
    if (!ctx) return CDX_EINVAL;
    if (!n_records || !n_programs) return set_error(ctx, CDX_EINVAL, "jsonl_parse: null pointer");
    *n_records = 0;
    *n_programs = 0;
    if (nbytes == 0) return CDX_OK;
    if (!text || !program || !step_index || !token_offset || !hesitant || !answer_off || !answer_arena)
        return set_error(ctx, CDX_EINVAL, "jsonl_parse: null pointer");
    if (nbytes >= (1ull << 32)) return set_error(ctx, CDX_EINVAL, "jsonl_parse: at most 4 GiB per call");
    const uint64_t nchunks = (nbytes + JL_CHUNK - 1) / JL_CHUNK;
    // phase 1 (small scratch): newline count per chunk, then its scan
    uint8_t* s1 = static_cast<uint8_t*>(
        scratch2(ctx, 4096 + nchunks * 4 + 256 + (nchunks / SL_TILE + 2) * 8 + 256 + nchunks * 256 * 8 + 256));
    if (!s1) return set_error(ctx, CDX_ECUDA, "jsonl_parse: scratch allocation failed");
    uint8_t* p1 = s1;
    uint64_t* misc = carve<uint64_t>(p1, 16);  // [0] newlines, [1] first bad line, [2] records, [3] scan total
    uint32_t* cnt = carve<uint32_t>(p1, nchunks);
    uint64_t* crec = carve<uint64_t>(p1, nchunks / SL_TILE + 2);
    cudaMemsetAsync(misc, 0, 16 * 8, ctx->stream);
    cudaMemsetAsync(misc + 1, 0xff, 8, ctx->stream);
    uint64_t* nlm = carve<uint64_t>(p1, nchunks * 256);
    nl_count<<<static_cast<unsigned>(nchunks), 256, 0, ctx->stream>>>(text, nbytes, cnt, nlm);
    CDX_CHECK_LAUNCH(ctx, "jsonl(lines)");
    if (int st = scan_excl(ctx, LoadU32{cnt}, nchunks, cnt, false, crec, misc)) return st;  // in place
    uint64_t h_nl = 0;
    char last = 0;
    cudaMemcpyAsync(&h_nl, misc, 8, cudaMemcpyDeviceToHost, ctx->stream);
    cudaMemcpyAsync(&last, text + nbytes - 1, 1, cudaMemcpyDeviceToHost, ctx->stream);
    cudaError_t e = cudaStreamSynchronize(ctx->stream);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "jsonl_parse");
    const uint64_t n_lines = h_nl + (last == '\n' ? 0 : 1);  // std::getline semantics
    // phase 2 (dedicated buffer sized from the line count): every later array is bounded by
    // n_lines records and nbytes of text
    const uint64_t nl1 = n_lines + 1;
    const size_t bulk = 256 * 40 + nl1 * (8 + 1 + 8 * 4 + 4 + 8 + 1 + 4 + 4 + 4 + 1) + (nl1 / 1024 + 2) * 4 +
                        nl1 * (8 + 4 + 4 + 8 + 1 + 8 + 8 + 4 + 4) + (3 * nbytes / 2 + 2 * nl1 + 64) +
                        radix_scratch_words(nl1) * 4;
    if (ctx->jl_bytes < bulk) {
        cudaStreamSynchronize(ctx->stream);
        if (ctx->jl_buf) cudaFree(ctx->jl_buf);
        ctx->jl_buf = nullptr;
        ctx->jl_bytes = 0;
        if (cudaMalloc(&ctx->jl_buf, bulk) != cudaSuccess) return set_error(ctx, CDX_ECUDA, "jsonl_parse: allocation");
        ctx->jl_bytes = bulk;
    }
    uint8_t* s = static_cast<uint8_t*>(ctx->jl_buf);
    uint8_t* p = s;
    const size_t bytes = bulk;
    uint64_t* nl = carve<uint64_t>(p, h_nl + 1);
    nl_scatter<<<static_cast<unsigned>(nchunks), 256, 0, ctx->stream>>>(nlm, nbytes, cnt, nl);
    CDX_CHECK_LAUNCH(ctx, "jsonl(line ends)");
    LineOut o;
    o.st = carve<uint8_t>(p, n_lines);
    o.pid_b = carve<uint64_t>(p, n_lines);
    o.pid_e = carve<uint64_t>(p, n_lines);
    o.ans_b = carve<uint64_t>(p, n_lines);
    o.ans_e = carve<uint64_t>(p, n_lines);
    o.step = carve<int32_t>(p, n_lines);
    o.tok = carve<int64_t>(p, n_lines);
    o.hes = carve<uint8_t>(p, n_lines);
    o.pid_len = carve<uint32_t>(p, n_lines);
    o.ans_len = carve<uint32_t>(p, n_lines);
    o.esc = carve<uint8_t>(p, n_lines);
    uint32_t* pos = carve<uint32_t>(p, n_lines);
    uint64_t* srec = carve<uint64_t>(p, (n_lines + SL_TILE - 1) / SL_TILE + 2);  // scan tile records + ticket
    parse_lines<<<gridn(ctx, n_lines), 128, 0, ctx->stream>>>(text, nbytes, nl, h_nl, n_lines, o,
                                                              reinterpret_cast<unsigned long long*>(misc + 1));
    CDX_CHECK_LAUNCH(ctx, "jsonl(parse)");
    if (int st = scan_excl(ctx, LoadRecordFlag{o.st}, n_lines, pos, false, srec, misc + 2)) return st;
    uint64_t hm[2];
    cudaMemcpyAsync(hm, misc + 1, 16, cudaMemcpyDeviceToHost, ctx->stream);
    e = cudaStreamSynchronize(ctx->stream);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "jsonl_parse");
    const uint64_t first_parse_bad = hm[0];
    const uint64_t nr = hm[1];
    if (nr > cap_records) return set_error(ctx, CDX_EINVAL, "jsonl_parse: more records than cap_records");
    // records (line order) + decoded string sizes
    uint64_t* r_line = carve<uint64_t>(p, nr + 1);
    uint32_t* pid_len = carve<uint32_t>(p, nr + 1);
    uint32_t* ans_len = carve<uint32_t>(p, nr + 1);
    uint64_t* pid_off = carve<uint64_t>(p, nr + 1);
    char* pid_arena = carve<char>(p, 3 * nbytes / 2 + 2 * nr + 64);
    uint8_t* why = carve<uint8_t>(p, nr + 1);
    uint64_t* k0 = carve<uint64_t>(p, nr + 1);
    uint64_t* k1 = carve<uint64_t>(p, nr + 1);
    uint32_t* v0 = carve<uint32_t>(p, nr + 1);
    uint32_t* v1 = carve<uint32_t>(p, nr + 1);
    uint32_t* lb = carve<uint32_t>(p, radix_scratch_words(nr + 1));
    if (static_cast<size_t>(p - s) > bytes) return set_error(ctx, CDX_ECUDA, "jsonl_parse: scratch layout overflow");
    if (nr) {
        gather_records<<<gridn(ctx, n_lines), 128, 0, ctx->stream>>>(text, o.st, pos, n_lines, o, step_index,
                                                                     token_offset, hesitant, r_line, pid_len, ans_len);
        CDX_CHECK_LAUNCH(ctx, "jsonl(records)");
        // arena offsets: exclusive scans of the decoded lengths
        if (int st = scan_excl(ctx, LoadU32{ans_len}, nr, answer_off, true, srec, nullptr)) return st;
        if (int st = scan_excl(ctx, LoadU32{pid_len}, nr, pid_off, true, srec, nullptr)) return st;
        write_strings<<<gridn(ctx, n_lines), 128, 0, ctx->stream>>>(text, nbytes, o.st, pos, n_lines, o, pid_off, pid_arena,
                                                                    answer_off, answer_arena);
        CDX_CHECK_LAUNCH(ctx, "jsonl(strings)");
        // exact program interning (sentinel-wrapped: trimming cannot merge ids).  A trace holds
        // one program id per ~P records, so most keys are distinct within any tile: the direct
        // one-thread-per-record form (CDX_JSONL_INTERN=ws: K1's tiled serving kernel)
        uint64_t np = 0;
        const char* iv = getenv("CDX_JSONL_INTERN");
        if (iv && std::strcmp(iv, "ws") == 0) {
            if (int st = cdx_canon_intern(ctx, pid_arena, pid_off, nr, nullptr, 0, program, nullptr, program_first, &np))
                return st;
        } else if (int st = canon_intern_direct(ctx, pid_arena, pid_off, nr, program, program_first, &np)) {
            return st;
        }
        *n_programs = np;
        if (program_off && program_arena) {
            unwrap_pids<<<gridn(ctx, nr + 1), 256, 0, ctx->stream>>>(pid_off, pid_arena, nr, program_off, program_arena);
            CDX_CHECK_LAUNCH(ctx, "jsonl(program ids)");
        }
        // previous record of the same program: stable sort by program id
        widen_ids<<<gridn(ctx, nr), 256, 0, ctx->stream>>>(program, nr, k0, v0);
        CDX_CHECK_LAUNCH(ctx, "jsonl(keys)");
        int which = 0;
        if (int st = radix_sort_pairs(ctx, k0, v0, k1, v1, nr, lb, &which)) return st;
        cudaMemsetAsync(why, 0, nr, ctx->stream);
        order_check<<<gridn(ctx, nr), 256, 0, ctx->stream>>>(which ? v1 : v0, which ? k1 : k0, nr, step_index,
                                                             token_offset, r_line,
                                                             reinterpret_cast<unsigned long long*>(misc + 1), why);
        CDX_CHECK_LAUNCH(ctx, "jsonl(order)");
    }
    uint64_t bad = 0;
    cudaMemcpyAsync(&bad, misc + 1, 8, cudaMemcpyDeviceToHost, ctx->stream);
    e = cudaStreamSynchronize(ctx->stream);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "jsonl_parse");
    if (bad != ~0ull) {
        std::string what;
        if (bad == first_parse_bad) {
            uint8_t stl = 0;
            cudaMemcpy(&stl, o.st + bad, 1, cudaMemcpyDeviceToHost);
            what = stl == L_BADJSON ? "invalid JSON"
                                    : (stl == L_UNSUPPORTED ? "missing or mistyped field: unsupported number "
                                                              "(outside the device parser's exact range)"
                                                            : "missing or mistyped field");
        } else {
            // the order violation at line `bad`: find its record (records are in line order)
            std::vector<uint64_t> lines(nr);
            std::vector<uint8_t> w(nr);
            cudaMemcpy(lines.data(), r_line, nr * 8, cudaMemcpyDeviceToHost);
            cudaMemcpy(w.data(), why, nr, cudaMemcpyDeviceToHost);
            const size_t r = static_cast<size_t>(std::lower_bound(lines.begin(), lines.end(), bad) - lines.begin());
            what = (r < nr && w[r] == 2) ? "step_index does not increase" : "token_offset does not increase";
        }
        return set_error(ctx, CDX_ERUNTIME, "trace line " + std::to_string(bad + 1) + ": " + what);
    }
    *n_records = nr;
    return CDX_OK;
}
