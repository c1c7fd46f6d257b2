// CSV ingestion on the device: the data format feeding device X (SURVEY §8(f) row 4,
// reference renyi::load_csv, proj/src/csv.cpp:63-115; read_record 13-47; parse_cell 49-60;
// contract proj/include/renyi/csv.hpp:8-15).
//
// The text is byte work, so the design is HBM/latency-bound and flat:
//   K1 csv_chunk_stats  one CTA per 8 KB chunk: quote parity of the chunk and, for BOTH possible
//                       quote states at the chunk start, the number of record ('\n') and field
//                       (',') separators outside quotes — one read of the text, no serial
//                       dependence between chunks;
//   K2 csv_chunk_scan   one CTA scans the per-chunk summaries: the true quote state at each chunk
//                       start and the global record / field index of its first separator;
//   K3 csv_emit         second read of the text: every separator writes its byte position, the
//                       record it closes fields for, and (for '\n') the record's last field;
//   K4 csv_records      one thread per record: blank-line rule and field-count check;
//   K5                  exclusive scan of the data-row flags (cub);
//   K6 csv_parse        one thread per cell: quote/CR removal on the fly and a strtod-exact parse
//                       (grammar of glibc strtod in the C locale; decimal values by Clinger's exact
//                       path, Eisel-Lemire, and exact big-decimal shifting for what those leave
//                       undecided; hex floats with round-to-nearest-even; inf/nan with glibc's
//                       payload rule) straight into the column-major n x d fp64 matrix.
// Errors keep the reference's first-failure order: the smallest (row, column) key wins, a
// row's field-count error (column 0) before its cells. Header names, the label column and error
// texts are strings, cleaned on the host from the caller's buffer by the same state machine.
#include <cub/cub.cuh>

#include <cstdio>
#include <cstring>
#include <fstream>
#include <limits>

#include "engine.h"
#include "pow10_table.h"

namespace rb {

namespace {

constexpr int kCsvThreads = 256;
constexpr int kCsvPerThread = 32;
constexpr int kCsvChunk = kCsvThreads * kCsvPerThread;  // bytes per CTA in K1 / K3

struct ChunkStats {
    uint32_t parity;  // quote count mod 2
    uint32_t nl[2];   // '\n' outside quotes, if the chunk starts outside (0) / inside (1) quotes
    uint32_t sep[2];  // ','  outside quotes, same
};

__device__ __forceinline__ void load_bytes(const uint8_t* t, int64_t off, uint8_t (&b)[kCsvPerThread]) {
    const uint4* p = reinterpret_cast<const uint4*>(t + off);
#pragma unroll
    for (int i = 0; i < kCsvPerThread / 16; ++i) {
        const uint4 u = p[i];
        memcpy(b + 16 * i, &u, 16);
    }
}

// XOR-exclusive prefix of one bit per thread over the CTA; *total = XOR of all
template <int THREADS>
__device__ __forceinline__ uint32_t block_xor_prefix(uint32_t bit, uint32_t* total) {
    __shared__ uint32_t warp_par[THREADS / 32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t bal = __ballot_sync(0xffffffffu, bit);
    const uint32_t in_warp = __popc(bal & ((1u << lane) - 1u)) & 1u;
    if (lane == 0) warp_par[warp] = __popc(bal) & 1u;
    __syncthreads();
    uint32_t before = 0, all = 0;
#pragma unroll
    for (int w = 0; w < THREADS / 32; ++w) {
        if (w < warp) before ^= warp_par[w];
        all ^= warp_par[w];
    }
    __syncthreads();
    *total = all;
    return before ^ in_warp;
}

__global__ void __launch_bounds__(kCsvThreads) csv_chunk_stats(const uint8_t* __restrict__ text,
                                                               ChunkStats* __restrict__ stats) {
    uint8_t b[kCsvPerThread];
    load_bytes(text, static_cast<int64_t>(blockIdx.x) * kCsvChunk + threadIdx.x * kCsvPerThread, b);
    uint32_t p = 0, nl[2] = {0, 0}, sp[2] = {0, 0};
#pragma unroll
    for (int i = 0; i < kCsvPerThread; ++i) {
        const uint8_t c = b[i];
        // the byte is outside quotes iff (start state) == p
        if (c == '"') p ^= 1u;
        else if (c == '\n') ++nl[p];
        else if (c == ',') ++sp[p];
    }
    uint32_t total;
    const uint32_t pre = block_xor_prefix<kCsvThreads>(p, &total);
    // chunk start state S: this thread starts in S ^ pre, so its counts for hypothesis S are [S ^ pre]
    uint32_t v[4] = {nl[pre], nl[pre ^ 1u], sp[pre], sp[pre ^ 1u]};
    using R = cub::BlockReduce<uint32_t, kCsvThreads>;
    __shared__ typename R::TempStorage tmp;
    uint32_t s[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        s[k] = R(tmp).Sum(v[k]);
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        ChunkStats o;
        o.parity = total;
        o.nl[0] = s[0], o.nl[1] = s[1], o.sep[0] = s[2], o.sep[1] = s[3];
        stats[blockIdx.x] = o;
    }
}

// one CTA: true start state and first record / field index of every chunk; totals in out3
__global__ void __launch_bounds__(1024) csv_chunk_scan(const ChunkStats* __restrict__ stats, int64_t chunks,
                                                       uint8_t* __restrict__ state, int64_t* __restrict__ rec0,
                                                       int64_t* __restrict__ fld0, int64_t* __restrict__ out3) {
    using Scan = cub::BlockScan<unsigned long long, 1024>;
    __shared__ typename Scan::TempStorage tmp;
    uint32_t carry_state = 0;
    unsigned long long carry_rec = 0, carry_fld = 0;
    for (int64_t base = 0; base < chunks; base += 1024) {
        const int64_t c = base + threadIdx.x;
        ChunkStats st{};
        if (c < chunks) st = stats[c];
        uint32_t tot;
        const uint32_t s = carry_state ^ block_xor_prefix<1024>(c < chunks ? st.parity : 0u, &tot);
        const unsigned long long nl = c < chunks ? st.nl[s] : 0, fl = c < chunks ? st.nl[s] + st.sep[s] : 0;
        // pack (fields, records) into one 64-bit scan: per-chunk counts are <= 8192, sums < 2^40
        unsigned long long pre_nl, pre_fl, agg_nl, agg_fl;
        Scan(tmp).ExclusiveSum(nl, pre_nl, agg_nl);
        __syncthreads();
        Scan(tmp).ExclusiveSum(fl, pre_fl, agg_fl);
        __syncthreads();
        if (c < chunks) {
            state[c] = static_cast<uint8_t>(s);
            rec0[c] = static_cast<int64_t>(carry_rec + pre_nl);
            fld0[c] = static_cast<int64_t>(carry_fld + pre_fl);
        }
        carry_state ^= tot;
        carry_rec += agg_nl;
        carry_fld += agg_fl;
    }
    if (threadIdx.x == 0) {
        out3[0] = static_cast<int64_t>(carry_rec);  // '\n' separators
        out3[1] = static_cast<int64_t>(carry_fld);  // all separators
        out3[2] = carry_state;                      // quote state at the end of the text
    }
}

__global__ void __launch_bounds__(kCsvThreads) csv_emit(const uint8_t* __restrict__ text, int64_t len,
                                                        const uint8_t* __restrict__ state,
                                                        const int64_t* __restrict__ rec0,
                                                        const int64_t* __restrict__ fld0,
                                                        int64_t* __restrict__ sep_pos, int64_t* __restrict__ fld_rec,
                                                        int64_t* __restrict__ rec_last) {
    const int64_t off = static_cast<int64_t>(blockIdx.x) * kCsvChunk + threadIdx.x * kCsvPerThread;
    uint8_t b[kCsvPerThread];
    load_bytes(text, off, b);
    uint32_t p = 0;
#pragma unroll
    for (int i = 0; i < kCsvPerThread; ++i) p ^= (b[i] == '"');
    uint32_t tot;
    const uint32_t s0 = state[blockIdx.x] ^ block_xor_prefix<kCsvThreads>(p, &tot);
    uint32_t s = s0, nl = 0, fl = 0;
#pragma unroll
    for (int i = 0; i < kCsvPerThread; ++i) {
        const uint8_t c = b[i];
        if (c == '"') s ^= 1u;
        else if (s == 0 && (c == '\n' || c == ',')) {
            ++fl;
            nl += (c == '\n');
        }
    }
    using Scan = cub::BlockScan<unsigned long long, kCsvThreads>;
    __shared__ typename Scan::TempStorage tmp;
    unsigned long long pre;
    Scan(tmp).ExclusiveSum((static_cast<unsigned long long>(fl) << 32) | nl, pre);
    int64_t f = fld0[blockIdx.x] + static_cast<int64_t>(pre >> 32);
    int64_t r = rec0[blockIdx.x] + static_cast<int64_t>(pre & 0xffffffffull);
    if (fl == 0) return;
    s = s0;
#pragma unroll
    for (int i = 0; i < kCsvPerThread; ++i) {
        const uint8_t c = b[i];
        if (c == '"') s ^= 1u;
        else if (s == 0 && (c == '\n' || c == ',')) {
            sep_pos[f] = off + i;
            fld_rec[f] = r;
            if (c == '\n') rec_last[r++] = f;
            ++f;
        }
    }
    (void)len;
}

// --------------------------------------------------------------------------------------------
// Cell text: read_record's quote handling (csv.cpp:19-41) applied on the fly. Every field starts
// outside quotes (it follows a separator outside quotes, or the start of the text).
struct CleanReader {
    const uint8_t* t;
    int64_t pos, end;
    int inq;
    __device__ __forceinline__ int next() {
        while (pos < end) {
            const int c = t[pos++];
            if (!inq) {
                if (c == '"') {
                    inq = 1;
                    continue;
                }
                if (c == '\r') continue;
                return c;
            }
            if (c == '"') {
                if (pos < end && t[pos] == '"') {  // "" inside quotes: a literal quote
                    ++pos;
                    return '"';
                }
                inq = 0;
                continue;
            }
            return c;
        }
        return -1;
    }
};

// strtod sees the cell through std::string::c_str(): the text ends at the first NUL
struct CStrReader {
    CleanReader r;
    bool done = false;
    __device__ __forceinline__ int get() {
        if (done) return -1;
        const int c = r.next();
        if (c <= 0) {
            done = true;
            return -1;
        }
        return c;
    }
};

__device__ __forceinline__ bool is_space_c(int c) { return c == ' ' || (c >= '\t' && c <= '\r'); }
__device__ __forceinline__ int lower_c(int c) { return (c >= 'A' && c <= 'Z') ? c + 32 : c; }
__device__ __forceinline__ int hexval(int c) {
    if (c >= '0' && c <= '9') return c - '0';
    const int l = lower_c(c);
    if (l >= 'a' && l <= 'f') return l - 'a' + 10;
    return -1;
}

// ---- exact decimal -> binary64 through decimal shifting (the classic slow path) ----
struct Dec {
    static constexpr int kMax = 800;  // digits kept; later nonzero digits only set trunc
    static constexpr int kPad = 20;   // room for the new leading digits of one left shift
    uint8_t d[kMax + kPad];
    int nd;
    int64_t dp;  // value = 0.d[0]d[1]... x 10^dp
    bool trunc;
};

__device__ void dec_trim(Dec& a) {
    while (a.nd > 0 && a.d[a.nd - 1] == 0) --a.nd;
    if (a.nd == 0) a.dp = 0;
}

constexpr int kMaxShift = 60;

__device__ void dec_rshift(Dec& a, int k) {  // a /= 2^k, k <= 60
    int r = 0, w = 0;
    uint64_t n = 0;
    for (; (n >> k) == 0; ++r) {
        if (r >= a.nd) {
            if (n == 0) {
                a.nd = 0;
                return;
            }
            while ((n >> k) == 0) {
                n *= 10;
                ++r;
            }
            break;
        }
        n = n * 10 + a.d[r];
    }
    a.dp -= r - 1;
    const uint64_t mask = (uint64_t(1) << k) - 1;
    for (; r < a.nd; ++r) {
        const uint64_t dig = n >> k;
        n &= mask;
        a.d[w++] = static_cast<uint8_t>(dig);
        n = n * 10 + a.d[r];
    }
    while (n > 0) {
        const uint64_t dig = n >> k;
        n &= mask;
        if (w < Dec::kMax) a.d[w++] = static_cast<uint8_t>(dig);
        else if (dig > 0) a.trunc = true;
        n *= 10;
    }
    a.nd = w;
    dec_trim(a);
}

__device__ void dec_lshift(Dec& a, int k) {  // a *= 2^k, k <= 60 (at most 19 new digits)
    int w = a.nd + Dec::kPad;
    uint64_t n = 0;
    for (int r = a.nd - 1; r >= 0; --r) {  // w - r stays kPad: unread digits are never overwritten
        n += static_cast<uint64_t>(a.d[r]) << k;
        const uint64_t q = n / 10;
        a.d[--w] = static_cast<uint8_t>(n - 10 * q);
        n = q;
    }
    while (n > 0) {
        const uint64_t q = n / 10;
        a.d[--w] = static_cast<uint8_t>(n - 10 * q);
        n = q;
    }
    const int delta = Dec::kPad - w;
    const int total = a.nd + delta;
    const int keep = total < Dec::kMax ? total : Dec::kMax;
    for (int i = 0; i < keep; ++i) a.d[i] = a.d[w + i];
    for (int i = keep; i < total; ++i)
        if (a.d[w + i]) a.trunc = true;
    a.nd = keep;
    a.dp += delta;
    dec_trim(a);
}

__device__ void dec_shift(Dec& a, int k) {
    if (a.nd == 0) return;
    if (k > 0) {
        while (k > kMaxShift) {
            dec_lshift(a, kMaxShift);
            k -= kMaxShift;
        }
        dec_lshift(a, k);
    } else if (k < 0) {
        while (k < -kMaxShift) {
            dec_rshift(a, kMaxShift);
            k += kMaxShift;
        }
        dec_rshift(a, -k);
    }
}

__device__ bool dec_round_up(const Dec& a, int64_t nd) {
    if (nd < 0 || nd >= a.nd) return false;
    if (a.d[nd] == 5 && nd + 1 == a.nd) {  // exactly halfway: round to even unless digits were dropped
        if (a.trunc) return true;
        return nd > 0 && (a.d[nd - 1] & 1);
    }
    return a.d[nd] >= 5;
}

__device__ uint64_t dec_rounded_integer(const Dec& a) {
    if (a.dp > 20) return ~uint64_t(0);
    int64_t i = 0;
    uint64_t n = 0;
    for (; i < a.dp && i < a.nd; ++i) n = n * 10 + a.d[i];
    for (; i < a.dp; ++i) n *= 10;
    if (dec_round_up(a, a.dp)) ++n;
    return n;
}

__device__ uint64_t dec_to_bits(Dec& a, bool neg) {
    constexpr int bias = -1023, mantbits = 52, expmax = 2047;
    const int powtab[9] = {1, 3, 6, 9, 13, 16, 19, 23, 26};
    int exp = 0;
    uint64_t mant = 0;
    bool overflow = false, zero = false;
    if (a.nd == 0 || a.dp < -330) {
        zero = true;
    } else if (a.dp > 310) {
        overflow = true;
    } else {
        while (a.dp > 0) {
            const int n = a.dp >= 9 ? 27 : powtab[a.dp];
            dec_shift(a, -n);
            exp += n;
        }
        while (a.dp < 0 || (a.dp == 0 && a.d[0] < 5)) {
            const int n = -a.dp >= 9 ? 27 : powtab[-a.dp];
            dec_shift(a, n);
            exp -= n;
        }
        --exp;  // value in [1, 2) x 2^exp
        if (exp < bias + 1) {
            const int n = bias + 1 - exp;
            dec_shift(a, -n);
            exp += n;
        }
        if (exp - bias >= expmax) {
            overflow = true;
        } else {
            dec_shift(a, 1 + mantbits);
            mant = dec_rounded_integer(a);
            if (mant == (uint64_t(2) << mantbits)) {
                mant >>= 1;
                ++exp;
                if (exp - bias >= expmax) overflow = true;
            }
            if (!overflow && (mant & (uint64_t(1) << mantbits)) == 0) exp = bias;  // subnormal
        }
    }
    if (zero) mant = 0, exp = bias;
    if (overflow) mant = 0, exp = expmax + bias;
    uint64_t bits = mant & ((uint64_t(1) << mantbits) - 1);
    bits |= static_cast<uint64_t>((exp - bias) & expmax) << mantbits;
    if (neg) bits |= uint64_t(1) << 63;
    return bits;
}

// m x 2^e2 (+ sticky below m's last bit) rounded to nearest-even binary64 (hex floats)
__device__ uint64_t bin_to_bits(uint64_t m, int64_t e2, bool sticky, bool neg) {
    const uint64_t sign = neg ? (uint64_t(1) << 63) : 0;
    if (m == 0) return sign;
    const int top = 63 - __clzll(static_cast<long long>(m));
    const int64_t E = top + e2;  // value in [2^E, 2^(E+1))
    if (E > 1023) return sign | 0x7ff0000000000000ull;
    const int64_t bits = E >= -1022 ? 53 : E + 1075;  // significant bits the result can hold
    const int64_t shift = top + 1 - bits;             // low bits of m to drop
    uint64_t kept;
    if (shift <= 0) {
        kept = m << (-shift);
    } else if (shift > 64) {
        kept = 0;  // below half of the smallest subnormal
        return sign;
    } else {
        kept = shift == 64 ? 0 : (m >> shift);
        const bool half = (m >> (shift - 1)) & 1;
        const bool rest = sticky || (shift >= 2 && (m & ((uint64_t(1) << (shift - 1)) - 1)) != 0);
        if (half && (rest || (kept & 1))) ++kept;
    }
    // kept < 2^53 (normal, with the implicit bit) or < 2^52 (subnormal); rounding may carry one bit
    if (E >= -1022) {
        int64_t ex = E;
        if (kept >> 53) {
            kept >>= 1;
            ++ex;
        }
        if (ex > 1023) return sign | 0x7ff0000000000000ull;
        return sign | (static_cast<uint64_t>(ex + 1023) << 52) | (kept & ((uint64_t(1) << 52) - 1));
    }
    return sign | kept;  // subnormal (a carry into bit 52 is exactly the smallest normal encoding)
}

__device__ __forceinline__ bool is_nchar(int c) {
    return (c >= '0' && c <= '9') || (c >= 'A' && c <= 'Z') || (c >= 'a' && c <= 'z') || c == '_';
}

// Eisel-Lemire: man x 10^e10 -> binary64 bits when the 128-bit product of the normalised mantissa and
// the truncated 128-bit mantissa of 10^e10 (pow10_table.h) decides the rounding. Returns false on a
// possible ambiguity, a subnormal or overflowing result, or e10 outside the table: the caller then
// takes the exact big-decimal path.
__device__ bool eisel_lemire(uint64_t man, int64_t e10, bool neg, uint64_t* bits) {
    if (man == 0 || e10 < kPow10Min || e10 > kPow10Max) return false;
    const int clz = __clzll(static_cast<long long>(man));
    man <<= clz;
    uint64_t ret_exp2 = static_cast<uint64_t>(((217706 * e10) >> 16) + 64 + 1023) - static_cast<uint64_t>(clz);
    const uint64_t* p = kPow10[e10 - kPow10Min];
    uint64_t x_hi = __umul64hi(man, p[1]), x_lo = man * p[1];
    if ((x_hi & 0x1FF) == 0x1FF && x_lo + man < man) {  // the low product could carry into the top bits
        const uint64_t y_hi = __umul64hi(man, p[0]), y_lo = man * p[0];
        uint64_t m_hi = x_hi, m_lo = x_lo + y_hi;
        if (m_lo < x_lo) ++m_hi;
        if ((m_hi & 0x1FF) == 0x1FF && m_lo + 1 == 0 && y_lo + man < man) return false;
        x_hi = m_hi, x_lo = m_lo;
    }
    const uint64_t msb = x_hi >> 63;
    uint64_t mant = x_hi >> (msb + 9);
    ret_exp2 -= 1 ^ msb;
    if (x_lo == 0 && (x_hi & 0x1FF) == 0 && (mant & 3) == 1) return false;  // exactly halfway: undecided
    mant += mant & 1;
    mant >>= 1;
    if (mant >> 53) {
        mant >>= 1;
        ++ret_exp2;
    }
    if (ret_exp2 - 1 >= 0x7FF - 1) return false;  // subnormal or overflow
    *bits = (ret_exp2 << 52) | (mant & 0x000FFFFFFFFFFFFFull) | (neg ? (uint64_t(1) << 63) : 0);
    return true;
}

// Decimal body (digits, optional '.', optional exponent) followed by trailing spaces and the end of the
// cell. c is the current character; zero0 = a leading '0' was already consumed. Values with at most 15
// significant digits and |e10| <= 22 are exact in one double operation (Clinger); up to 19 digits go
// through Eisel-Lemire, longer ones through Eisel-Lemire on both truncation brackets (w, w + 1);
// whatever stays undecided is re-read into the big decimal and converted exactly.
__device__ bool parse_decimal(CStrReader& in, int c, bool zero0, bool neg, const uint8_t* text, int64_t s,
                              int64_t e, double* out, Dec& dec) {
    int64_t nd_all = 0, dp = 0, ex = 0;
    bool dot = false, any = zero0, many = false;
    uint64_t w = 0;
    int wd = 0, pend = 0;
    for (;; c = in.get()) {
        if (c == '.' && !dot) {
            dot = true;
            dp = nd_all;
            continue;
        }
        if (!(c >= '0' && c <= '9')) break;
        any = true;
        if (c == '0' && nd_all == 0) {  // leading zero
            --dp;
            continue;
        }
        ++nd_all;
        if (c == '0') {
            ++pend;
        } else {
            if (many || wd + pend + 1 > 19) {  // w keeps the leading digits only; later ones are dropped
                many = true;
            } else {
                for (int z = 0; z < pend; ++z) w *= 10;
                w = w * 10 + static_cast<uint64_t>(c - '0');
                wd += pend + 1;
            }
            pend = 0;
        }
    }
    if (!any) return false;
    if (!dot) dp = nd_all;
    if (c == 'e' || c == 'E') {
        c = in.get();
        bool eneg = false;
        if (c == '+' || c == '-') {
            eneg = c == '-';
            c = in.get();
        }
        if (!(c >= '0' && c <= '9')) return false;
        for (; c >= '0' && c <= '9'; c = in.get())
            if (ex < 100000) ex = ex * 10 + (c - '0');
        if (eneg) ex = -ex;
    }
    while (c == ' ') c = in.get();
    if (c != -1) return false;
    const int64_t sig = nd_all - pend;  // significant digits without trailing zeros
    if (sig == 0) {
        *out = neg ? -0.0 : 0.0;
        return true;
    }
    // value = w x 10^e10 (w holds wd digits: all significant ones when !many, else the leading wd of them
    // and the value lies strictly between w x 10^e10 and (w + 1) x 10^e10)
    const int64_t e10 = dp + ex - wd;
    if (!many && sig <= 15 && e10 >= -22 && e10 <= 22) {
        constexpr double p10[23] = {1e0,  1e1,  1e2,  1e3,  1e4,  1e5,  1e6,  1e7,  1e8,  1e9,  1e10, 1e11,
                                    1e12, 1e13, 1e14, 1e15, 1e16, 1e17, 1e18, 1e19, 1e20, 1e21, 1e22};
        double v = static_cast<double>(w);
        v = e10 >= 0 ? v * p10[e10] : v / p10[-e10];
        *out = neg ? -v : v;
        return true;
    }
    {
        uint64_t b0 = 0, b1 = 1;
        const bool ok0 = eisel_lemire(w, e10, neg, &b0);
        const bool ok1 = many && ok0 && eisel_lemire(w + 1, e10, neg, &b1);
        if (ok0 && (!many || (ok1 && b0 == b1))) {
            memcpy(out, &b0, 8);
            return true;
        }
    }
    // exact path: the significant digits (first Dec::kMax kept, the rest only as a sticky flag)
    CStrReader in2{CleanReader{text, s, e, 0}};
    int d = in2.get();
    while (d >= 0 && is_space_c(d)) d = in2.get();
    if (d == '+' || d == '-') d = in2.get();
    dec.nd = 0;
    dec.dp = 0;
    dec.trunc = false;
    bool dot2 = false;
    int64_t all2 = 0;
    for (;; d = in2.get()) {
        if (d == '.' && !dot2) {
            dot2 = true;
            dec.dp = all2;
            continue;
        }
        if (!(d >= '0' && d <= '9')) break;
        if (d == '0' && all2 == 0) {
            --dec.dp;
            continue;
        }
        ++all2;
        if (dec.nd < Dec::kMax) dec.d[dec.nd++] = static_cast<uint8_t>(d - '0');
        else if (d != '0') dec.trunc = true;
    }
    if (!dot2) dec.dp = all2;
    dec.dp += ex;
    const uint64_t b = dec_to_bits(dec, neg);
    memcpy(out, &b, 8);
    return true;
}

// parse_cell (csv.cpp:49-60): std::strtod over the whole cell (glibc grammar, C locale: leading
// isspace, sign, decimal / hex float / inf / infinity / nan / nan(n-char-seq)), then only trailing
// spaces. Returns false for "not numeric".
__device__ bool parse_cell(const uint8_t* text, int64_t s, int64_t e, double* out, Dec& dec) {
    CStrReader in{CleanReader{text, s, e, 0}};
    int c = in.get();
    bool only_spaces = true;
    int64_t lead = 0;
    for (; c >= 0 && is_space_c(c); c = in.get(), ++lead) only_spaces &= c == ' ';
    if (c == -1) {
        // no conversion: strtod leaves end at the start, and parse_cell's trailing-space loop then walks
        // over a cell of spaces only — such a cell reads as 0 (csv.cpp:53-56); an empty one is an error
        if (lead > 0 && only_spaces) {
            *out = 0.0;
            return true;
        }
        return false;
    }
    bool neg = false;
    if (c == '+' || c == '-') {
        neg = c == '-';
        c = in.get();
    }
    uint64_t bits;
    const int lc = lower_c(c);
    if (lc == 'i') {
        if (lower_c(in.get()) != 'n' || lower_c(in.get()) != 'f') return false;
        c = in.get();
        if (lower_c(c) == 'i') {
            if (lower_c(in.get()) != 'n' || lower_c(in.get()) != 'i' || lower_c(in.get()) != 't' ||
                lower_c(in.get()) != 'y')
                return false;
            c = in.get();
        }
        bits = 0x7ff0000000000000ull;
    } else if (lc == 'n') {
        if (lower_c(in.get()) != 'a' || lower_c(in.get()) != 'n') return false;
        bits = 0x7ff8000000000000ull;
        c = in.get();
        if (c == '(') {
            // glibc: the n-char-sequence is read with strtoull(seq, &end, 0); when that consumes the whole
            // sequence its value becomes the payload (low 51 bits, quiet bit kept)
            int base = 10, st = 0;  // st: 0 start, 1 after a leading '0', 2 in digits, 3 stopped early
            int64_t ndig = 0;
            uint64_t v = 0;
            bool ovf = false, seen_x = false;
            for (c = in.get(); c >= 0 && is_nchar(c); c = in.get()) {
                if (st == 3) continue;
                if (st == 0) {
                    if (c == '0') {
                        st = 1;
                        ndig = 1;
                        base = 8;
                    } else if (c >= '1' && c <= '9') {
                        st = 2;
                        v = static_cast<uint64_t>(c - '0');
                        ndig = 1;
                    } else {
                        st = 3;
                    }
                    continue;
                }
                if (st == 1 && !seen_x && ndig == 1 && v == 0 && (c == 'x' || c == 'X')) {
                    seen_x = true;  // "0x" prefix: needs a hex digit, else strtoull stops after the '0'
                    base = 16;
                    ndig = 0;
                    continue;
                }
                const int dv = hexval(c);
                if (dv < 0 || dv >= base) {
                    st = 3;
                    continue;
                }
                const unsigned __int128 nv = static_cast<unsigned __int128>(v) * static_cast<unsigned>(base) +
                                             static_cast<unsigned>(dv);
                if (nv >> 64) ovf = true;
                v = static_cast<uint64_t>(nv);
                ++ndig;
            }
            if (c != ')') return false;
            c = in.get();
            const bool full = st != 3 && !(seen_x && ndig == 0);
            if (full) {
                const uint64_t mant = ovf ? ~uint64_t(0) : v;
                bits = 0x7ff8000000000000ull | (mant & ((uint64_t(1) << 51) - 1));
            }
        }
    } else if (c == '0') {
        const int c2 = in.get();
        if (c2 != 'x' && c2 != 'X') return parse_decimal(in, c2, true, neg, text, s, e, out, dec);
        // hex float: at least one hex digit, optional '.', optional binary exponent
        uint64_t m = 0;
        int64_t e2 = 0;
        bool sticky = false, any = false, dot = false;
        for (c = in.get();; c = in.get()) {
            if (c == '.' && !dot) {
                dot = true;
                continue;
            }
            const int h = hexval(c);
            if (h < 0) break;
            any = true;
            if (m >> 60) {  // 64-bit mantissa full: integer digits scale, fraction digits only stick
                sticky |= h != 0;
                if (!dot) e2 += 4;
            } else {
                m = (m << 4) | static_cast<uint64_t>(h);
                if (dot) e2 -= 4;
            }
        }
        if (!any) return false;
        if (c == 'p' || c == 'P') {
            c = in.get();
            bool eneg = false;
            if (c == '+' || c == '-') {
                eneg = c == '-';
                c = in.get();
            }
            if (!(c >= '0' && c <= '9')) return false;
            int64_t ev = 0;
            for (; c >= '0' && c <= '9'; c = in.get())
                if (ev < 100000) ev = ev * 10 + (c - '0');
            e2 += eneg ? -ev : ev;
        }
        while (c == ' ') c = in.get();
        if (c != -1) return false;
        const uint64_t b = bin_to_bits(m, e2, sticky, neg);
        memcpy(out, &b, 8);
        return true;
    } else {
        return parse_decimal(in, c, false, neg, text, s, e, out, dec);
    }
    if (neg) bits |= uint64_t(1) << 63;
    while (c == ' ') c = in.get();
    if (c != -1) return false;
    memcpy(out, &bits, 8);
    return true;
}

__device__ __forceinline__ int64_t field_start(const int64_t* sep_pos, int64_t f) {
    return f == 0 ? 0 : sep_pos[f - 1] + 1;
}

// K4: one thread per record r >= 1
__global__ void csv_records(const uint8_t* __restrict__ text, const int64_t* __restrict__ sep_pos,
                            const int64_t* __restrict__ rec_last, int64_t records, int64_t header_fields,
                            int* __restrict__ is_data, unsigned long long* __restrict__ err) {
    const int64_t r = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (r >= records) return;
    if (r == 0) {
        is_data[0] = 0;
        return;
    }
    const int64_t first = rec_last[r - 1] + 1, last = rec_last[r];
    const int64_t nf = last - first + 1;
    int data = 1;
    if (nf == 1) {  // blank line: one field whose cleaned text is empty (csv.cpp:89)
        CleanReader cr{text, field_start(sep_pos, first), sep_pos[first], 0};
        if (cr.next() < 0) data = 0;
    }
    if (data && nf != header_fields) {
        data = 0;
        atomicMin(err, static_cast<unsigned long long>(r + 1) << 24);  // row r+1, column 0: count error
    }
    is_data[r] = data;
}

// K6: one thread per field of the data records
__global__ void __launch_bounds__(128) csv_parse(const uint8_t* __restrict__ text, const int64_t* __restrict__ sep_pos,
                                                 const int64_t* __restrict__ fld_rec,
                                                 const int64_t* __restrict__ rec_last,
                                                 const int* __restrict__ is_data, const int* __restrict__ row_of,
                                                 int64_t f0, int64_t fields, int64_t n, int label,
                                                 double* __restrict__ x, int64_t* __restrict__ label_span,
                                                 unsigned long long* __restrict__ err) {
    const int64_t f = f0 + static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (f >= fields) return;
    const int64_t r = fld_rec[f];
    if (!is_data[r]) return;
    const int64_t col = f - (rec_last[r - 1] + 1);
    const int64_t i = row_of[r];
    const int64_t s = field_start(sep_pos, f), e = sep_pos[f];
    if (col == label) {
        label_span[2 * i] = s;
        label_span[2 * i + 1] = e;
        return;
    }
    Dec dec;
    double v;
    if (!parse_cell(text, s, e, &v, dec)) {
        atomicMin(err, (static_cast<unsigned long long>(r + 1) << 24) | static_cast<unsigned long long>(col + 1));
        return;
    }
    const int64_t j = (label >= 0 && col > label) ? col - 1 : col;
    x[j * n + i] = v;
}

__global__ void csv_set_tail(int64_t* sep_pos, int64_t* fld_rec, int64_t* rec_last, int64_t f, int64_t r, int64_t len) {
    sep_pos[f] = len;
    fld_rec[f] = r;
    rec_last[r] = f;
}

// host: read_record's cleaning of one field (names, labels, error text)
std::string clean_host(const char* t, int64_t s, int64_t e) {
    std::string out;
    bool inq = false;
    for (int64_t p = s; p < e; ++p) {
        const char c = t[p];
        if (!inq) {
            if (c == '"') inq = true;
            else if (c != '\r') out.push_back(c);
        } else if (c == '"') {
            if (p + 1 < e && t[p + 1] == '"') {
                out.push_back('"');
                ++p;
            } else {
                inq = false;
            }
        } else {
            out.push_back(c);
        }
    }
    return out;
}



}  // namespace

std::unique_ptr<Dataset> load_csv_text(Context& ctx, const char* text, size_t len, const char* label_column,
                                       const std::string& source) {
    cuda_check(cudaSetDevice(ctx.device()), "cudaSetDevice");
    const std::string src = "'" + source + "'";
    if (len == 0) fail(kParseError, src + ": missing header row");
    if (!text) fail(kInvalidArgument, "csv text is NULL");
    cudaStream_t st = ctx.stream();
    const int64_t L = static_cast<int64_t>(len);
    const int64_t chunks = (L + kCsvChunk - 1) / kCsvChunk;
    DevBuf dtext, dstats, dstate, drec0, dfld0, dtot;
    dtext.alloc(static_cast<size_t>(chunks) * kCsvChunk);
    cuda_check(cudaMemsetAsync(dtext.as<uint8_t>() + L, 0, static_cast<size_t>(chunks) * kCsvChunk - L, st),
               "memset");
    h2d_staged(ctx, dtext.as<void>(), text, len);  // engine.cu: page-locked double buffering
    dstats.alloc(static_cast<size_t>(chunks) * sizeof(ChunkStats));
    dstate.alloc(static_cast<size_t>(chunks));
    drec0.alloc(static_cast<size_t>(chunks) * sizeof(int64_t));
    dfld0.alloc(static_cast<size_t>(chunks) * sizeof(int64_t));
    dtot.alloc(4 * sizeof(int64_t));
    const uint8_t* t = dtext.as<uint8_t>();
    csv_chunk_stats<<<static_cast<unsigned>(chunks), kCsvThreads, 0, st>>>(t, dstats.as<ChunkStats>());
    cuda_check(cudaGetLastError(), "csv_chunk_stats");
    csv_chunk_scan<<<1, 1024, 0, st>>>(dstats.as<ChunkStats>(), chunks, dstate.as<uint8_t>(), drec0.as<int64_t>(),
                                       dfld0.as<int64_t>(), dtot.as<int64_t>());
    cuda_check(cudaGetLastError(), "csv_chunk_scan");
    ctx.launches += 2;
    int64_t tot[3];
    d2h(ctx, tot, dtot.as<void>(), sizeof(tot));
    ctx.sync();
    const int64_t n_nl = tot[0], n_sep = tot[1];
    DevBuf dsep, dfrec, drlast;
    dsep.alloc(static_cast<size_t>(n_sep + 1) * sizeof(int64_t));
    dfrec.alloc(static_cast<size_t>(n_sep + 1) * sizeof(int64_t));
    drlast.alloc(static_cast<size_t>(n_nl + 1) * sizeof(int64_t));
    csv_emit<<<static_cast<unsigned>(chunks), kCsvThreads, 0, st>>>(t, L, dstate.as<uint8_t>(), drec0.as<int64_t>(),
                                                                    dfld0.as<int64_t>(), dsep.as<int64_t>(),
                                                                    dfrec.as<int64_t>(), drlast.as<int64_t>());
    cuda_check(cudaGetLastError(), "csv_emit");
    ++ctx.launches;
    // a record ends at EOF when bytes follow the last '\n' separator (read_record returns data at EOF)
    int64_t last_nl = -1;
    if (n_nl > 0) {
        int64_t f_last;
        d2h(ctx, &f_last, drlast.as<int64_t>() + (n_nl - 1), sizeof(int64_t));
        ctx.sync();
        d2h(ctx, &last_nl, dsep.as<int64_t>() + f_last, sizeof(int64_t));
        ctx.sync();
    }
    const bool tail = last_nl < L - 1;
    const int64_t F = n_sep + (tail ? 1 : 0), R = n_nl + (tail ? 1 : 0);
    if (tail) {
        csv_set_tail<<<1, 1, 0, st>>>(dsep.as<int64_t>(), dfrec.as<int64_t>(), drlast.as<int64_t>(), F - 1, R - 1, L);
        cuda_check(cudaGetLastError(), "csv_set_tail");
        ++ctx.launches;
    }
    // header: record 0
    int64_t H;
    d2h(ctx, &H, drlast.as<int64_t>(), sizeof(int64_t));
    ctx.sync();
    H += 1;
    std::vector<int64_t> hsep(static_cast<size_t>(H));
    d2h(ctx, hsep.data(), dsep.as<int64_t>(), static_cast<size_t>(H) * sizeof(int64_t));
    ctx.sync();
    auto ds = std::make_unique<Dataset>();
    std::vector<std::string> header(static_cast<size_t>(H));
    for (int64_t j = 0; j < H; ++j) header[j] = clean_host(text, j == 0 ? 0 : hsep[j - 1] + 1, hsep[j]);
    int label = -1;
    if (label_column) {
        for (int64_t j = 0; j < H; ++j)
            if (header[j] == label_column) label = static_cast<int>(j);
        if (label < 0) fail(kParseError, src + ": no column named '" + std::string(label_column) + "'");
    }
    for (int64_t j = 0; j < H; ++j)
        if (j != label) ds->names.push_back(header[j]);
    // records: blank lines, field counts
    DevBuf dis, drow, derr;
    dis.alloc(static_cast<size_t>(R) * sizeof(int));
    drow.alloc(static_cast<size_t>(R) * sizeof(int));
    derr.alloc(sizeof(unsigned long long));
    cuda_check(cudaMemsetAsync(derr.as<void>(), 0xff, sizeof(unsigned long long), st), "memset");
    csv_records<<<static_cast<unsigned>((R + 255) / 256), 256, 0, st>>>(t, dsep.as<int64_t>(), drlast.as<int64_t>(), R,
                                                                        H, dis.as<int>(), derr.as<unsigned long long>());
    cuda_check(cudaGetLastError(), "csv_records");
    ++ctx.launches;
    size_t tmp_bytes = 0;
    cuda_check(cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, dis.as<int>(), drow.as<int>(), static_cast<int>(R), st),
               "scan");
    DevBuf dtmp;
    dtmp.alloc(tmp_bytes > 0 ? tmp_bytes : 1);
    cuda_check(cub::DeviceScan::ExclusiveSum(dtmp.as<void>(), tmp_bytes, dis.as<int>(), drow.as<int>(),
                                             static_cast<int>(R), st),
               "scan");
    ++ctx.launches;
    int lastv[2];
    d2h(ctx, &lastv[0], dis.as<int>() + (R - 1), sizeof(int));
    d2h(ctx, &lastv[1], drow.as<int>() + (R - 1), sizeof(int));
    ctx.sync();
    const int64_t n = static_cast<int64_t>(lastv[0]) + lastv[1];
    const int64_t d = H - (label >= 0 ? 1 : 0);
    ds->n = n;
    ds->d = d;
    ds->features.alloc(static_cast<size_t>(n > 0 ? n : 1) * (d > 0 ? d : 1) * sizeof(double));
    DevBuf dlab;
    if (label >= 0) dlab.alloc(static_cast<size_t>(n > 0 ? n : 1) * 2 * sizeof(int64_t));
    if (F > H) {
        csv_parse<<<static_cast<unsigned>((F - H + 127) / 128), 128, 0, st>>>(
            t, dsep.as<int64_t>(), dfrec.as<int64_t>(), drlast.as<int64_t>(), dis.as<int>(), drow.as<int>(), H, F, n,
            label, ds->features.as<double>(), label >= 0 ? dlab.as<int64_t>() : nullptr,
            derr.as<unsigned long long>());
        cuda_check(cudaGetLastError(), "csv_parse");
        ++ctx.launches;
    }
    unsigned long long ek;
    d2h(ctx, &ek, derr.as<void>(), sizeof(ek));
    ctx.sync();
    if (ek != ~0ull) {
        const int64_t row = static_cast<int64_t>(ek >> 24), col = static_cast<int64_t>(ek & 0xffffff);
        const int64_t r = row - 1;
        int64_t bounds[2];
        d2h(ctx, bounds, drlast.as<int64_t>() + (r - 1), 2 * sizeof(int64_t));
        ctx.sync();
        if (col == 0)
            fail(kParseError, "row " + std::to_string(row) + ": expected " + std::to_string(H) + " fields, got " +
                                  std::to_string(bounds[1] - bounds[0]));
        const int64_t f = bounds[0] + col;  // first field of the row is bounds[0] + 1
        int64_t se[2];
        d2h(ctx, se, dsep.as<int64_t>() + (f - 1), 2 * sizeof(int64_t));
        ctx.sync();
        fail(kParseError, "row " + std::to_string(row) + ", column " + std::to_string(col) + ": '" +
                              clean_host(text, se[0] + 1, se[1]) + "' is not numeric");
    }
    if (n < 2) fail(kParseError, src + ": need at least 2 data rows, got " + std::to_string(n));
    if (label >= 0) {
        std::vector<int64_t> spans(static_cast<size_t>(2 * n));
        d2h(ctx, spans.data(), dlab.as<void>(), spans.size() * sizeof(int64_t));
        ctx.sync();
        ds->labels.reserve(static_cast<size_t>(n));
        for (int64_t i = 0; i < n; ++i) ds->labels.push_back(clean_host(text, spans[2 * i], spans[2 * i + 1]));
    }
    return ds;
}

std::unique_ptr<Dataset> load_csv_file(Context& ctx, const std::string& path, const char* label_column) {
    std::ifstream in(path, std::ios::binary);
    if (!in) fail(kParseError, "cannot open '" + path + "'");
    in.seekg(0, std::ios::end);
    const std::streamoff size = in.tellg();
    in.seekg(0, std::ios::beg);
    std::string buf(static_cast<size_t>(size > 0 ? size : 0), '\0');
    if (size > 0) in.read(buf.data(), size);
    return load_csv_text(ctx, buf.data(), buf.size(), label_column, path);
}

}  // namespace rb
