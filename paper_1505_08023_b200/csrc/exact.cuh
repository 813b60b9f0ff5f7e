// exact.cuh — exactly-rounded dot products on the device (reading C5).
//
// dot(u,v) = RN( sum_i^exact fl(u_i * v_i) ): independent of summation order, tiling and
// rank count, which is what makes the GPU CG bit-identical to the oracle and to itself at any
// partition (any ulp-level change in a dot changes ||r_k|| by O(1) within 50
// iterations on this problem, so nothing weaker meets the north-star tolerances).
//
// Three levels, all exact:
//   1. per thread: a floating-point expansion of NEXP doubles, updated by Knuth's TwoSum
//      cascade; whatever the last level cannot hold ("spill") goes to level 2;
//   2. per CTA: a fixed-point superaccumulator in shared memory: ACC_DIGITS signed int64
//      words, word i weighting 2^(32 i - 1074); a double adds < 2^33 to each of <= 3 words;
//   3. per rank / globally: the CTA words are added to a global copy with int64 atomicAdd;
//      across ranks an int64-SUM all-reduce (associative, so deterministic).
// A consumer kernel normalises the carries and rounds once (acc_finalize_warp).
// Capacity: < 2^29 additions per accumulator word (any n < 5e8 terms) keeps every word and
// carry inside int64.  Word ACC_FLAG counts non-finite inputs (then the result is NaN).
#pragma once
#include <cstdint>

namespace minife {

constexpr int ACC_DIGITS = 68;            // bits 0..2175 relative to 2^-1074
constexpr int ACC_FLAG = ACC_DIGITS;      // non-finite counter
constexpr int ACC_WORDS = 72;             // padded (576 B)
constexpr int NEXP = 4;                   // expansion length per thread

__device__ __forceinline__ void two_sum(double a, double b, double &s, double &e) {
    s = __dadd_rn(a, b);
    const double bb = __dsub_rn(s, a);
    e = __dadd_rn(__dsub_rn(a, __dsub_rn(s, bb)), __dsub_rn(b, bb));
}

// Add one double to a superaccumulator (shared or global words) with 64-bit atomics.
__device__ __forceinline__ void acc_add(unsigned long long *w, double x) {
    const unsigned long long bits = (unsigned long long)__double_as_longlong(x);
    const int e = (int)((bits >> 52) & 0x7ff);
    const unsigned long long frac = bits & 0xfffffffffffffull;
    if (e == 0x7ff) {                      // inf / nan
        atomicAdd(&w[ACC_FLAG], 1ull);
        return;
    }
    if (e == 0 && frac == 0) return;
    // x = m * 2^(pos - 1074)
    const unsigned long long m = e ? (frac | (1ull << 52)) : frac;
    const int pos = e ? e - 1 : 0;
    const int d = pos >> 5, s = pos & 31;
    const unsigned long long a = (m & 0xffffffffull) << s;   // < 2^63
    const unsigned long long b = (m >> 32) << s;             // < 2^53
    long long w0 = (long long)(a & 0xffffffffull);
    long long w1 = (long long)((a >> 32) + (b & 0xffffffffull));
    long long w2 = (long long)(b >> 32);
    if (bits >> 63) {
        w0 = -w0;
        w1 = -w1;
        w2 = -w2;
    }
    if (w0) atomicAdd(&w[d], (unsigned long long)w0);
    if (w1) atomicAdd(&w[d + 1], (unsigned long long)w1);
    if (w2) atomicAdd(&w[d + 2], (unsigned long long)w2);
}

struct Expansion {
    double c[NEXP];
    __device__ __forceinline__ void init() {
#pragma unroll
        for (int j = 0; j < NEXP; ++j) c[j] = 0.0;
    }
    // exact: c[0]+..+c[NEXP-1] (+ spilled) == previous total + x, always
    __device__ __forceinline__ void add(double x, unsigned long long *spill) {
#pragma unroll
        for (int j = 0; j < NEXP; ++j) two_sum(c[j], x, c[j], x);
        if (x != 0.0) acc_add(spill, x);   // also routes NaN to the flag word
    }
    __device__ __forceinline__ void flush(unsigned long long *acc) const {
#pragma unroll
        for (int j = 0; j < NEXP; ++j)
            if (c[j] != 0.0) acc_add(acc, c[j]);
    }
    // Warp-aggregated flush (all 32 lanes must call it, converged).  For each component
    // index j the lanes' values are cut into signed 16-bit chunks on a common grid anchored
    // at the warp's largest value (digit D weighs 2^(16 D - 1074)); 13 integer warp sums
    // (REDUX) cover the window D in [Dmax-8, Dmax+4], and lane 0 adds each nonzero sum
    // (|sum| < 2^21) to the accumulator word D/2.  A value more than 128 bits below the
    // warp's largest one, or non-finite, takes acc_add.  Exact: integer sums of exact chunks.
    __device__ __forceinline__ void warp_flush(unsigned long long *acc) const {
        const unsigned FULL = 0xffffffffu;
        const unsigned lane = threadIdx.x & 31u;
#pragma unroll
        for (int j = 0; j < NEXP; ++j) {
            const double v = c[j];
            const unsigned long long bits = (unsigned long long)__double_as_longlong(v);
            const int e = (int)((bits >> 52) & 0x7ff);
            const unsigned long long frac = bits & 0xfffffffffffffull;
            const bool nz = (e != 0 || frac != 0) && e != 0x7ff;
            const unsigned long long m = e ? (frac | (1ull << 52)) : frac;
            const int pos = e ? e - 1 : 0;
            const int d16 = pos >> 4, s16 = pos & 15;
            const unsigned dmax1 = __reduce_max_sync(FULL, nz ? (unsigned)d16 + 1u : 0u);
            if (e == 0x7ff) acc_add(acc, v);                      // flag word
            if (dmax1 == 0u) continue;                            // warp-uniform
            const int lo = (int)dmax1 - 1 - 8;
            const bool inwin = nz && d16 >= lo;
            if (nz && !inwin) acc_add(acc, v);                    // far below: slow path
            // m << s16 as five 16-bit chunks (m < 2^53, s16 < 16: < 2^69)
            const unsigned long long mlo = m << s16;
            const unsigned long long mhi = s16 ? (m >> (64 - s16)) : 0ull;
            int ch[5];
            ch[0] = (int)(mlo & 0xffff);
            ch[1] = (int)((mlo >> 16) & 0xffff);
            ch[2] = (int)((mlo >> 32) & 0xffff);
            ch[3] = (int)(mlo >> 48);
            ch[4] = (int)mhi;
            if (bits >> 63) {
#pragma unroll
                for (int q = 0; q < 5; ++q) ch[q] = -ch[q];
            }
#pragma unroll
            for (int t = 0; t < 13; ++t) {
                const int D = lo + t;
                const int q = D - d16;
                int contrib = 0;
#pragma unroll
                for (int qq = 0; qq < 5; ++qq) contrib = (inwin && q == qq) ? ch[qq] : contrib;
                const int sum = __reduce_add_sync(FULL, contrib);
                if (lane == 0 && sum != 0 && D >= 0) {
                    const long long val = (long long)sum * ((D & 1) ? 65536ll : 1ll);
                    atomicAdd(&acc[D >> 1], (unsigned long long)val);
                }
            }
        }
    }
};

// 16-bit digit grid of warp_flush as 32-bit shared counters: dig[D] weighs 2^(16 D - 1074).
// A warp contributes |sum| < 2^21 per digit, so a CTA of <= 1024 warps stays inside int32,
// and 32-bit shared atomics are native (the 64-bit ones are CAS loops).
constexpr int ACC_DIG16 = 2 * ACC_DIGITS;

#ifdef FLUSH_STATS
// Diagnostic builds only (tools/flush_stats.py): [kernel: 0 SpMV, 1 K6 (256 threads)][calls
// with a nonzero value, lanes on the slow path, sum of warp sums, calls]
static __device__ unsigned long long g_flush_stats[2][4];
#endif
// One value per lane into the 16-bit digit counters, warp-aggregated (all lanes, converged)
__device__ __forceinline__ void flush_value_digits(double v, int *dig, unsigned long long *acc) {
    const unsigned FULL = 0xffffffffu;
    const unsigned lane = threadIdx.x & 31u;
    const unsigned long long bits = (unsigned long long)__double_as_longlong(v);
    const int e = (int)((bits >> 52) & 0x7ff);
    const unsigned long long frac = bits & 0xfffffffffffffull;
    const bool nz = (e != 0 || frac != 0) && e != 0x7ff;
    const unsigned long long m = e ? (frac | (1ull << 52)) : frac;
    const int pos = e ? e - 1 : 0;
    const int d16 = pos >> 4, s16 = pos & 15;
    const unsigned dmax1 = __reduce_max_sync(FULL, nz ? (unsigned)d16 + 1u : 0u);
#ifdef FLUSH_STATS
    if (lane == 0) atomicAdd(&g_flush_stats[blockDim.x == 256 ? 1 : 0][3], 1ull);
#endif
    if (e == 0x7ff) acc_add(acc, v);                          // flag word
    if (dmax1 == 0u) return;                                  // warp-uniform
    const unsigned long long mlo = m << s16;
    const unsigned long long mhi = s16 ? (m >> (64 - s16)) : 0ull;
    int ch[5];
    ch[0] = (int)(mlo & 0xffff);
    ch[1] = (int)((mlo >> 16) & 0xffff);
    ch[2] = (int)((mlo >> 32) & 0xffff);
    ch[3] = (int)(mlo >> 48);
    ch[4] = (int)mhi;
    if (bits >> 63) {
#pragma unroll
        for (int q = 0; q < 5; ++q) ch[q] = -ch[q];
    }
    if (__all_sync(FULL, !nz || d16 == (int)dmax1 - 1)) {
        // every nonzero lane has the same top digit (the usual case): the window is that
        // digit's five chunks, summed straight across the warp
        int mine = 0;
#pragma unroll
        for (int t = 0; t < 5; ++t) {
            const int sum = __reduce_add_sync(FULL, nz ? ch[t] : 0);
            mine = lane == (unsigned)t ? sum : mine;
        }
        const int D = (int)dmax1 - 1 + (int)lane;
        if (lane < 5u && mine != 0 && D < ACC_DIG16) atomicAdd(&dig[D], mine);
#ifdef FLUSH_STATS
        if (lane == 0) {
            const int kk = blockDim.x == 256 ? 1 : 0;
            atomicAdd(&g_flush_stats[kk][0], 1ull);
            atomicAdd(&g_flush_stats[kk][2], 5ull);
        }
#endif
        return;
    }
    if (__all_sync(FULL, !nz || d16 >= (int)dmax1 - 2)) {
        // top digits one apart: a 6-digit window from dmax - 1; a lane whose top digit is
        // dmax contributes its chunk t - 1 to window digit t
        const bool up = nz && d16 == (int)dmax1 - 1;
        int mine = 0;
#pragma unroll
        for (int t = 0; t < 6; ++t) {
            const int c = !nz ? 0 : (up ? (t >= 1 ? ch[t - 1] : 0) : (t <= 4 ? ch[t] : 0));
            const int sum = __reduce_add_sync(FULL, c);
            mine = lane == (unsigned)t ? sum : mine;
        }
        const int D = (int)dmax1 - 2 + (int)lane;
        if (lane < 6u && mine != 0 && D >= 0 && D < ACC_DIG16) atomicAdd(&dig[D], mine);
#ifdef FLUSH_STATS
        if (lane == 0) {
            const int kk = blockDim.x == 256 ? 1 : 0;
            atomicAdd(&g_flush_stats[kk][0], 1ull);
            atomicAdd(&g_flush_stats[kk][2], 6ull);
        }
#endif
        return;
    }
    const bool inwin = nz && d16 >= (int)dmax1 - 1 - 8;
    if (nz && !inwin) acc_add(acc, v);                        // far below: slow path
    // window [lo, dmax + 4]: from the lowest in-window digit, so lanes of similar magnitude
    // need ~6 warp sums instead of 13
    const int lo = (int)__reduce_min_sync(FULL, inwin ? (unsigned)d16 : 0xffffffffu);
    const int nsum = (int)dmax1 + 4 - lo;
#ifdef FLUSH_STATS
    {
        const unsigned slow = __popc(__ballot_sync(FULL, nz && !inwin));
        if (lane == 0) {
            const int kk = blockDim.x == 256 ? 1 : 0;
            atomicAdd(&g_flush_stats[kk][0], 1ull);
            atomicAdd(&g_flush_stats[kk][1], (unsigned long long)slow);
            atomicAdd(&g_flush_stats[kk][2], (unsigned long long)nsum);
        }
    }
#endif
    // the nsum (<= 13) warp sums back to back, then lane t adds sum t
    int mine = 0;
#pragma unroll
    for (int t = 0; t < 13; ++t) {
        if (t < nsum) {                                       // warp-uniform
            const int q = lo + t - d16;
            int contrib = 0;
#pragma unroll
            for (int qq = 0; qq < 5; ++qq) contrib = (inwin && q == qq) ? ch[qq] : contrib;
            const int sum = __reduce_add_sync(FULL, contrib);
            mine = lane == (unsigned)t ? sum : mine;
        }
    }
    const int D = lo + (int)lane;
    if ((int)lane < nsum && mine != 0 && D >= 0 && D < ACC_DIG16) atomicAdd(&dig[D], mine);
}

__device__ __forceinline__ void expansion_flush_digits(const Expansion &ex, int *dig,
                                                       unsigned long long *acc) {
#pragma unroll
    for (int j = 0; j < NEXP; ++j) flush_value_digits(ex.c[j], dig, acc);
}

// Tiered expansion for long per-thread sums: what the first expansion (N1 terms) cannot hold
// -- a term far below its running total, e.g. late in CG the Dirichlet rows' tiny products --
// goes to a second one (N2 terms), then a third (N3, optional), and only what none holds
// reaches the shared-memory atomics (64-bit CAS loops).  Exact like Expansion; costs nothing
// while the first tier absorbs every term.
#ifdef EXP_STATS
// Diagnostic builds only: how many additions reach the second tier / the shared atomics
static __device__ unsigned long long g_exp_stats[4];
extern "C" int minife_dbg_exp_stats(unsigned long long *out, int reset);
#endif
template <int N1, int N2, int N3 = 0> struct ExpansionT {
    double a[N1], b[N2], c[N3 > 0 ? N3 : 1];
#ifdef EXP_STATS
    unsigned n_add = 0, n_t2 = 0, n_spill = 0;
#endif
    __device__ __forceinline__ void init() {
#pragma unroll
        for (int j = 0; j < N1; ++j) a[j] = 0.0;
#pragma unroll
        for (int j = 0; j < N2; ++j) b[j] = 0.0;
#pragma unroll
        for (int j = 0; j < N3; ++j) c[j] = 0.0;
    }
    __device__ __forceinline__ void add(double x, unsigned long long *spill) {
#ifdef EXP_STATS
        ++n_add;
#endif
#pragma unroll
        for (int j = 0; j < N1; ++j) two_sum(a[j], x, a[j], x);
        if (x != 0.0) {
#ifdef EXP_STATS
            ++n_t2;
#endif
#pragma unroll
            for (int j = 0; j < N2; ++j) two_sum(b[j], x, b[j], x);

            if (N3 > 0 && x != 0.0) {
#pragma unroll
                for (int j = 0; j < N3; ++j) two_sum(c[j], x, c[j], x);
            }
#ifdef EXP_STATS
            if (x != 0.0) ++n_spill;
#endif
            if (x != 0.0) acc_add(spill, x);  // also routes NaN to the flag word
        }
    }
};
using Expansion2 = ExpansionT<NEXP, NEXP>;

template <int N1, int N2, int N3>
__device__ __forceinline__ void expansion_flush_digits(const ExpansionT<N1, N2, N3> &ex, int *dig,
                                                       unsigned long long *acc) {
#ifdef EXP_STATS
    {
        const unsigned v[3] = {ex.n_add, ex.n_t2, ex.n_spill};
        for (int q = 0; q < 3; ++q) {
            const unsigned t = __reduce_add_sync(0xffffffffu, v[q]);
            if ((threadIdx.x & 31) == 0) atomicAdd(&g_exp_stats[q], (unsigned long long)t);
        }
    }
#endif
#pragma unroll
    for (int j = 0; j < N1; ++j) flush_value_digits(ex.a[j], dig, acc);
#pragma unroll
    for (int j = 0; j < N2; ++j) flush_value_digits(ex.b[j], dig, acc);
#pragma unroll
    for (int j = 0; j < N3; ++j) flush_value_digits(ex.c[j], dig, acc);
}

__device__ __forceinline__ void acc_zero_shared(unsigned long long *s, int *dig) {
    for (int i = threadIdx.x; i < ACC_WORDS; i += blockDim.x) s[i] = 0ull;
    for (int i = threadIdx.x; i < ACC_DIG16; i += blockDim.x) dig[i] = 0;
}
__device__ __forceinline__ void acc_merge_to_global(const unsigned long long *s, const int *dig,
                                                    unsigned long long *g) {
    for (int w = threadIdx.x; w < ACC_WORDS; w += blockDim.x) {
        long long v = (long long)s[w];
        if (w < ACC_DIGITS) v += (long long)dig[2 * w] + (long long)dig[2 * w + 1] * 65536ll;
        if (v) atomicAdd(&g[w], (unsigned long long)v);
    }
}

// acc[w] += dig[2w] + 2^16 dig[2w+1] (one warp), then dig = 0
__device__ __forceinline__ void digits_to_words(int *dig, unsigned long long *acc) {
    for (int w = threadIdx.x & 31; w < ACC_DIGITS; w += 32) {
        const long long v = (long long)dig[2 * w] + (long long)dig[2 * w + 1] * 65536ll;
        acc[w] += (unsigned long long)v;
        dig[2 * w] = 0;
        dig[2 * w + 1] = 0;
    }
}

// CTA helpers: zero the shared words (all threads), merge them into a global accumulator.
__device__ __forceinline__ void acc_zero_shared(unsigned long long *s) {
    for (int i = threadIdx.x; i < ACC_WORDS; i += blockDim.x) s[i] = 0ull;
}
__device__ __forceinline__ void acc_merge_to_global(const unsigned long long *s,
                                                    unsigned long long *g) {
    for (int i = threadIdx.x; i < ACC_WORDS; i += blockDim.x) {
        const unsigned long long v = s[i];
        if (v) atomicAdd(&g[i], v);
    }
}

// Cooperative copy of a global accumulator into shared memory (all threads of the CTA).
__device__ __forceinline__ void acc_load_shared(unsigned long long *s,
                                                const unsigned long long *g) {
    for (int i = threadIdx.x; i < ACC_WORDS; i += blockDim.x) s[i] = __ldcg(g + i);
}

// Round a 96-bit window (digits T, T-1, T-2 of the magnitude, 32 bits each) plus a sticky
// bit to nearest-even; T = index of the top nonzero digit (units of 2^(32 T - 1074)).
__device__ __forceinline__ double round_window(int T, uint32_t dT, uint32_t d1, uint32_t d2,
                                               bool below) {
    const int t = 32 * T + 31 - __clz(dT);     // top bit, in units of 2^-1074
    if (t <= 52) {                             // T <= 1: the value is digits T..0, exact
        const unsigned long long v =
            T == 1 ? ((unsigned long long)dT << 32) | d1 : (unsigned long long)dT;
        return scalbn((double)v, -1074);       // < 2^53 ulps of 2^-1074: exact
    }
    const unsigned __int128 W = ((unsigned __int128)dT << 64) |
                                ((unsigned __int128)d1 << 32) | (unsigned __int128)d2;
    const int sh = t - 32 * (T - 2);           // top bit position inside W, in [64, 95]
    unsigned long long M = (unsigned long long)(W >> (sh - 52));   // 53 bits
    const int guard = (int)((W >> (sh - 53)) & 1u);
    const bool sticky = below || (W & ((((unsigned __int128)1) << (sh - 53)) - 1)) != 0;
    int top = t;
    if (guard && (sticky || (M & 1ull))) {
        ++M;
        if (M == (1ull << 53)) {
            M >>= 1;
            ++top;
        }
    }
    return scalbn((double)M, top - 52 - 1074);   // inf iff round-to-nearest overflows
}

// Carry maps of the warp-parallel normalisation: a digit with pre-carry value u (in
// [-2^31, 2^32 + 2^31)) maps an incoming carry c in {-1, 0, 1} to floor((u + c) / 2^32),
// again in {-1, 0, 1}.  Encoded as three 2-bit fields (field c+1 holds result+1).
__device__ __forceinline__ unsigned carry_map(long long u) {
    unsigned m = 0;
#pragma unroll
    for (int c = 0; c < 3; ++c) m |= (unsigned)(((u + (c - 1)) >> 32) + 1) << (2 * c);
    return m;
}
__device__ __forceinline__ unsigned map_at(unsigned m, unsigned c) { return (m >> (2 * c)) & 3u; }
__device__ __forceinline__ unsigned map_after(unsigned g, unsigned f) {   // g o f
    return map_at(g, map_at(f, 0)) | (map_at(g, map_at(f, 1)) << 2) |
           (map_at(g, map_at(f, 2)) << 4);
}

// Normalise carries and round to nearest-even, cooperatively: the 32 lanes of one warp call
// it converged with the same s (the accumulator words); every lane returns RN(value).  Exact
// zero -> +0.0, a nonzero ACC_FLAG -> NaN.
//   value = sum_i s_i 2^(32 i - 1074), s_i signed int64, i < ACC_DIGITS.
// Lane l owns digits 3l..3l+2 (96 digits; those >= ACC_DIGITS are 0).  Splitting every word
// into lo (32 bits, unsigned) + hi (signed) leaves u_i = lo_i + hi_(i-1), after which each
// carry is -1, 0 or +1; the carries are resolved by a warp scan of carry maps (composition is
// associative), giving the 96-digit two's-complement value.  Sign = the carry out of the top
// digit; the magnitude's top digit, its two lower neighbours and the sticky OR of the rest
// are found with warp votes and rounded once (round_window).  O(log 32) dependent steps in
// place of a 68-step carry chain on one thread.
__device__ __forceinline__ double acc_finalize_warp(const unsigned long long *s) {
    const unsigned FULL = 0xffffffffu;
    const int lane = (int)(threadIdx.x & 31u);
    if (s[ACC_FLAG] != 0ull) return __longlong_as_double(0x7ff8000000000000ll);
    long long lo[3], hi[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const int i = 3 * lane + k;
        const long long w = i < ACC_DIGITS ? (long long)s[i] : 0ll;
        lo[k] = w & 0xffffffffll;
        hi[k] = w >> 32;                                   // arithmetic: floor(w / 2^32)
    }
    const long long hprev = __shfl_up_sync(FULL, hi[2], 1);
    const long long u[3] = {lo[0] + (lane ? hprev : 0ll), lo[1] + hi[0], lo[2] + hi[1]};
    unsigned G = map_after(carry_map(u[2]), map_after(carry_map(u[1]), carry_map(u[0])));
    // inclusive scan G_l o ... o G_0; a constant map (carry out independent of the carry in:
    // the usual case for every lane) is its own prefix, so the scan is skipped when all are
    const bool cst = map_at(G, 0) == map_at(G, 1) && map_at(G, 1) == map_at(G, 2);
    if (!__all_sync(FULL, cst)) {
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const unsigned prev = __shfl_up_sync(FULL, G, off);
            if (lane >= off) G = map_after(G, prev);
        }
    }
    const unsigned Gex = __shfl_up_sync(FULL, G, 1);
    long long c = lane ? (long long)map_at(Gex, 1) - 1 : 0ll;   // carry into digit 3l
    const bool negative = (int)map_at(__shfl_sync(FULL, G, 31), 1) - 1 < 0;
    uint32_t d[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const long long v = u[k] + c;
        d[k] = (uint32_t)(v & 0xffffffffll);
        c = v >> 32;
    }
    if (negative) {                                        // magnitude = two's complement
        int low = 96;
#pragma unroll
        for (int k = 2; k >= 0; --k)
            if (d[k]) low = 3 * lane + k;
        low = (int)__reduce_min_sync(FULL, (unsigned)low);
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            const int i = 3 * lane + k;
            d[k] = i < low ? 0u : (i == low ? 0u - d[k] : ~d[k]);
        }
    }
    int top = -1;
#pragma unroll
    for (int k = 0; k < 3; ++k)
        if (d[k]) top = 3 * lane + k;
    const int T = (int)__reduce_max_sync(FULL, (unsigned)(top + 1)) - 1;
    if (T < 0) return 0.0;
    uint32_t dw[3];                                        // digits T, T-1, T-2 (0 if < 0)
#pragma unroll
    for (int q = 0; q < 3; ++q) {
        const int idx = T - q;
        const int src = idx >= 0 ? idx / 3 : 0;
        const int k = idx - 3 * lane;
        const uint32_t mine = (idx >= 0 && lane == src) ? (k == 0 ? d[0] : (k == 1 ? d[1] : d[2]))
                                                        : 0u;
        dw[q] = __shfl_sync(FULL, mine, src);
    }
    bool below = false;
#pragma unroll
    for (int k = 0; k < 3; ++k) below |= (3 * lane + k < T - 2) && d[k] != 0u;
    below = __any_sync(FULL, below);
    const double mag = round_window(T, dw[0], dw[1], dw[2], below);
    return negative ? -mag : mag;
}

}  // namespace minife
