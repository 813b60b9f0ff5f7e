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
// A consumer kernel normalises the carries and rounds once (acc_finalize).
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

// One window of the digit scan: the top nonzero digit seen so far, the two digits below it,
// and whether anything below those is nonzero.
struct DigitWindow {
    int T = -1;
    uint32_t dT = 0, d1 = 0, d2 = 0;
    bool sticky = false;
    uint32_t prev1 = 0, prev2 = 0;    // digits i-1, i-2 of the scan
    bool below = false;               // OR of digits <= i-3
    __device__ __forceinline__ void push(int i, uint32_t d) {
        if (d != 0) {
            T = i;
            dT = d;
            d1 = prev1;
            d2 = prev2;
            sticky = below;
        }
        below |= prev2 != 0;
        prev2 = prev1;
        prev1 = d;
    }
};

// Normalise carries and round to nearest-even (one thread; s = shared copy of the words).
// Exact zero -> +0.0.  One pass from the least significant digit with constant state:
// the sign is only known at the end, so the window is tracked for both the value and its
// two's-complement negation (digit e_i = -d_i while every lower digit is 0, else ~d_i).
static __device__ __noinline__ double acc_finalize(const unsigned long long *s) {
    if (s[ACC_FLAG] != 0ull) return __longlong_as_double(0x7ff8000000000000ll);
    long long carry = 0;
    bool all_zero = true;
    DigitWindow pos, neg;
#pragma unroll 4
    for (int i = 0; i < ACC_DIGITS; ++i) {
        const long long v = (long long)s[i] + carry;
        const uint32_t d = (uint32_t)((unsigned long long)v & 0xffffffffull);
        carry = (v - (long long)d) >> 32;      // exact floor division by 2^32
        pos.push(i, d);
        neg.push(i, all_zero ? 0u - d : ~d);
        all_zero = all_zero && d == 0;
    }
    const bool negative = carry < 0;           // value = sum d_i 2^(32i) - [neg] 2^(32*68)
    const DigitWindow &w = negative ? neg : pos;
    const int T = w.T;
    if (T < 0) return 0.0;
    const uint32_t dT = w.dT, d1 = w.d1, d2 = w.d2;
    const int t = 32 * T + 31 - __clz(dT);     // top bit, in units of 2^-1074
    double mag;
    if (t <= 52) {                             // T <= 1: the value is digits T..0, exact
        const unsigned long long v =
            T == 1 ? ((unsigned long long)dT << 32) | d1 : (unsigned long long)dT;
        mag = scalbn((double)v, -1074);        // < 2^53 ulps of 2^-1074: exact
    } else {
        // 96-bit window of digits T, T-1, T-2 (missing digits read as 0)
        const unsigned __int128 W = ((unsigned __int128)dT << 64) |
                                    ((unsigned __int128)d1 << 32) | (unsigned __int128)d2;
        const int sh = t - 32 * (T - 2);        // top bit position inside W, in [64, 95]
        unsigned long long M = (unsigned long long)(W >> (sh - 52));   // 53 bits
        const int guard = (int)((W >> (sh - 53)) & 1u);
        bool sticky = w.sticky || (W & ((((unsigned __int128)1) << (sh - 53)) - 1)) != 0;
        int top = t;
        if (guard && (sticky || (M & 1ull))) {
            ++M;
            if (M == (1ull << 53)) {
                M >>= 1;
                ++top;
            }
        }
        mag = scalbn((double)M, top - 52 - 1074);   // inf iff round-to-nearest overflows
    }
    return negative ? -mag : mag;
}

}  // namespace minife
