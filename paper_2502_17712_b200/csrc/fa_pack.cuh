// fa_pack.cuh — exact integer helpers shared by the packers (fa_pack.cu,
// fa_baselines.cu).  All follow numpy int64 semantics of packing.py.
#pragma once
#include "fa_common.cuh"

// numpy int64 semantics of -((-num * t) // den) (packing.py:349)
__device__ __forceinline__ long long np_ceil_scaled(long long num, long long t, long long den) {
    unsigned long long prod = (0ull - (unsigned long long)num) * (unsigned long long)t;  // wrapping
    long long a = (long long)prod;
    long long q = a / den;
    if ((a % den != 0) && ((a < 0) != (den < 0))) q -= 1;  // floor
    return (long long)(0ull - (unsigned long long)q);
}

// exact ceil(p / d) for 0 <= p < 2^53, 0 < d < 2^53: the round-to-nearest
// float64 quotient truncates to within one of the true floor (quotients are
// < 2^53), fixed by integer remainder checks.  (__ddiv_rn is the hardware-
// assisted division; the directed-rounding variants take a slow path.)
__device__ __forceinline__ long long ceil_div_small(long long p, long long d) {
    long long q = (long long)__ddiv_rn((double)p, (double)d);
    long long r = p - q * d;
    while (r < 0) { q -= 1; r += d; }
    while (r >= d) { q += 1; r -= d; }
    return q + (r != 0);
}

// exact floor(n / d) for n < 2^64, 0 < d < 2^63 with a quotient < 2^52
// (replaces the u64 division routine on the hot path)
__device__ __forceinline__ unsigned long long floor_div_u64_small_q(unsigned long long n, unsigned long long d) {
    unsigned long long q = (unsigned long long)__ddiv_rn((double)n, (double)d);
    long long r = (long long)(n - q * d);  // |r| < 2d: exact as a wrapped difference
    while (r < 0) { q -= 1; r += (long long)d; }
    while (r >= (long long)d) { q += 1; r -= (long long)d; }
    return q;
}

// max(ceil(num*t/den), min_dim) + 2*pad  (packing.py:348-350)
__device__ __forceinline__ long long scaled_dim(long long t, long long num, long long den, long long min_dim,
                                                long long pad) {
    long long s;
    if (num >= 0 && num < (1ll << 26) && t >= 0 && t < (1ll << 26) && den > 0 && den < (1ll << 53))
        s = ceil_div_small(num * t, den);  // num*t < 2^52: same value as the numpy expression
    else
        s = np_ceil_scaled(num, t, den);
    if (s < min_dim) s = min_dim;
    return s + 2 * pad;
}

// scaled_dim with a precomputed rdn = 1.0 / den (round to nearest): the
// estimate num*t*rdn is within 2 of the true quotient for quotients < 2^51,
// and the integer remainder loops make it exact.
__device__ __forceinline__ long long scaled_dim_rcp(long long t, long long num, long long den, double rdn,
                                                    long long min_dim, long long pad) {
    long long s;
    if (num >= 0 && num < (1ll << 26) && t >= 0 && t < (1ll << 26) && den > 0 && den < (1ll << 51)) {
        const long long p = num * t;
        long long q = (long long)((double)p * rdn);
        long long r = p - q * den;
        while (r < 0) { q -= 1; r += den; }
        while (r >= den) { q += 1; r -= den; }
        s = q + (r != 0);
    } else {
        s = np_ceil_scaled(num, t, den);
    }
    if (s < min_dim) s = min_dim;
    return s + 2 * pad;
}

// binary (Stein) gcd: shifts and subtractions, no 64-bit division loop
__device__ __forceinline__ long long gcd_ll(long long a, long long b) {
    unsigned long long u = a < 0 ? 0ull - (unsigned long long)a : (unsigned long long)a;
    unsigned long long v = b < 0 ? 0ull - (unsigned long long)b : (unsigned long long)b;
    if (u == 0) return (long long)v;
    if (v == 0) return (long long)u;
    const int sh = __ffsll((long long)(u | v)) - 1;
    u >>= __ffsll((long long)u) - 1;
    do {
        v >>= __ffsll((long long)v) - 1;
        if (u > v) {
            unsigned long long t = u;
            u = v;
            v = t;
        }
        v -= u;
    } while (v);
    return (long long)(u << sh);
}

// x / g for g = gcd(...) > 0: a shift when g is a power of two (always after
// a dyadic snap), else a 64-bit division
__device__ __forceinline__ long long div_by_gcd(long long x, long long g) {
    if ((g & (g - 1)) == 0) return x >> (__ffsll(g) - 1);
    return x / g;
}
