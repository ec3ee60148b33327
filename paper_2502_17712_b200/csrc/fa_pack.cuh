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

// exact ceil(p / d) for 0 <= p < 2^53, 0 < d < 2^53: a float64 quotient is
// within one of the true floor, fixed by one integer remainder check
__device__ __forceinline__ long long ceil_div_small(long long p, long long d) {
    long long q = (long long)__ddiv_rz((double)p, (double)d);
    long long r = p - q * d;
    if (r < 0) { q -= 1; r += d; }
    else if (r >= d) { q += 1; r -= d; }
    return q + (r != 0);
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

__device__ __forceinline__ long long gcd_ll(long long a, long long b) {
    if (a < 0) a = -a;
    if (b < 0) b = -b;
    while (b) {
        long long t = a % b;
        a = b;
        b = t;
    }
    return a;
}
