// modarith.cuh -- 64-bit RNS modular arithmetic on the integer pipes (sm_100a).
//
// Moduli are odd primes q < 2^60 (the O1 rule gives 40- and 50-bit primes, R1).
//  * Shoup multiplication by a constant w (w' = floor(w 2^64 / q)): any a < 2^64 -> [0, 2q) -> canonical.
//  * Barrett reduction of a 128-bit value x < 2^(2w+2), w = bitlen(q), mu = floor(2^(2w+2) / q):
//      qhat = floor(floor(x / 2^(w-2)) * mu / 2^(w+4)),  x - qhat q in [0, 3q)  (error analysis: DESIGN.md).
// Every kernel output word is canonical in [0, q), which is what makes GPU == oracle bit-exact.
#pragma once
#include <cstdint>

namespace ensi {

struct Barrett {
    uint64_t q;
    uint64_t mu;   // floor(2^(2w+2) / q)
    uint32_t w;    // bit length of q
};

__device__ __forceinline__ uint64_t mulhi64(uint64_t a, uint64_t b) { return __umul64hi(a, b); }

__device__ __forceinline__ uint64_t csub(uint64_t a, uint64_t q) { return a >= q ? a - q : a; }

__device__ __forceinline__ uint64_t add_mod(uint64_t a, uint64_t b, uint64_t q) { return csub(a + b, q); }
__device__ __forceinline__ uint64_t sub_mod(uint64_t a, uint64_t b, uint64_t q) { return csub(a + q - b, q); }

// a * w mod q with w' = floor(w * 2^64 / q); result in [0, q)
__device__ __forceinline__ uint64_t mul_shoup(uint64_t a, uint64_t w, uint64_t wp, uint64_t q) {
    uint64_t hi = mulhi64(a, wp);
    uint64_t r = a * w - hi * q;
    return csub(r, q);
}
// lazy variant, result in [0, 2q)
__device__ __forceinline__ uint64_t mul_shoup_lazy(uint64_t a, uint64_t w, uint64_t wp, uint64_t q) {
    uint64_t hi = mulhi64(a, wp);
    return a * w - hi * q;
}

// 128-bit (hi:lo) mod q, requires hi:lo < 2^(2w+2)
__device__ __forceinline__ uint64_t barrett128(uint64_t hi, uint64_t lo, const Barrett& b) {
    const uint32_t a = b.w - 2;          // 1 <= a <= 58
    const uint32_t s = b.w + 4;          // 36 <= s <= 64
    uint64_t xs = (lo >> a) | (hi << (64 - a));
    uint64_t plo = xs * b.mu;
    uint64_t phi = mulhi64(xs, b.mu);
    uint64_t qhat = (s == 64) ? phi : ((plo >> s) | (phi << (64 - s)));
    uint64_t r = lo - qhat * b.q;
    r = csub(r, b.q);
    return csub(r, b.q);
}
__device__ __forceinline__ uint64_t reduce64(uint64_t x, const Barrett& b) { return barrett128(0, x, b); }

// a * b mod q for a, b < q
__device__ __forceinline__ uint64_t mul_mod(uint64_t a, uint64_t b, const Barrett& br) {
    return barrett128(mulhi64(a, b), a * b, br);
}

// 128-bit accumulate helper
struct U128 {
    uint64_t lo, hi;
};
__device__ __forceinline__ void mac128(U128& acc, uint64_t a, uint64_t b) {
    uint64_t lo = a * b, hi = mulhi64(a, b);
    acc.lo += lo;
    acc.hi += hi + (acc.lo < lo ? 1 : 0);
}

// signed 64-bit accumulator -> canonical [0, q)
__device__ __forceinline__ uint64_t reduce_signed(int64_t v, const Barrett& b) {
    if (v >= 0) return reduce64((uint64_t)v, b);
    uint64_t r = reduce64((uint64_t)(-v), b);
    return r ? b.q - r : 0;
}

__device__ __forceinline__ uint32_t bitrev(uint32_t x, uint32_t bits) { return __brev(x) >> (32 - bits); }

// NTT-domain Galois automorphism: out[k] = in[perm(k)] with 2 brv(perm)+1 == (2 brv(k)+1) g mod 2N'
// (only the product mod 2N' <= 2^18 is needed, so 32-bit arithmetic -- the low bits of a product -- is exact)
__device__ __forceinline__ uint32_t galois_src_index(uint32_t k, uint64_t g, uint32_t log_n) {
    const uint32_t mask = (2u << log_n) - 1;            // mod 2N'
    const uint32_t e = ((2u * bitrev(k, log_n) + 1u) * (uint32_t)g) & mask;
    return bitrev((e - 1) >> 1, log_n);
}

}  // namespace ensi
