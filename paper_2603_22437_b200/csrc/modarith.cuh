// modarith.cuh -- 64-bit modular arithmetic on the integer pipes of sm_100a.
//
// SURVEY §8(a) a2 ("64-bit modular multiply-add"): all primes q < 2^60, so
// lazy values in [0, 4q) fit in 62 bits.  Three products:
//   * Shoup (fixed operand w with w' = floor(w 2^64 / q)): twiddles, base
//     conversion constants, scalar plaintext constants;
//   * Montgomery (R = 2^64, q' = -q^{-1} mod 2^64): variable x variable products
//     (ciphertext x evaluation key, ciphertext x plaintext), operands held in
//     Montgomery form where one side is stored;
//   * 128-bit lazy multiply-accumulate + one Montgomery reduction (base
//     conversion, key inner product, tensor sums).
// No tensor cores: the path is exact 64-bit modular integer work.
#pragma once
#include <cstdint>

namespace mmfhe {

struct U128 {
    uint64_t lo, hi;
};

__device__ __forceinline__ uint64_t mulhi64(uint64_t a, uint64_t b) { return __umul64hi(a, b); }

// a + b*c into a 128-bit accumulator (mad.lo.cc / madc.hi).
__device__ __forceinline__ void mac128(U128 &acc, uint64_t b, uint64_t c)
{
    asm("mad.lo.cc.u64 %0, %2, %3, %0;\n\t"
        "madc.hi.u64 %1, %2, %3, %1;"
        : "+l"(acc.lo), "+l"(acc.hi)
        : "l"(b), "l"(c));
}

__device__ __forceinline__ U128 mul128(uint64_t a, uint64_t b)
{
    U128 r;
    r.lo = a * b;
    r.hi = __umul64hi(a, b);
    return r;
}

__device__ __forceinline__ uint64_t csub(uint64_t a, uint64_t q) { return a >= q ? a - q : a; }

// Reduction of a lazily accumulated x < 2^17 q to [0, q) by an fp32 quotient estimate:
// qinv_est(q) = fl(1/q)(1 - 2^-18), k = floor(x qinv - 2^-14) is floor(x/q) or one less
// (combined relative error of the three roundings and the approximate reciprocal is
// < 2^-21 < the 2^-18 margin), so x - kq lies in [0, 2q) and one subtraction finishes.
__device__ __forceinline__ float qinv_est(uint64_t q) { return __fdividef(1.0f, __ull2float_rn(q)) * (1.0f - 0x1p-18f); }
__device__ __forceinline__ uint64_t reduce_est(uint64_t x, uint64_t q, float qinv)
{
    const float y = fmaxf(__fmaf_rn(__ull2float_rn(x), qinv, -0x1p-14f), 0.0f);
    const uint64_t r = x - (uint64_t)__float2uint_rz(y) * q;
    return r >= q ? r - q : r;
}

__device__ __forceinline__ uint64_t add_mod(uint64_t a, uint64_t b, uint64_t q) { return csub(a + b, q); }
__device__ __forceinline__ uint64_t sub_mod(uint64_t a, uint64_t b, uint64_t q) { return a >= b ? a - b : a + q - b; }

// Shoup product, result in [0, 2q) for any a < 2^64 (w < q).
__device__ __forceinline__ uint64_t shoup_lazy(uint64_t a, uint64_t w, uint64_t wp, uint64_t q)
{
    return a * w - __umul64hi(a, wp) * q;
}
__device__ __forceinline__ uint64_t shoup(uint64_t a, uint64_t w, uint64_t wp, uint64_t q)
{
    return csub(shoup_lazy(a, w, wp, q), q);
}

// Shoup product with a truncated quotient, result in [0, 4q) for any a < 2^64 (w < q).
// With a = ah 2^32 + al and wp = wh 2^32 + wl, a wp / 2^64 = ah wh + (ah wl + al wh) / 2^32
// + al wl / 2^64: dropping al wl and the fractions of the two middle terms leaves an
// integer Q' <= floor(a wp / 2^64) short by at most 2, so a w - Q' q < 2q + 2q.  One
// 32x32->64 and two 32x32->hi32 products replace the four wide products of __umul64hi.
__device__ __forceinline__ uint64_t shoup_lazy4(uint64_t a, uint64_t w, uint64_t wp, uint64_t q)
{
    uint64_t Q;
    asm("{\n\t.reg .u32 al, ah, wl, wh, t1, t2;\n\t.reg .u64 s;\n\t"
        "mov.b64 {al, ah}, %1;\n\tmov.b64 {wl, wh}, %2;\n\t"
        "mul.hi.u32 t1, ah, wl;\n\tmad.hi.cc.u32 t1, al, wh, t1;\n\taddc.u32 t2, 0, 0;\n\t"
        "mov.b64 s, {t1, t2};\n\tmad.wide.u32 %0, ah, wh, s;\n\t}"
        : "=l"(Q)
        : "l"(a), "l"(wp));
    // a w - Q q = a w + Q (2^64 - q) mod 2^64: with -q a (hoisted) operand the two low products chain
    // into one another (IMAD.WIDE accumulate) and no 64-bit negation is issued per butterfly; the asm
    // keeps the compiler from folding it back into a subtraction
    const uint64_t nq = 0 - q;
    uint64_t r;
    asm("mul.lo.u64 %0, %1, %2;\n\tmad.lo.u64 %0, %3, %4, %0;" : "=&l"(r) : "l"(Q), "l"(nq), "l"(a), "l"(w));
    return r;
}

// Montgomery reduction of x = hi*2^64 + lo < q*2^64: returns x*2^-64 mod q in [0, 2q).
__device__ __forceinline__ uint64_t redc_lazy(U128 x, uint64_t q, uint64_t qinv_neg)
{
    uint64_t m = x.lo * qinv_neg;
    return x.hi + __umul64hi(m, q) + (x.lo != 0);
}
__device__ __forceinline__ uint64_t redc(U128 x, uint64_t q, uint64_t qinv_neg) { return csub(redc_lazy(x, q, qinv_neg), q); }

// a*b*2^-64 mod q (canonical), a,b < q (or a*b < q*2^64).
__device__ __forceinline__ uint64_t mont_mul(uint64_t a, uint64_t b, uint64_t q, uint64_t qinv_neg)
{
    return redc(mul128(a, b), q, qinv_neg);
}

// Per-prime constants kept in registers by the kernels.
struct Mod {
    uint64_t q;
    uint64_t qinv_neg;  // -q^{-1} mod 2^64
    uint64_t r2;        // 2^128 mod q  (mont_mul(x, r2) = x*2^64 mod q)
};

} // namespace mmfhe
