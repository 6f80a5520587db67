// poly.cu -- RNS polynomial kernels of the CKKS evaluator (SURVEY §8(a)
// a4-a10, §2.7 CK4-CK10): elementwise add/sub, Montgomery conversion, the
// NTT-domain automorphism, ModUp / ModDown fast base conversion, the key inner
// product, rescale pre/post steps, and fused multi-operand sums (tensor sums,
// plaintext inner products, scalar modular matrix products).
//
// All outputs are canonical residues in [0, q).  Thread mapping: one thread per
// coefficient index (consecutive threads = consecutive words: coalesced
// 256-byte warp accesses), grid.y over limbs/rows, grid.z over batch items;
// per-prime constants are warp-uniform loads (L1 broadcast).
#include <algorithm>
#include <cstdlib>

#include "modarith.cuh"
#include "ops.h"

namespace mmfhe {

namespace {

constexpr int kTB = 256;
// DMAX = 3 instantiations of the digit-templated kernels for dnum = 3 (PS3 / PS4 / PSV)
#ifndef MMFHE_D3
#define MMFHE_D3 1
#endif

__device__ __forceinline__ uint32_t bitrev(uint32_t x, uint32_t log_n) { return __brev(x) >> (32 - log_n); }

// NTT-domain automorphism sigma_g as a gather: (sigma_g a)[j] = a[galois_perm(j)] with
// perm(j) = bitrev(((2 bitrev(j) + 1) g mod 2N - 1) / 2) (slot j holds a(psi^(2 bitrev(j)+1))).
// The top t bits of perm(j) depend only on the top t bits of j, so 32 consecutive j map
// onto one aligned 32-word span: a warp's gather is as coalesced as a plain read, and
// the permutation fuses into any elementwise kernel for the price of the index math.
__device__ __forceinline__ uint32_t galois_perm(uint32_t j, uint32_t g, uint32_t log_n)
{
    if (g == 1) return j;
    const uint32_t ex = ((2u * bitrev(j, log_n) + 1u) * g) & ((2u << log_n) - 1u);
    return bitrev((ex - 1u) >> 1, log_n);
}

inline dim3 grid3(uint32_t n, uint32_t rows, uint32_t batch = 1) { return dim3((n + kTB - 1) / kTB, rows, batch); }

// ------------------------------------------------------------------ elementwise
__global__ void k_addsub(uint64_t *__restrict__ out, const uint64_t *__restrict__ a, const uint64_t *__restrict__ b,
                         KTables kt, PrimeMap pm, int sub)
{
    const uint32_t r = blockIdx.y;
    const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= kt.n) return;
    const uint64_t q = kt.q[pm.idx[r % pm.period]];
    const size_t i = (size_t)r * kt.n + k;
    out[i] = sub ? sub_mod(a[i], b[i], q) : add_mod(a[i], b[i], q);
}

__global__ void k_to_mont(uint64_t *__restrict__ x, KTables kt, PrimeMap pm)
{
    const uint32_t r = blockIdx.y;
    const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= kt.n) return;
    const uint32_t p = pm.idx[r % pm.period];
    const size_t i = (size_t)r * kt.n + k;
    x[i] = mont_mul(x[i], kt.r2[p], kt.q[p], kt.qinv_neg[p]);
}

// sigma_g in the bit-reversed evaluation domain: slot j holds a(psi^(2 br(j) + 1)),
// and sigma_g(a)(psi^e) = a(psi^(e g)).
// ------------------------------------------------------------------ base conversion
struct ModUpDigit {
    const TwPair *hat_inv;
    const uint64_t *hat;
    const uint32_t *tgt;
    size_t y_off;  // words
    uint32_t lo, hi, n_tgt;
};
struct ModUpArgs {
    ModUpDigit d[16];
    size_t xs, ys;  // item strides (words)
    uint32_t level, L;
};

__device__ __forceinline__ uint32_t ext_prime(uint32_t r, uint32_t level, uint32_t L)
{
    return r <= level ? r : L + 1 + (r - level - 1);
}

// y_{j,t} = sum_{i in I_j} [x_i [Qhat_i^{-1}]_{q_i}]_{q_i} [Qhat_i]_t mod t
// AMAX >= digit width (compile-time bound keeps v[] in registers).  The conversion is a
// small modular matrix product (n_tgt x alpha per coefficient) and MAC-bound at PS3/PS4:
// the digit's constants are staged in shared memory once per CTA (broadcast reads) and
// each thread converts kBcK coefficients, so every constant feeds kBcK MAC chains.
#ifndef MMFHE_BCK
#define MMFHE_BCK 2
#endif
constexpr int kBcK = MMFHE_BCK;

template <int AMAX>
__global__ void __launch_bounds__(kTB) k_modup(uint64_t *__restrict__ y_base, const uint64_t *__restrict__ x_base,
                                               KTables kt, ModUpArgs args)
{
    extern __shared__ uint64_t sh[];  // hat [na][n_tgt], then target q and -q^{-1}
    const ModUpDigit &dg = args.d[blockIdx.y];
    const uint32_t na = dg.hi - dg.lo, nt = dg.n_tgt;
    uint64_t *s_hat = sh, *s_q = sh + na * nt, *s_qi = s_q + nt;
    for (uint32_t i = threadIdx.x; i < na * nt; i += blockDim.x) s_hat[i] = dg.hat[i];
    for (uint32_t i = threadIdx.x; i < nt; i += blockDim.x) {
        const uint32_t pt = ext_prime(dg.tgt[i], args.level, args.L);
        s_q[i] = kt.q[pt];
        s_qi[i] = kt.qinv_neg[pt];
    }
    __syncthreads();
    const uint64_t *x = x_base + (size_t)blockIdx.z * args.xs;
    uint64_t *y = y_base + (size_t)blockIdx.z * args.ys + dg.y_off;
    const uint32_t k0 = blockIdx.x * (kBcK * kTB) + threadIdx.x;
    uint64_t v[kBcK][AMAX];
#pragma unroll
    for (int i = 0; i < AMAX; ++i) {
        if (i < (int)na) {
            const uint32_t pi = dg.lo + i;
            const TwPair h = dg.hat_inv[i];
            const uint64_t qp = kt.q[pi];
#pragma unroll
            for (int c = 0; c < kBcK; ++c) {
                const uint32_t k = k0 + c * kTB;
                v[c][i] = k < kt.n ? shoup(x[(size_t)pi * kt.n + k], h.w, h.wp, qp) : 0;
            }
        }
    }
    for (uint32_t ti = 0; ti < nt; ++ti) {
        U128 acc[kBcK];
#pragma unroll
        for (int c = 0; c < kBcK; ++c) acc[c] = U128{0, 0};
#pragma unroll
        for (int i = 0; i < AMAX; ++i)
            if (i < (int)na) {
                const uint64_t hc = s_hat[i * nt + ti];
#pragma unroll
                for (int c = 0; c < kBcK; ++c) mac128(acc[c], v[c][i], hc);
            }
        const uint64_t q = s_q[ti], qi = s_qi[ti];
#pragma unroll
        for (int c = 0; c < kBcK; ++c) {
            const uint32_t k = k0 + c * kTB;
            if (k < kt.n) y[(size_t)ti * kt.n + k] = redc(acc[c], q, qi);
        }
    }
}

struct IPArgs {
    size_t y_off[16];
    uint32_t lo[16], hi[16];
    size_t xs, ys;
    size_t oqs, oqp, ops, opp;  // output item / poly strides of the Q rows (accQ) and P rows (accP)
    uint32_t dnum, level, L, K, B, per_z;
    uint32_t gx, gy;  // sigma_g applied on the fly to the x / y reads (1 = none)
    IPEpi ep;         // fused output epilogue (double hoisting): poly-0 addend, accumulation
};

// The key inner product's output epilogue: poly 0 += the addend (read through sigma_ag; on Q
// rows optionally times [P]_{q_r}: the P lift of a hoisted baby step; on P rows only when the
// addend has them), and with accumulate both polys += the previous output contents.
__device__ __forceinline__ void ip_store(uint64_t *o, size_t opoly, uint64_t v0, uint64_t v1, const IPEpi &e,
                                         size_t b, uint32_t r, uint32_t level, uint32_t n, uint32_t kadd, uint64_t q,
                                         const TwPair *pm)
{
    if (e.add) {
        const bool isq = r <= level;
        if (isq) {
            uint64_t s = e.add[b * e.as + (size_t)r * n + kadd];
            if (pm) s = shoup(s, pm->w, pm->wp, q);
            v0 = add_mod(v0, s, q);
        } else if (e.apbase != ~(size_t)0) {
            v0 = add_mod(v0, e.add[b * e.as + e.apbase + (size_t)(r - level - 1) * n + kadd], q);
        }
    }
    if (e.add1 && r <= level) {  // poly 1's P lift (R31): Q rows only (P = 0 mod p_k)
        uint64_t s = e.add1[b * e.as + (size_t)r * n + kadd];
        if (pm) s = shoup(s, pm->w, pm->wp, q);
        v1 = add_mod(v1, s, q);
    }
    if (e.accumulate) {
        v0 = add_mod(v0, o[0], q);
        v1 = add_mod(v1, o[opoly], q);
    }
    o[0] = v0;
    o[opoly] = v1;
}

// Key inner product (see k_key_ip below for the formula).
// Low-register variant for 5..8 digits: 32-bit in-item source offsets instead of
// per-digit pointers and strides, held to 3 CTAs/SM (78 registers, no spills; the
// pointer version needs 121 and fits 2).  Measured on C2: 9.6 -> 8.9 ms/step.  For
// <= 4 digits the pointer version (k_key_ip, no min-blocks bound) is faster.  Measured and
// not kept: re-reading the key words per item from L2 (64 registers, 4 CTAs/SM: 12% slower
// on C2) and one output pair per thread with 4 items per CTA sharing the key words through
// L1 (C2 5.3 -> 7.3 ms/step, C4 66 -> 99 ms): holding a coefficient's key words in
// registers across the batch items is what makes this kernel cheap.  Also not kept: two
// items per loop iteration (both items' source loads in flight before the MACs) spills
// 396 B at 3 CTAs/SM (C2 5194 -> 5000 frames/s) and at 2 CTAs/SM (no spills) is 0.6%
// slower (5165): the kernel already has enough loads in flight at 3 CTAs/SM.
template <int DMAX, bool EPI = false>
__global__ void __launch_bounds__(kTB, 3) k_key_ip_lr(uint64_t *__restrict__ accQ, uint64_t *__restrict__ accP,
                                                const uint64_t *__restrict__ x, const uint64_t *__restrict__ y,
                                                const uint64_t *__restrict__ key, KTables kt, IPArgs a)
{
    const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= kt.n) return;
    const uint32_t r = blockIdx.y;
    const uint32_t b0 = blockIdx.z * a.per_z, b1 = min(a.B, b0 + a.per_z);
    const uint32_t pr = ext_prime(r, a.level, a.L);
    const uint64_t q = kt.q[pr], qi = kt.qinv_neg[pr];
    const size_t key_rows = a.L + 1 + a.K;
    uint64_t kb[DMAX], ka[DMAX];
    // source of digit j inside an item: x row r (r in I_j) or its ModUp'd row of y; offsets
    // fit 32 bits (T*N <= 2^24), bit j of xm selects x
    uint32_t so[DMAX];
    uint32_t xm = 0;
    const uint32_t kx = galois_perm(k, a.gx, kt.log_n), ky = galois_perm(k, a.gy, kt.log_n);
#pragma unroll
    for (int j = 0; j < DMAX; ++j) {
        if (j < (int)a.dnum) {
            kb[j] = __ldg(key + ((size_t)(2 * j) * key_rows + pr) * kt.n + k);
            ka[j] = __ldg(key + ((size_t)(2 * j + 1) * key_rows + pr) * kt.n + k);
            if (r >= a.lo[j] && r < a.hi[j]) {
                so[j] = r * kt.n + kx;
                xm |= 1u << j;
            } else {
                const uint32_t row = r < a.lo[j] ? r : r - (a.hi[j] - a.lo[j]);
                so[j] = (uint32_t)a.y_off[j] + row * kt.n + ky;
            }
        }
    }
    const bool isq = r <= a.level;
    uint64_t *o = isq ? accQ + (size_t)r * kt.n + k : accP + (size_t)(r - a.level - 1) * kt.n + k;
    const size_t ostride = isq ? a.oqs : a.ops;
    const size_t opoly = isq ? a.oqp : a.opp;
    const uint32_t kadd = EPI && (a.ep.add || a.ep.add1) ? galois_perm(k, a.ep.ag, kt.log_n) : 0;
    const TwPair *pmq = (EPI && a.ep.pmod && isq) ? a.ep.pmod + r : nullptr;
    for (uint32_t b = b0; b < b1; ++b) {
        const uint64_t *xb = x + (size_t)b * a.xs, *yb = y + (size_t)b * a.ys;
        uint64_t s[DMAX];
#pragma unroll
        for (int j = 0; j < DMAX; ++j)
            if (j < (int)a.dnum) s[j] = ((xm >> j) & 1 ? xb : yb)[so[j]];
        U128 acc0{0, 0}, acc1{0, 0};
#pragma unroll
        for (int j = 0; j < DMAX; ++j) {
            if (j < (int)a.dnum) {
                mac128(acc0, s[j], kb[j]);
                mac128(acc1, s[j], ka[j]);
            }
        }
        if (EPI) {
            ip_store(o + (size_t)b * ostride, opoly, redc(acc0, q, qi), redc(acc1, q, qi), a.ep, b, r, a.level, kt.n,
                     kadd, q, pmq);
        } else {
            o[(size_t)b * ostride] = redc(acc0, q, qi);
            o[(size_t)b * ostride + opoly] = redc(acc1, q, qi);
        }
    }
}

// For every batch item b: (accQ|accP)_{b,p}[r] = sum_j src_{b,j}[r] (.) evk_j[p][r] with
// src = x_b[r] for r in I_j, else the ModUp'd row.  The 2*dnum key words of (r, k) are
// loaded once per thread and reused for its per_z items (grid.z splits the batch).
// dnum = 3: 5 CTAs/SM (48 registers, 8-28 B of spills outside the item loop): C4 key_ip
// 2.78 -> 2.55 ms against 4 CTAs/SM (62 registers; ncu long_scoreboard 0.76), r02cc
#ifndef MMFHE_KIP3_MINB
#define MMFHE_KIP3_MINB 5
#endif
template <int DMAX, bool EPI = false>
__global__ void __launch_bounds__(kTB, DMAX == 3 ? MMFHE_KIP3_MINB : DMAX <= 4 ? 4 : 1) k_key_ip(uint64_t *__restrict__ accQ, uint64_t *__restrict__ accP,
                                                const uint64_t *__restrict__ x, const uint64_t *__restrict__ y,
                                                const uint64_t *__restrict__ key, KTables kt, IPArgs a)
{
    const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= kt.n) return;
    const uint32_t r = blockIdx.y;
    const uint32_t b0 = blockIdx.z * a.per_z, b1 = min(a.B, b0 + a.per_z);
    const uint32_t pr = ext_prime(r, a.level, a.L);
    const uint64_t q = kt.q[pr], qi = kt.qinv_neg[pr];
    const size_t key_rows = a.L + 1 + a.K;
    uint64_t kb[DMAX], ka[DMAX];
    const uint64_t *src[DMAX];
    size_t sstr[DMAX];
    const uint32_t kx = galois_perm(k, a.gx, kt.log_n), ky = galois_perm(k, a.gy, kt.log_n);
#pragma unroll
    for (int j = 0; j < DMAX; ++j) {
        if (j < (int)a.dnum) {
            kb[j] = __ldg(key + ((size_t)(2 * j) * key_rows + pr) * kt.n + k);
            ka[j] = __ldg(key + ((size_t)(2 * j + 1) * key_rows + pr) * kt.n + k);
            if (r >= a.lo[j] && r < a.hi[j]) {
                src[j] = x + (size_t)r * kt.n + kx;
                sstr[j] = a.xs;
            } else {
                const uint32_t row = r < a.lo[j] ? r : r - (a.hi[j] - a.lo[j]);
                src[j] = y + a.y_off[j] + (size_t)row * kt.n + ky;
                sstr[j] = a.ys;
            }
        }
    }
    const bool isq = r <= a.level;
    uint64_t *o = isq ? accQ + (size_t)r * kt.n + k : accP + (size_t)(r - a.level - 1) * kt.n + k;
    const size_t ostride = isq ? a.oqs : a.ops;
    const size_t opoly = isq ? a.oqp : a.opp;
    const uint32_t kadd = EPI && (a.ep.add || a.ep.add1) ? galois_perm(k, a.ep.ag, kt.log_n) : 0;
    const TwPair *pmq = (EPI && a.ep.pmod && isq) ? a.ep.pmod + r : nullptr;
    // (a software-pipelined variant loading item b+1's digit words during item b's MACs measured
    // slower on C4: 72 registers, 3 CTAs/SM, 9.96 -> 10.44 ms/step; so did two items per
    // iteration with both items' loads issued first (32-bit offsets, 62 / 80 registers): C4
    // key_ip 2.86 -> 3.17 ms, 3.46 with the epilogue instantiation at 4 CTAs/SM, r02bo)
    for (uint32_t b = b0; b < b1; ++b) {
        uint64_t s[DMAX];
#pragma unroll
        for (int j = 0; j < DMAX; ++j)
            if (j < (int)a.dnum) s[j] = src[j][(size_t)b * sstr[j]];
        U128 acc0{0, 0}, acc1{0, 0};
#pragma unroll
        for (int j = 0; j < DMAX; ++j) {
            if (j < (int)a.dnum) {
                mac128(acc0, s[j], kb[j]);
                mac128(acc1, s[j], ka[j]);
            }
        }
        if (EPI) {
            ip_store(o + (size_t)b * ostride, opoly, redc(acc0, q, qi), redc(acc1, q, qi), a.ep, b, r, a.level, kt.n,
                     kadd, q, pmq);
        } else {
            o[(size_t)b * ostride] = redc(acc0, q, qi);
            o[(size_t)b * ostride + opoly] = redc(acc1, q, qi);
        }
    }
}

// A group of hoisted rotations left over Q_l u P (double hoisting's baby steps, R22/R27) in one
// launch: for every step s, item b, PQ row r and coefficient j
//   r_s[j] = sum_d y_d[perm_s(j)] evk_s[d][j] (+ [P]_{q_r} c0[perm_s(j)] on poly 0's Q rows).
// A thread owns the source index k = perm_s(j) instead: y_d[k] and c0[k] are the same for every
// step, so the CTA stages its tile of them for all B items in shared memory once, then walks
// the steps: each step's 2 dnum key words are gathered at j = perm_s^{-1}(k) (an aligned
// 32-word span maps onto one aligned span: the gathers stay coalesced), reused across the B
// items, and the results are scattered to j.  y, x and c0 are read from HBM once for the whole
// group instead of once per step; every key word once per launch.
constexpr int kHTile = 128;
struct HoistIPArgs {
    const uint64_t *key[kDiagMax];
    uint64_t *out[kDiagMax];      // PQ ciphertexts: [B][2][l+1] Q rows, then [B][2][K] P rows
    uint32_t ginv[kDiagMax];      // inverse Galois elements (perm_s^{-1})
    size_t y_off[16];
    uint32_t lo[16], hi[16];
    size_t xs, ys, cs, os;        // item strides: x (c1), y (ModUp'd digits), c0, outputs
    uint32_t dnum, level, L, K, B, nsteps;
};

template <int DMAX>
__global__ void __launch_bounds__(kHTile) k_hoisted_ip_pq(const uint64_t *__restrict__ x, const uint64_t *__restrict__ y,
                                                        const uint64_t *__restrict__ c0, const TwPair *__restrict__ pmod,
                                                        KTables kt, HoistIPArgs a)
{
    extern __shared__ uint64_t sh[];  // [B][dnum][kHTile] digit words, then [B][kHTile] c0 (Q rows)
    const uint32_t r = blockIdx.y;    // PQ row: 0..l = q_r, l+1.. = p_{r-l-1}
    const uint32_t k0 = blockIdx.x * kHTile, t = threadIdx.x, k = k0 + t;
    const bool isq = r <= a.level;
    const uint32_t pr = ext_prime(r, a.level, a.L);
    const uint64_t q = kt.q[pr], qi = kt.qinv_neg[pr];
    uint64_t *sy = sh, *sc = sh + (size_t)a.B * a.dnum * kHTile;
    for (uint32_t b = 0; b < a.B; ++b) {
        for (uint32_t j = 0; j < a.dnum; ++j) {
            const uint64_t *src;
            if (r >= a.lo[j] && r < a.hi[j]) {
                src = x + (size_t)b * a.xs + (size_t)r * kt.n;
            } else {
                const uint32_t row = r < a.lo[j] ? r : r - (a.hi[j] - a.lo[j]);
                src = y + (size_t)b * a.ys + a.y_off[j] + (size_t)row * kt.n;
            }
            sy[((size_t)b * a.dnum + j) * kHTile + t] = src[k];
        }
        // [P]_r c0[k]: the same P lift for every step (the steps differ only in where it lands)
        if (isq)
            sc[(size_t)b * kHTile + t] = shoup(c0[(size_t)b * a.cs + (size_t)r * kt.n + k], pmod[r].w, pmod[r].wp, q);
    }
    __syncthreads();
    const size_t key_rows = a.L + 1 + a.K;
    const size_t qrow = isq ? (size_t)r * kt.n : 0;
    const size_t prow = isq ? 0 : (size_t)(2 * (a.level + 1) + (r - a.level - 1)) * kt.n;
    const size_t opoly = isq ? (size_t)(a.level + 1) * kt.n : (size_t)a.K * kt.n;
    // the next step's key words are loaded while this step's items are computed
    uint64_t nkb[DMAX], nka[DMAX];
    uint32_t nj = galois_perm(k, a.ginv[0], kt.log_n);
#pragma unroll
    for (int d = 0; d < DMAX; ++d) {
        if (d < (int)a.dnum) {
            nkb[d] = __ldg(a.key[0] + ((size_t)(2 * d) * key_rows + pr) * kt.n + nj);
            nka[d] = __ldg(a.key[0] + ((size_t)(2 * d + 1) * key_rows + pr) * kt.n + nj);
        }
    }
    for (uint32_t s = 0; s < a.nsteps; ++s) {
        const uint32_t j = nj;
        uint64_t kb[DMAX], ka[DMAX];
#pragma unroll
        for (int d = 0; d < DMAX; ++d) {
            kb[d] = nkb[d];
            ka[d] = nka[d];
        }
        if (s + 1 < a.nsteps) {
            nj = galois_perm(k, a.ginv[s + 1], kt.log_n);
#pragma unroll
            for (int d = 0; d < DMAX; ++d) {
                if (d < (int)a.dnum) {
                    nkb[d] = __ldg(a.key[s + 1] + ((size_t)(2 * d) * key_rows + pr) * kt.n + nj);
                    nka[d] = __ldg(a.key[s + 1] + ((size_t)(2 * d + 1) * key_rows + pr) * kt.n + nj);
                }
            }
        }
        uint64_t *o = a.out[s] + (isq ? qrow : prow) + j;
        for (uint32_t b = 0; b < a.B; ++b) {
            U128 acc0{0, 0}, acc1{0, 0};
            const uint64_t *v = sy + (size_t)b * a.dnum * kHTile + t;
#pragma unroll
            for (int d = 0; d < DMAX; ++d) {
                if (d < (int)a.dnum) {
                    const uint64_t w = v[d * kHTile];
                    mac128(acc0, w, kb[d]);
                    mac128(acc1, w, ka[d]);
                }
            }
            uint64_t v0 = redc(acc0, q, qi);
            if (isq) v0 = add_mod(v0, sc[(size_t)b * kHTile + t], q);
            o[(size_t)b * a.os] = v0;
            o[(size_t)b * a.os + opoly] = redc(acc1, q, qi);
        }
    }
}

// Double hoisting's first rotate-and-sum level (R27) in ONE pass: for every item b, PQ row r and
// coefficient j, the sum of the lift and of every hoisted PQ step s,
//   acc_0[j] = [P]_r c0[j] + sum_s ( IP_s,0[j] + [P]_r c0[perm_s(j)] ),   acc_1[j] = [P]_r c1[j] + sum_s IP_s,1[j]
// with IP_s,p[j] = sum_d src_d[perm_s(j)] evk_s[d][p][j] (Q rows: [P]_r terms; P rows: the inner products
// only) -- the oracle's lift_pq + hoisted_step_pq + add_pq chain (rotsum_dh_all), whose modular sum is exact
// in any order.  The thread owns the OUTPUT index j and gathers the sources at perm_s(j) (an aligned
// 32-word span maps onto an aligned span: the gathers stay coalesced, and a row's sources stay L2-resident
// across its CTAs), so the steps accumulate in registers and only the sum reaches HBM: no per-step PQ
// outputs and no PQ additions.  Steps outer, items inner: each step's 2 dnum key words are loaded once
// into registers and reused for the CTA's chunk of up to RB items (grid.z splits larger batches), whose
// running sums stay in the thread's own shared-memory column (16 KiB-per-item-chunk: no barriers), so the
// group may have any number of steps and occupancy is not bound by a key tile.
constexpr int kRTile = 128;
constexpr int kRItems = 16;  // items per CTA (running sums in shared memory)
constexpr int kRSteps = 64;  // steps per launch (kernel-parameter arrays)
struct HoistSumArgs {
    const uint64_t *key[kRSteps];
    uint32_t g[kRSteps];  // Galois elements (perm_s)
    size_t y_off[16];
    uint32_t lo[16], hi[16];
    size_t xs, ys, cs, os;  // item strides: x (c1), y (ModUp'd digits), c0, output
    uint32_t dnum, level, L, K, B, nsteps;
};

#ifndef MMFHE_RS_MINB
#define MMFHE_RS_MINB 4  // measured: 4 (123 regs) 4.18 ms, 1 (128 regs) 5.98, 5 (96) 4.69, 6 (80) 5.34 (C4 K2b + FC)
#endif
// dnum = 3 (DMAX = 3): 5 CTAs/SM with 4 steps per 128-bit sum (96 registers, no spills): C4's
// rotate-and-sums 3.97 -> 3.85 ms against 4 CTAs/SM with 5 steps (r02bx; 6 CTAs/SM with 3 steps 3.91)
template <int DMAX>
__global__ void __launch_bounds__(kRTile, DMAX == 3 ? 5 : MMFHE_RS_MINB) k_hoisted_rotsum_pq(uint64_t *__restrict__ out, const uint64_t *__restrict__ x,
                                                            const uint64_t *__restrict__ y,
                                                            const uint64_t *__restrict__ c0,
                                                            const TwPair *__restrict__ pmod, KTables kt,
                                                            HoistSumArgs a)
{
    __shared__ uint64_t sacc[kRItems][2][kRTile];  // this thread's column: the chunk's running sums
    const uint32_t r = blockIdx.y, t = threadIdx.x, j = blockIdx.x * kRTile + t;
    const uint32_t b0 = blockIdx.z * kRItems, nb = min((uint32_t)kRItems, a.B - b0);
    const bool isq = r <= a.level;
    const uint32_t pr = ext_prime(r, a.level, a.L);
    const uint64_t q = kt.q[pr], qi = kt.qinv_neg[pr];
    const size_t key_rows = a.L + 1 + a.K;
    // digit d's source row: x row r (r in I_d) or its ModUp'd row of y (item b0 onwards)
    const uint64_t *src[DMAX];
    size_t sst[DMAX];
#pragma unroll
    for (int d = 0; d < DMAX; ++d) {
        if (d < (int)a.dnum) {
            if (r >= a.lo[d] && r < a.hi[d]) {
                src[d] = x + (size_t)b0 * a.xs + (size_t)r * kt.n;
                sst[d] = a.xs;
            } else {
                const uint32_t row = r < a.lo[d] ? r : r - (a.hi[d] - a.lo[d]);
                src[d] = y + (size_t)b0 * a.ys + a.y_off[d] + (size_t)row * kt.n;
                sst[d] = a.ys;
            }
        }
    }
    const uint64_t *c0r = c0 + (size_t)b0 * a.cs + (size_t)r * kt.n;
    const TwPair pm = isq ? pmod[r] : TwPair{0, 0};
    for (uint32_t b = 0; b < nb; ++b) {
        uint64_t v0 = 0, v1 = 0;
        if (isq) {
            v0 = shoup(c0r[(size_t)b * a.cs + j], pm.w, pm.wp, q);
            v1 = shoup(x[(size_t)(b0 + b) * a.xs + (size_t)r * kt.n + j], pm.w, pm.wp, q);
        }
        sacc[b][0][t] = v0;
        sacc[b][1][t] = v1;
    }
    // steps in chunks of kRChunk: the chunk's key words and source indices in registers, then per item
    // the chunk's products summed in 128 bits (<= 16 terms < q^2 each: < q 2^64 for q < 2^60) and its c0 words summed before ONE Shoup product by [P]_r (P times a sum
    // = the sum of the P multiples): one Montgomery reduction per poly per chunk instead of per step
#ifndef MMFHE_RS_TERMS
#define MMFHE_RS_TERMS 16
#endif
    static_assert(MMFHE_RS_TERMS <= 16, "128-bit accumulation bound: <= 16 products < q^2, q < 2^60");
    constexpr int kRTerms = DMAX == 3 ? 12 : MMFHE_RS_TERMS;
    constexpr int kRChunk = kRTerms / DMAX > 0 ? kRTerms / DMAX : 1;  // steps per 128-bit sum
    for (uint32_t s0 = 0; s0 < a.nsteps; s0 += kRChunk) {
        const uint32_t ns = min((uint32_t)kRChunk, a.nsteps - s0);
        uint64_t kb[kRChunk][DMAX], ka[kRChunk][DMAX];
        uint32_t kk[kRChunk];
#pragma unroll
        for (int u = 0; u < kRChunk; ++u) {
            kk[u] = 0;
            if (u < (int)ns) {
                const uint64_t *ks = a.key[s0 + u] + (size_t)pr * kt.n + j;
#pragma unroll
                for (int d = 0; d < DMAX; ++d) {
                    if (d < (int)a.dnum) {
                        kb[u][d] = __ldg(ks + (size_t)(2 * d) * key_rows * kt.n);
                        ka[u][d] = __ldg(ks + (size_t)(2 * d + 1) * key_rows * kt.n);
                    }
                }
                kk[u] = galois_perm(j, a.g[s0 + u], kt.log_n);
            }
        }
        for (uint32_t b = 0; b < nb; ++b) {
            U128 p0{0, 0}, p1{0, 0};
            uint64_t csum = 0;  // < kRChunk q
#pragma unroll
            for (int u = 0; u < kRChunk; ++u) {
                if (u < (int)ns) {
                    uint64_t w[DMAX];
#pragma unroll
                    for (int d = 0; d < DMAX; ++d)
                        if (d < (int)a.dnum) w[d] = src[d][(size_t)b * sst[d] + kk[u]];
                    if (isq) csum += c0r[(size_t)b * a.cs + kk[u]];
#pragma unroll
                    for (int d = 0; d < DMAX; ++d) {
                        if (d < (int)a.dnum) {
                            mac128(p0, w[d], kb[u][d]);
                            mac128(p1, w[d], ka[u][d]);
                        }
                    }
                }
            }
            uint64_t v0 = add_mod(sacc[b][0][t], redc(p0, q, qi), q);
            if (isq) v0 = add_mod(v0, shoup(csum, pm.w, pm.wp, q), q);
            sacc[b][0][t] = v0;
            sacc[b][1][t] = add_mod(sacc[b][1][t], redc(p1, q, qi), q);
        }
    }
    const size_t orow = isq ? (size_t)r * kt.n : (size_t)(2 * (a.level + 1) + (r - a.level - 1)) * kt.n;
    const size_t opoly = isq ? (size_t)(a.level + 1) * kt.n : (size_t)a.K * kt.n;
    for (uint32_t b = 0; b < nb; ++b) {
        uint64_t *o = out + (size_t)(b0 + b) * a.os + orow + j;
        o[0] = sacc[b][0][t];
        o[opoly] = sacc[b][1][t];
    }
}

struct MDArgs {
    const TwPair *phat_inv;  // [ns] [(S/s_k)^{-1}]_{s_k} of the sources
    const uint64_t *phat;    // [ns][L+1] [S/s_k]_{q_i} Montgomery
    const TwPair *pinv;      // [L+1]
    const uint64_t *zq;      // R31: the q_level rows [B*npoly][N] as an extra source (S = P q_l), or null
    uint32_t level, L, K;
};

// w_i = sum_k [z_k [Phat_k^{-1}]_{p_k}]_{p_k} [Phat_k]_{q_i} mod q_i; grid.y = item*2 + poly.
// Same structure as k_modup: constants in shared memory, kBcK coefficients per thread.
template <int KMAX>
__global__ void __launch_bounds__(kTB) k_moddown_bconv(uint64_t *__restrict__ w, const uint64_t *__restrict__ zP,
                                                       KTables kt, MDArgs a)
{
    extern __shared__ uint64_t sh[];  // phat [ns][targets], then q_i and -q_i^{-1}
    // sources: p_0..p_{K-1} (zP), plus q_level (zq) for the merged ModDown + rescale (R31), whose
    // targets are q_0..q_{level-1}
    const uint32_t ns = a.K + (a.zq ? 1u : 0u);
    const uint32_t L1 = a.zq ? a.level : a.level + 1;
    uint64_t *s_hat = sh, *s_q = sh + ns * L1, *s_qi = s_q + L1;
    for (uint32_t t = threadIdx.x; t < ns * L1; t += blockDim.x)
        s_hat[t] = a.phat[(size_t)(t / L1) * (a.L + 1) + t % L1];
    for (uint32_t i = threadIdx.x; i < L1; i += blockDim.x) {
        s_q[i] = kt.q[i];
        s_qi[i] = kt.qinv_neg[i];
    }
    __syncthreads();
    const uint32_t ip = blockIdx.y;  // item * 2 + poly
    const uint32_t k0 = blockIdx.x * (kBcK * kTB) + threadIdx.x;
    uint64_t v[kBcK][KMAX];
#pragma unroll
    for (int kk = 0; kk < KMAX; ++kk) {
        if (kk < (int)ns) {
            const bool pk = kk < (int)a.K;
            const uint32_t pi = pk ? a.L + 1 + kk : a.level;
            const TwPair h = a.phat_inv[kk];
            const uint64_t qp = kt.q[pi];
            const uint64_t *row = pk ? zP + ((size_t)ip * a.K + kk) * kt.n : a.zq + (size_t)ip * kt.n;
#pragma unroll
            for (int c = 0; c < kBcK; ++c) {
                const uint32_t k = k0 + c * kTB;
                v[c][kk] = k < kt.n ? shoup(row[k], h.w, h.wp, qp) : 0;
            }
        }
    }
    for (uint32_t i = 0; i < L1; ++i) {
        U128 acc[kBcK];
#pragma unroll
        for (int c = 0; c < kBcK; ++c) acc[c] = U128{0, 0};
#pragma unroll
        for (int kk = 0; kk < KMAX; ++kk)
            if (kk < (int)ns) {
                const uint64_t hc = s_hat[kk * L1 + i];
#pragma unroll
                for (int c = 0; c < kBcK; ++c) mac128(acc[c], v[c][kk], hc);
            }
        const uint64_t q = s_q[i], qi = s_qi[i];
#pragma unroll
        for (int c = 0; c < kBcK; ++c) {
            const uint32_t k = k0 + c * kTB;
            if (k < kt.n) w[((size_t)ip * L1 + i) * kt.n + k] = redc(acc[c], q, qi);
        }
    }
}

// One pair (the common case: squarings, K7 products): d0 = a0 b0, d1 = a0 b1 + a1 b0,
// d2 = a1 b1.  The two a-inputs are taken to Montgomery form once (a R = mont(a, R^2))
// so each output is a single REDC of a product sum (two corrections instead of three
// output fix-ups), and each thread handles two coefficients to keep more loads in flight.
__global__ void __launch_bounds__(kTB) k_tensor1(uint64_t *__restrict__ out_base, size_t os,
                                                 const uint64_t *__restrict__ A, const uint64_t *__restrict__ Bp,
                                                 size_t is, KTables kt, uint32_t level, int accumulate)
{
    const uint32_t r = blockIdx.y;
    const size_t boff = (size_t)blockIdx.z * is;
    uint64_t *out = out_base + (size_t)blockIdx.z * os;
    const uint64_t q = kt.q[r], qi = kt.qinv_neg[r], r2 = kt.r2[r];
    const size_t ps = (size_t)(level + 1) * kt.n;
    const uint32_t k0 = blockIdx.x * (2 * kTB) + threadIdx.x;
    uint64_t a0[2], a1[2], b0[2], b1[2];
#pragma unroll
    for (int c = 0; c < 2; ++c) {
        const uint32_t k = min(k0 + c * kTB, kt.n - 1);
        const size_t off = boff + (size_t)r * kt.n + k;
        a0[c] = A[off];
        a1[c] = A[ps + off];
        b0[c] = Bp[off];
        b1[c] = Bp[ps + off];
    }
#pragma unroll
    for (int c = 0; c < 2; ++c) {
        const uint32_t k = k0 + c * kTB;
        if (k >= kt.n) break;
        const uint64_t x0 = mont_mul(a0[c], r2, q, qi), x1 = mont_mul(a1[c], r2, q, qi);
        U128 m1 = mul128(x0, b1[c]);
        const U128 m2 = mul128(x1, b0[c]);
        m1.lo += m2.lo;
        m1.hi += m2.hi + (m1.lo < m2.lo);
        uint64_t d0 = redc(mul128(x0, b0[c]), q, qi), d1 = redc(m1, q, qi), d2 = redc(mul128(x1, b1[c]), q, qi);
        const size_t off = (size_t)r * kt.n + k;
        if (accumulate) {
            d0 = add_mod(d0, out[off], q);
            d1 = add_mod(d1, out[ps + off], q);
            d2 = add_mod(d2, out[2 * ps + off], q);
        }
        out[off] = d0;
        out[ps + off] = d1;
        out[2 * ps + off] = d2;
    }
}

// (ModDown's and the rescale's final steps are the forward NTT row pass's epilogue, RowEpi)

// ------------------------------------------------------------------ fused sums
// d0 = sum a0 b0, d1 = sum a0 b1 + a1 b0, d2 = sum a1 b1 over n pairs; grid.z = item.
// DESIGN R32: the terms of d (x) s(d), s = sigma_g a permutation of the NTT domain (g = 2N - 1: the
// conjugation): t0 = d0 s(d0), t1 = d1 s(d0) into the 2-poly batch t01, t2 = d0 s(d1) into t2 and
// t3 = d1 s(d1) into t3 (single polys); grid (n / kTB, level + 1, B)
__global__ void __launch_bounds__(kTB) k_conj_tensor(uint64_t *__restrict__ t01, size_t t01s, uint64_t *__restrict__ t2,
                                                     uint64_t *__restrict__ t3, size_t t23s,
                                                     const uint64_t *__restrict__ d, size_t ds, KTables kt,
                                                     uint32_t level, uint32_t g)
{
    const uint32_t r = blockIdx.y, b = blockIdx.z;
    const uint32_t j = blockIdx.x * kTB + threadIdx.x;
    if (j >= kt.n) return;
    const uint64_t q = kt.q[r], qi = kt.qinv_neg[r], r2 = kt.r2[r];
    const size_t ps = (size_t)(level + 1) * kt.n;
    const uint64_t *d0 = d + (size_t)b * ds + (size_t)r * kt.n, *d1 = d0 + ps;
    const uint32_t pj = galois_perm(j, g, kt.log_n);
    const uint64_t x0 = mont_mul(d0[j], r2, q, qi), x1 = mont_mul(d1[j], r2, q, qi);
    const uint64_t s0 = d0[pj], s1 = d1[pj];
    const size_t o = (size_t)r * kt.n + j;
    t01[(size_t)b * t01s + o] = redc(mul128(x0, s0), q, qi);
    t01[(size_t)b * t01s + ps + o] = redc(mul128(x1, s0), q, qi);
    t2[(size_t)b * t23s + o] = redc(mul128(x0, s1), q, qi);
    t3[(size_t)b * t23s + o] = redc(mul128(x1, s1), q, qi);
}

__global__ void __launch_bounds__(kTB) k_tensor_sum(uint64_t *__restrict__ out_base, size_t os, PtrList A, PtrList B,
                                                    size_t is, int n, KTables kt, uint32_t level, int accumulate)
{
    const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= kt.n) return;
    const uint32_t r = blockIdx.y;
    const size_t boff = (size_t)blockIdx.z * is;
    uint64_t *out = out_base + (size_t)blockIdx.z * os;
    const uint64_t q = kt.q[r], qi = kt.qinv_neg[r];
    const size_t ps = (size_t)(level + 1) * kt.n;
    const size_t off = (size_t)r * kt.n + k;
    uint64_t s0 = 0, s1 = 0, s2 = 0;
    int p = 0;
    while (p < n) {
        U128 a0c{0, 0}, a1c{0, 0}, a2c{0, 0};
        const int end = min(n, p + 7);  // <= 14 products < q*2^60 each in acc1
        for (; p < end; ++p) {
            const uint64_t *pa = A.p[p] + boff, *pb = B.p[p] + boff;
            const uint64_t a0 = pa[off], a1 = pa[ps + off];
            if (pa == pb) {
                mac128(a0c, a0, a0);
                const U128 m = mul128(a0, a1);
                mac128(a1c, a0, a1);
                a1c.lo += m.lo;
                a1c.hi += m.hi + (a1c.lo < m.lo);
                mac128(a2c, a1, a1);
            } else {
                const uint64_t b0 = pb[off], b1 = pb[ps + off];
                mac128(a0c, a0, b0);
                mac128(a1c, a0, b1);
                mac128(a1c, a1, b0);
                mac128(a2c, a1, b1);
            }
        }
        s0 = add_mod(s0, redc(a0c, q, qi), q);
        s1 = add_mod(s1, redc(a1c, q, qi), q);
        s2 = add_mod(s2, redc(a2c, q, qi), q);
    }
    const uint64_t r2 = kt.r2[r];
    uint64_t d0 = mont_mul(s0, r2, q, qi), d1 = mont_mul(s1, r2, q, qi), d2 = mont_mul(s2, r2, q, qi);
    if (accumulate) {
        d0 = add_mod(d0, out[off], q);
        d1 = add_mod(d1, out[ps + off], q);
        d2 = add_mod(d2, out[2 * ps + off], q);
    }
    out[off] = d0;
    out[ps + off] = d1;
    out[2 * ps + off] = d2;
}

// out_p = sum_t ct_t[p] (.) pt_t, pt in Montgomery form shared by the batch.
__global__ void __launch_bounds__(kTB) k_pmult_sum(uint64_t *__restrict__ out_base, size_t os, PtrList PT,
                                                   PtrList CT, size_t is, int n, KTables kt, uint32_t level,
                                                   int accumulate)
{
    const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= kt.n) return;
    const uint32_t r = blockIdx.y;
    const size_t boff = (size_t)blockIdx.z * is;
    uint64_t *out = out_base + (size_t)blockIdx.z * os;
    const uint64_t q = kt.q[r], qi = kt.qinv_neg[r];
    const size_t ps = (size_t)(level + 1) * kt.n;
    const size_t off = (size_t)r * kt.n + k;
    uint64_t s0 = 0, s1 = 0;
    int t = 0;
    while (t < n) {
        U128 c0{0, 0}, c1{0, 0};
        const int end = min(n, t + 15);
        for (; t < end; ++t) {
            const uint64_t w = __ldg(PT.p[t] + off);
            const uint64_t *c = CT.p[t] + boff;
            mac128(c0, c[off], w);
            mac128(c1, c[ps + off], w);
        }
        s0 = add_mod(s0, redc(c0, q, qi), q);
        s1 = add_mod(s1, redc(c1, q, qi), q);
    }
    if (accumulate) {
        s0 = add_mod(s0, out[off], q);
        s1 = add_mod(s1, out[ps + off], q);
    }
    out[off] = s0;
    out[ps + off] = s1;
}

// BSGS inner sums of all giant steps in one pass, plaintext-stationary:
//   out_o = sum_c pt[o][c] (.) ct_c   (pt[o][c] == nullptr: no term)
// for every item of a batch.  A CTA owns kDmTK = 32 coefficients of one residue row: it stages
// that tile's word of every (o, c) plaintext in shared memory once (the plaintexts are read
// from HBM once per launch, not once per item), then its warps walk the batch items: each
// lane loads its coefficient of the nc baby steps into registers and produces all no outputs
// (nc 64x64->128 MACs from shared memory + one Montgomery reduction each).  Rows of PQ
// operands (double hoisting: pk = K extra limbs) map to the special primes.
constexpr int kDmTK = 32;
struct DiagMacArgs {
    const uint64_t *ct[kDiagIn];
    const uint64_t *pt[kDiagMax][kDiagIn];
    uint64_t *out[kDiagMax];
    size_t is, os;
    int nc, no;
    uint32_t level, L, pk, B;
};

template <int NCMAX>
__global__ void __launch_bounds__(128) k_diag_mac(DiagMacArgs a, KTables kt)
{
    extern __shared__ uint64_t spt[];  // [no][nc][kDmTK]
    const uint32_t L1 = a.level + 1;
    const uint32_t pr = blockIdx.y;  // residue row of the basis: q_0..q_l, then p_0..p_{pk-1}
    const uint32_t prime = pr < L1 ? pr : a.L + 1 + (pr - L1);
    const uint32_t k0 = blockIdx.x * kDmTK;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const int nt = a.no * a.nc;
    for (int t0 = warp * 4; t0 < nt; t0 += nw * 4) {  // four 256-byte rows in flight per warp
        uint64_t v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int t = t0 + u;
            const uint64_t *p = t < nt ? a.pt[t / a.nc][t % a.nc] : nullptr;
            v[u] = p ? __ldg(p + (size_t)pr * kt.n + k0 + lane) : 0;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u)
            if (t0 + u < nt) spt[(t0 + u) * kDmTK + lane] = v[u];
    }
    __syncthreads();
    const uint64_t q = kt.q[prime], qi = kt.qinv_neg[prime];
    // item rows: Q part [2][L1] then P part [2][pk]; this CTA's two rows (poly 0 / 1)
    const size_t r0 = pr < L1 ? pr : 2 * L1 + (pr - L1);
    const size_t pstride = pr < L1 ? L1 : a.pk;
    for (uint32_t u = warp; u < 2 * a.B; u += nw) {
        const uint32_t b = u >> 1, poly = u & 1;
        const size_t off = (r0 + poly * pstride) * kt.n + k0 + lane;
        uint64_t x[NCMAX];
#pragma unroll
        for (int c = 0; c < NCMAX; ++c) x[c] = c < a.nc ? a.ct[c][(size_t)b * a.is + off] : 0;
        const uint64_t *w = spt + lane;
        for (int o = 0; o < a.no; ++o, w += a.nc * kDmTK) {
            // <= 16 terms < q^2 each per 128-bit sum (< q 2^64 for q < 2^60); absent terms are 0; a
            // 32-wide instantiation reduces its first 16 terms before the next 16
            U128 acc{0, 0};
            uint64_t part = 0;
#pragma unroll
            for (int c = 0; c < NCMAX; ++c) {
                if (c == 16) {
                    part = redc(acc, q, qi);
                    acc = U128{0, 0};
                }
                if (c < a.nc) mac128(acc, x[c], w[c * kDmTK]);
            }
            const uint64_t v = redc(acc, q, qi);
            a.out[o][(size_t)b * a.os + off] = NCMAX > 16 ? add_mod(v, part, q) : v;
        }
    }
}

// The L2-shared variant (round 1's design): grid.x = tile * B + item, so the B CTAs of a tile
// read its plaintext words from L2; one (poly, residue row) per CTA; the next output's
// plaintext words are prefetched into registers while the current output accumulates.
template <int NCMAX>
__global__ void __launch_bounds__(256) k_diag_mac_l2(DiagMacArgs a, KTables kt)
{
    const uint32_t item = blockIdx.x % a.B, tile = blockIdx.x / a.B;
    const uint32_t k = tile * blockDim.x + threadIdx.x;
    if (k >= kt.n) return;
    const uint32_t L1 = a.level + 1, ry = blockIdx.y;
    uint32_t prow, prime;
    if (ry < 2 * L1) {
        prow = ry % L1;
        prime = prow;
    } else {
        const uint32_t kk = (ry - 2 * L1) % a.pk;
        prow = L1 + kk;
        prime = a.L + 1 + kk;
    }
    const size_t off = (size_t)ry * kt.n + k, poff = (size_t)prow * kt.n + k;
    const uint64_t q = kt.q[prime], qi = kt.qinv_neg[prime];
    uint64_t x[NCMAX], w[NCMAX];
#pragma unroll
    for (int c = 0; c < NCMAX; ++c) x[c] = c < a.nc ? a.ct[c][(size_t)item * a.is + off] : 0;
#pragma unroll
    for (int c = 0; c < NCMAX; ++c) w[c] = (c < a.nc && a.pt[0][c]) ? __ldg(a.pt[0][c] + poff) : 0;
    for (int o = 0; o < a.no; ++o) {
        uint64_t wn[NCMAX];
        const bool more = o + 1 < a.no;
#pragma unroll
        for (int c = 0; c < NCMAX; ++c)
            wn[c] = (more && c < a.nc && a.pt[o + 1][c]) ? __ldg(a.pt[o + 1][c] + poff) : 0;
        U128 acc{0, 0};  // <= 16 terms < q^2 each: < q 2^64 for q < 2^60; absent terms are 0
#pragma unroll
        for (int c = 0; c < NCMAX; ++c) mac128(acc, x[c], w[c]);
        a.out[o][(size_t)item * a.os + off] = redc(acc, q, qi);
#pragma unroll
        for (int c = 0; c < NCMAX; ++c) w[c] = wn[c];
    }
}

// K3's inner sums with Gauss's three-product complex multiplication:
// for giant g and baby s with plaintexts C = pc, S = ps, NS = pns (Eqs. dft_re / dft_im),
//   re_g = sum_s C xr + NS xi = sum_s C (xr + xi) - (C - NS) xi
//   im_g = sum_s S xr + C xi  = sum_s C (xr + xi) + (S - C) xr
// -- exact modular identities of the same encoded residues, so the outputs equal the four-
// product sums bit for bit with 3/4 of the MACs.  Staged like k_diag_mac: per tile the words
// C, S - C and C - NS of every (g, s) in shared memory, then the batch items.
struct K3MacArgs {
    const uint64_t *xr[kDiagMax], *xi[kDiagMax];
    const uint64_t *pc[kDiagMax][kDiagMax], *ps[kDiagMax][kDiagMax], *pns[kDiagMax][kDiagMax];  // [g][s]
    uint64_t *re[kDiagMax], *im[kDiagMax];
    size_t is, os;
    int nb, ng;
    uint32_t level, L, pk, B;
};

#ifndef MMFHE_K3_THREADS
#define MMFHE_K3_THREADS 128
#endif
template <int NB>
__global__ void __launch_bounds__(MMFHE_K3_THREADS) k_k3_gauss_mac(K3MacArgs a, KTables kt)
{
    extern __shared__ uint64_t sw[];  // [ng][3][nb][kDmTK]: C, S - C, C - NS (0 for absent)
    const uint32_t L1 = a.level + 1;
    const uint32_t pr = blockIdx.y;
    const uint32_t prime = pr < L1 ? pr : a.L + 1 + (pr - L1);
    const uint64_t q = kt.q[prime], qi = kt.qinv_neg[prime];
    const uint32_t k0 = blockIdx.x * kDmTK;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const int nt = a.ng * a.nb;
    for (int t = warp; t < nt; t += nw) {
        const int g = t / a.nb, s = t % a.nb;
        uint64_t c = 0, d = 0, e = 0;
        if (a.pc[g][s]) {
            const size_t o = (size_t)pr * kt.n + k0 + lane;
            c = __ldg(a.pc[g][s] + o);
            const uint64_t sv = __ldg(a.ps[g][s] + o), nv = __ldg(a.pns[g][s] + o);
            d = sub_mod(sv, c, q);
            e = sub_mod(c, nv, q);
        }
        uint64_t *dst = sw + ((size_t)(g * 3) * a.nb + s) * kDmTK + lane;
        dst[0] = c;
        dst[(size_t)a.nb * kDmTK] = d;
        dst[(size_t)2 * a.nb * kDmTK] = e;
    }
    __syncthreads();
    const size_t r0 = pr < L1 ? pr : 2 * L1 + (pr - L1);
    const size_t pstride = pr < L1 ? L1 : a.pk;
    for (uint32_t u = warp; u < 2 * a.B; u += nw) {
        const uint32_t b = u >> 1, poly = u & 1;
        const size_t off = (r0 + poly * pstride) * kt.n + k0 + lane;
        uint64_t xr[NB], xi[NB];
#pragma unroll
        for (int s = 0; s < NB; ++s) {
            xr[s] = s < a.nb ? a.xr[s][(size_t)b * a.is + off] : 0;
            xi[s] = s < a.nb ? a.xi[s][(size_t)b * a.is + off] : 0;
        }
        const uint64_t *w = sw + lane;
        for (int g = 0; g < a.ng; ++g, w += (size_t)3 * a.nb * kDmTK) {
            U128 k1{0, 0}, k2{0, 0}, k3{0, 0};  // <= 16 terms < q^2 each: < q 2^64 for q < 2^60
#pragma unroll
            for (int s = 0; s < NB; ++s) {
                if (s < a.nb) {
                    mac128(k1, add_mod(xr[s], xi[s], q), w[s * kDmTK]);
                    mac128(k2, xr[s], w[(a.nb + s) * kDmTK]);
                    mac128(k3, xi[s], w[(2 * a.nb + s) * kDmTK]);
                }
            }
            const uint64_t v1 = redc(k1, q, qi), v2 = redc(k2, q, qi), v3 = redc(k3, q, qi);
            a.re[g][(size_t)b * a.os + off] = sub_mod(v1, v3, q);
            a.im[g][(size_t)b * a.os + off] = add_mod(v1, v2, q);
        }
    }
}

constexpr int kJG = 4;  // outputs per thread in the modular matrix product (2 x 128-bit accumulators each)
constexpr int kFold = 128;  // input rows between hi-word folds in k_lincomb_mat

// out[j] = sum_w C[j][w] in[lo_j + w] for j in this CTA's group of kJG outputs.  Each
// term is one 64x64->128 multiply-accumulate per poly with the coefficient in Montgomery
// form (C[.].wp = c 2^64 mod q); every accumulator is reduced once at the end (hi word
// brought below q, then one Montgomery reduction).  Each term is < q^2 < 2^120, so a
// 128-bit sum of more than 256 terms could wrap: every kFold input rows the hi words are
// folded below q (subtracting multiples of q 2^64 leaves the Montgomery result unchanged),
// which keeps hi < q + kFold q / 16 < 2^17 q (the reduce_est precondition) for any W.
__global__ void __launch_bounds__(kTB) k_lincomb_mat(uint64_t *__restrict__ out, const uint64_t *__restrict__ in,
                                                     uint32_t M, uint32_t J, uint32_t W, int lo0, int lo_step,
                                                     const TwPair *__restrict__ C, KTables kt, uint32_t level)
{
    const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= kt.n) return;
    const uint32_t r = blockIdx.y;
    const uint32_t j0 = blockIdx.z * kJG;
    const uint32_t jn = min((uint32_t)kJG, J - j0);
    const uint64_t q = kt.q[r], qi = kt.qinv_neg[r];
    const uint32_t L1 = level + 1;
    const size_t ps = (size_t)L1 * kt.n, item = 2 * ps;
    const size_t off = (size_t)r * kt.n + k;
    int ilo = lo0 + (int)j0 * lo_step, ihi = lo0 + (int)(j0 + jn - 1) * lo_step + (int)W;
    if (lo_step < 0) {
        const int tmp = lo0 + (int)(j0 + jn - 1) * lo_step;
        ihi = lo0 + (int)j0 * lo_step + (int)W;
        ilo = tmp;
    }
    ilo = max(ilo, 0);
    ihi = min(ihi, (int)M);
    U128 a0[kJG], a1[kJG];
#pragma unroll
    for (int jj = 0; jj < kJG; ++jj) a0[jj] = a1[jj] = U128{0, 0};
    const float qinv = qinv_est(q);
    for (int i = ilo; i < ihi; ++i) {
        if (((i - ilo) & (kFold - 1)) == kFold - 1) {
#pragma unroll
            for (int jj = 0; jj < kJG; ++jj) {
                a0[jj].hi = reduce_est(a0[jj].hi, q, qinv);
                a1[jj].hi = reduce_est(a1[jj].hi, q, qinv);
            }
        }
        const uint64_t x0 = in[(size_t)i * item + off], x1 = in[(size_t)i * item + ps + off];
#pragma unroll
        for (int jj = 0; jj < kJG; ++jj) {
            if (jj < (int)jn) {
                const int w = i - (lo0 + (int)(j0 + jj) * lo_step);
                if (w >= 0 && w < (int)W) {
                    const uint64_t c = C[((size_t)(j0 + jj) * W + w) * L1 + r].wp;
                    mac128(a0[jj], x0, c);
                    mac128(a1[jj], x1, c);
                }
            }
        }
    }
#pragma unroll
    for (int jj = 0; jj < kJG; ++jj) {
        if (jj < (int)jn) {
            U128 x = a0[jj];
            x.hi = reduce_est(x.hi, q, qinv);
            out[(size_t)(j0 + jj) * item + off] = redc(x, q, qi);
            x = a1[jj];
            x.hi = reduce_est(x.hi, q, qinv);
            out[(size_t)(j0 + jj) * item + ps + off] = redc(x, q, qi);
        }
    }
}

// Symmetric Toeplitz rows (K5 FIR with linear-phase taps): every output j
// uses the same taps c_w on inputs lo0 + j + w with c_w == c_{W-1-w} as encoded integers
// (checked on the host), so out[j] = sum_{w < W/2} c_w (x_a + x_b) + c_mid x_mid exactly
// (mod q): half the modular products of k_lincomb_mat.  A CTA stages the input window of
// its kSymJT outputs for kSymK coefficients of one (poly, limb) row in shared memory
// (zeros outside [0, M)) together with the taps (Montgomery form); each thread owns one
// coefficient and kSymJT / kSymSplit outputs, computed kSymJB at a time: the kSymJB
// outputs' input pairs slide along the window (two shared-memory reads per tap for all
// kSymJB outputs) and each tap is one 64x64->128 multiply-accumulate per output, reduced
// once at the end (hi word brought below q, then one Montgomery reduction).
// Tile sweep on C2 (profiles/r01/sym_variants*_r01p.log, parity green for each): JB 4 /
// split 2 (kept) 5194 frames/s; JB 8: 5073; split 4: 4975; split 1 with JB 4 / 8 / 16:
// 5172-5182 / 5172-5191 / 5095 -- the defaults are at the optimum within run-to-run noise.
#ifndef MMFHE_SYM_JB
#define MMFHE_SYM_JB 4
#endif
#ifndef MMFHE_SYM_SPLIT
#define MMFHE_SYM_SPLIT 2
#endif
constexpr int kSymK = 128, kSymJT = 32, kSymSplit = MMFHE_SYM_SPLIT, kSymJB = MMFHE_SYM_JB;

__global__ void __launch_bounds__(kSymK *kSymSplit) k_lincomb_sym(uint64_t *__restrict__ out,
                                                                  const uint64_t *__restrict__ in, uint32_t M,
                                                                  uint32_t J, uint32_t W, int lo0,
                                                                  const TwPair *__restrict__ T, KTables kt,
                                                                  uint32_t level)
{
    extern __shared__ uint64_t X[];  // [kSymJT + W - 1][kSymK], then the taps [W / 2 + 1]
    const uint32_t L1 = level + 1;
    const uint32_t r = blockIdx.y % L1, poly = blockIdx.y / L1;
    const uint32_t k0 = blockIdx.x * kSymK, j0 = blockIdx.z * kSymJT;
    const uint64_t q = kt.q[r], qi = kt.qinv_neg[r];
    const size_t ps = (size_t)L1 * kt.n, item = 2 * ps;
    const size_t col = (size_t)poly * ps + (size_t)r * kt.n + k0;
    const int rows = kSymJT + (int)W - 1;
    uint64_t *cm = X + (size_t)rows * kSymK;
    for (int w = threadIdx.x; w <= (int)W / 2; w += blockDim.x) cm[w] = T[(size_t)w * L1 + r].wp;  // c 2^64 mod q
    for (int idx = threadIdx.x; idx < rows * kSymK; idx += blockDim.x) {
        const int i = lo0 + (int)j0 + idx / kSymK;
        X[idx] = (i >= 0 && i < (int)M) ? in[(size_t)i * item + col + idx % kSymK] : 0;
    }
    __syncthreads();
    const int k = threadIdx.x % kSymK, part = threadIdx.x / kSymK;
    const uint64_t *Xk = X + k;
    const float qinv = qinv_est(q);
    constexpr int per = kSymJT / kSymSplit;
    const int half = (int)W / 2;
    for (int jb = part * per; jb < (part + 1) * per; jb += kSymJB) {
        if (j0 + jb >= J) break;
        // lo[i] = X[jb + i + w], hi[i] = X[jb + i + W - 1 - w] at tap w
        uint64_t lo[kSymJB], hi[kSymJB];
        U128 acc[kSymJB];
#pragma unroll
        for (int i = 0; i < kSymJB; ++i) {
            lo[i] = Xk[(jb + i) * kSymK];
            hi[i] = Xk[(jb + i + (int)W - 1) * kSymK];
            acc[i] = U128{0, 0};
        }
        for (int w = 0; w < half; ++w) {
            const uint64_t c = cm[w];
#pragma unroll
            for (int i = 0; i < kSymJB; ++i) mac128(acc[i], lo[i] + hi[i], c);  // (< 2q) x (< q)
#pragma unroll
            for (int i = 0; i < kSymJB - 1; ++i) {
                lo[i] = lo[i + 1];
                hi[kSymJB - 1 - i] = hi[kSymJB - 2 - i];
            }
            lo[kSymJB - 1] = Xk[(jb + kSymJB + w) * kSymK];
            hi[0] = Xk[(jb + (int)W - 2 - w) * kSymK];
        }
        if (W & 1) {
            // after the loop lo[i] = X[jb + i + W/2]: the middle tap
            const uint64_t c = cm[half];
#pragma unroll
            for (int i = 0; i < kSymJB; ++i) mac128(acc[i], lo[i], c);
        }
#pragma unroll
        for (int i = 0; i < kSymJB; ++i) {
            const uint32_t j = j0 + jb + i;
            if (j >= J) break;
            // acc < (W/2 + 1) 2q^2 (<= 65 terms): hi < 2^17 q, reduced below q so that the
            // Montgomery reduction's input is < q 2^64 (subtracting multiples of q 2^64 does
            // not change the result mod q)
            U128 x = acc[i];
            x.hi = reduce_est(x.hi, q, qinv);
            out[(size_t)j * item + col + k] = redc(x, q, qi);
        }
    }
}

__global__ void k_batch_sum(uint64_t *__restrict__ out, const uint64_t *__restrict__ in, uint32_t B, size_t item,
                            KTables kt, uint32_t level)
{
    const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= kt.n) return;
    const uint32_t r = blockIdx.y;
    const uint64_t q = kt.q[r % (level + 1)];
    const size_t off = (size_t)r * kt.n + k;
    uint64_t s = 0;
    for (uint32_t b = 0; b < B; ++b) s = add_mod(s, in[(size_t)b * item + off], q);
    out[off] = s;
}

// out[b] = *src[b] for n items of `words` words (16-byte vector copies).
__global__ void k_gather(uint64_t *__restrict__ out, PtrList src, size_t words)
{
    const size_t i = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) * 2;
    if (i >= words) return;
    const uint64_t *s = src.p[blockIdx.y];
    uint64_t *o = out + (size_t)blockIdx.y * words;
    if (i + 1 < words) {
        *(ulonglong2 *)(o + i) = *(const ulonglong2 *)(s + i);
    } else {
        o[i] = s[i];
    }
}

__global__ void k_add_plain(uint64_t *__restrict__ c0, size_t s, const uint64_t *__restrict__ pt, KTables kt)
{
    const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= kt.n) return;
    const uint32_t r = blockIdx.y;
    const uint64_t q = kt.q[r];
    const size_t off = (size_t)r * kt.n + k;
    const uint64_t v = redc(U128{pt[off], 0}, q, kt.qinv_neg[r]);
    uint64_t *c = c0 + (size_t)blockIdx.z * s;
    c[off] = add_mod(c[off], v, q);
}

// Double hoisting's P lift: Q rows of out (+)= [P]_{q_i} (.) src, read
// through sigma_g (NTT-domain gather; g = 1: none); rows = npoly (l+1), row r = poly (l+1) + i.
__global__ void k_pq_lift(uint64_t *__restrict__ out, size_t os, size_t ops, const uint64_t *__restrict__ src,
                          size_t ss, size_t sps, const TwPair *__restrict__ pmod, KTables kt, uint32_t l1, uint32_t g,
                          int accumulate)
{
    const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= kt.n) return;
    const uint32_t poly = blockIdx.y / l1, i = blockIdx.y % l1;
    const uint64_t q = kt.q[i];
    const TwPair m = pmod[i];
    const uint64_t v = shoup(src[blockIdx.z * ss + poly * sps + (size_t)i * kt.n + galois_perm(k, g, kt.log_n)], m.w,
                             m.wp, q);
    uint64_t *o = out + blockIdx.z * os + poly * ops + (size_t)i * kt.n + k;
    *o = accumulate ? add_mod(*o, v, q) : v;
}

}  // namespace

// ------------------------------------------------------------------ launchers
#define LAUNCH_CHECK(c)                                                                           \
    do {                                                                                          \
        ++(c).launches;                                                                           \
        CUDA_CHECK(cudaGetLastError());                                                           \
    } while (0)

void launch_addsub(Ctx &c, uint64_t *out, const uint64_t *a, const uint64_t *b, uint32_t rows, const PrimeMap &pm,
                   bool sub)
{
    ProfScope ps(c, "addsub", 24.0 * rows * c.n);
    k_addsub<<<grid3(c.n, rows), kTB, 0, c.stream>>>(out, a, b, c.kt, pm, sub ? 1 : 0);
    LAUNCH_CHECK(c);
}

void launch_to_mont(Ctx &c, uint64_t *x, uint32_t rows, const PrimeMap &pm)
{
    ProfScope ps(c, "to_mont", 16.0 * rows * c.n);
    k_to_mont<<<grid3(c.n, rows), kTB, 0, c.stream>>>(x, c.kt, pm);
    LAUNCH_CHECK(c);
}


void launch_modup_bconv(Ctx &c, uint64_t *y, size_t ys, const uint64_t *x_coef, size_t xs, uint32_t level,
                        const std::vector<size_t> &off, uint32_t B)
{
    const auto &plans = c.modup[level];
    MMFHE_REQUIRE(plans.size() <= 16 && c.alpha <= 16, MMFHE_E_PARAMS, "dnum/alpha too large");
    ModUpArgs a{};
    a.level = level;
    a.L = c.L;
    a.xs = xs;
    a.ys = ys;
    double words = 0, macs = 0;
    for (const auto &p : plans) {
        words += (double)(p.hi - p.lo) + p.n_tgt;
        macs += (double)(p.hi - p.lo) * p.n_tgt;  // 64x64->128 MACs per coefficient
    }
    ProfScope ps(c, "modup_bconv", 8.0 * words * c.n * B, macs * c.n * B);
    for (size_t j = 0; j < plans.size(); ++j) {
        const ModUpPlan &p = plans[j];
        a.d[j].hat_inv = (const TwPair *)c.bconv_ptr(p.off_hat_inv);
        a.d[j].hat = (const uint64_t *)c.bconv_ptr(p.off_hat);
        a.d[j].tgt = (const uint32_t *)c.bconv_ptr(p.off_tgt);
        a.d[j].y_off = off[j] * c.n;
        a.d[j].lo = p.lo;
        a.d[j].hi = p.hi;
        a.d[j].n_tgt = p.n_tgt;
    }
    size_t smem = 0;
    for (const auto &p : plans) smem = std::max(smem, 8 * ((size_t)(p.hi - p.lo) * p.n_tgt + 2 * p.n_tgt));
    const dim3 g((c.n + kBcK * kTB - 1) / (kBcK * kTB), (uint32_t)plans.size(), B);
    if (c.alpha <= 1)
        k_modup<1><<<g, kTB, smem, c.stream>>>(y, x_coef, c.kt, a);
    else if (c.alpha <= 4)
        k_modup<4><<<g, kTB, smem, c.stream>>>(y, x_coef, c.kt, a);
    else if (c.alpha <= 8)
        k_modup<8><<<g, kTB, smem, c.stream>>>(y, x_coef, c.kt, a);
    else
        k_modup<16><<<g, kTB, smem, c.stream>>>(y, x_coef, c.kt, a);
    LAUNCH_CHECK(c);
}

void launch_key_ip(Ctx &c, uint64_t *accQ, uint64_t *accP, const uint64_t *x_ntt, size_t xs, const uint64_t *y,
                   size_t ys, const std::vector<size_t> &off, const uint64_t *key, uint32_t level, uint32_t B,
                   uint32_t gx, uint32_t gy, const IPOut *os, const IPEpi *ep)
{
    const auto &plans = c.modup[level];
    IPArgs a{};
    if (ep) a.ep = *ep;
    if (os) {
        a.oqs = os->qs;
        a.oqp = os->qp;
        a.ops = os->ps;
        a.opp = os->pp;
    } else {  // compact accQ [B][2][l+1][N], accP [B][2][K][N]
        a.oqp = (size_t)(level + 1) * c.n;
        a.oqs = 2 * a.oqp;
        a.opp = (size_t)c.K * c.n;
        a.ops = 2 * a.opp;
    }
    a.dnum = (uint32_t)plans.size();
    a.level = level;
    a.L = c.L;
    a.K = c.K;
    a.B = B;
    a.xs = xs;
    a.ys = ys;
    a.gx = gx;
    a.gy = gy;
    for (size_t j = 0; j < plans.size(); ++j) {
        a.y_off[j] = off[j] * c.n;
        a.lo[j] = plans[j].lo;
        a.hi[j] = plans[j].hi;
    }
    const double rows = level + 1 + c.K;  // per row: key 2 dnum words once; per item dnum in + 2 out
    ProfScope ps(c, "key_ip", 8.0 * rows * c.n * (2.0 * a.dnum + B * (a.dnum + 2.0)), 2.0 * a.dnum * rows * c.n * B);
    // split the batch over grid.z so that >= ~8 CTAs per SM are in flight; the key words
    // are then re-read once per z-chunk (negligible next to the per-item traffic)
    const uint32_t ctas_xy = ((c.n + kTB - 1) / kTB) * (level + 1 + c.K);
    uint32_t nz = std::max<uint32_t>(1, std::min<uint32_t>(B, (148 * 8 + ctas_xy - 1) / ctas_xy));
    a.per_z = (B + nz - 1) / nz;
    nz = (B + a.per_z - 1) / a.per_z;
    const dim3 g = grid3(c.n, level + 1 + c.K, nz);
    if (MMFHE_D3 && a.dnum == 3) {  // PS3 / PS4 / PSV: exact digit count
        if (ep)
            k_key_ip<3, true><<<g, kTB, 0, c.stream>>>(accQ, accP, x_ntt, y, key, c.kt, a);
        else
            k_key_ip<3><<<g, kTB, 0, c.stream>>>(accQ, accP, x_ntt, y, key, c.kt, a);
    } else if (ep) {  // the fused-epilogue instantiations (double hoisting) carry its registers alone
        if (a.dnum <= 4)
            k_key_ip<4, true><<<g, kTB, 0, c.stream>>>(accQ, accP, x_ntt, y, key, c.kt, a);
        else if (a.dnum <= 8)
            k_key_ip_lr<8, true><<<g, kTB, 0, c.stream>>>(accQ, accP, x_ntt, y, key, c.kt, a);
        else
            k_key_ip<16, true><<<g, kTB, 0, c.stream>>>(accQ, accP, x_ntt, y, key, c.kt, a);
    } else if (a.dnum <= 4)
        k_key_ip<4><<<g, kTB, 0, c.stream>>>(accQ, accP, x_ntt, y, key, c.kt, a);
    else if (a.dnum <= 8)
        k_key_ip_lr<8><<<g, kTB, 0, c.stream>>>(accQ, accP, x_ntt, y, key, c.kt, a);
    else
        k_key_ip<16><<<g, kTB, 0, c.stream>>>(accQ, accP, x_ntt, y, key, c.kt, a);
    LAUNCH_CHECK(c);
}

static MDArgs md_args(Ctx &c, uint32_t level, const uint64_t *zq)
{
    MDArgs a;
    if (zq) {  // R31: sources p_0..p_{K-1}, q_level; modulus M = P q_level
        a.phat_inv = (const TwPair *)c.bconv_ptr(c.off_mr_hinv) + (size_t)level * (c.K + 1);
        a.phat = (const uint64_t *)c.bconv_ptr(c.off_mr_hat) + (size_t)level * (c.K + 1) * (c.L + 1);
    } else {
        a.phat_inv = (const TwPair *)c.bconv_ptr(c.off_pd_hat_inv);
        a.phat = (const uint64_t *)c.bconv_ptr(c.off_pd_hat);
    }
    a.pinv = (const TwPair *)c.bconv_ptr(c.off_pd_pinv);
    a.zq = zq;
    a.level = level;
    a.L = c.L;
    a.K = c.K;
    return a;
}

void launch_moddown_bconv(Ctx &c, uint64_t *w, const uint64_t *zP, uint32_t level, uint32_t B, uint32_t npoly,
                          const uint64_t *zq)
{
    const uint32_t ns = c.K + (zq ? 1 : 0), nt = zq ? level : level + 1;
    MMFHE_REQUIRE(ns <= 16, MMFHE_E_PARAMS, "K too large");
    MMFHE_REQUIRE(!zq || level >= 1, MMFHE_E_DEPTH, "merged ModDown + rescale needs level >= 1");
    ProfScope ps(c, "moddown_bconv", 8.0 * npoly * (ns + nt) * c.n * B, (double)npoly * ns * nt * c.n * B);
    const size_t smem = 8 * ((size_t)ns * nt + 2 * nt);
    const dim3 g((c.n + kBcK * kTB - 1) / (kBcK * kTB), npoly * B);
    const MDArgs a = md_args(c, level, zq);
    if (ns <= 1)
        k_moddown_bconv<1><<<g, kTB, smem, c.stream>>>(w, zP, c.kt, a);
    else if (ns <= 4)
        k_moddown_bconv<4><<<g, kTB, smem, c.stream>>>(w, zP, c.kt, a);
    else if (ns <= 8)
        k_moddown_bconv<8><<<g, kTB, smem, c.stream>>>(w, zP, c.kt, a);
    else
        k_moddown_bconv<16><<<g, kTB, smem, c.stream>>>(w, zP, c.kt, a);
    LAUNCH_CHECK(c);
}


void launch_tensor_sum(Ctx &c, uint64_t *out, size_t os, const PtrList &a, const PtrList &b, size_t is, int n,
                       uint32_t level, bool accumulate, uint32_t B)
{
    double in_words = 0;
    for (int i = 0; i < n; ++i) in_words += (a.p[i] == b.p[i]) ? 2.0 : 4.0;
    ProfScope ps(c, "tensor_sum", 8.0 * (level + 1) * c.n * B * (in_words + 3.0 + (accumulate ? 3.0 : 0.0)));
    if (n == 1)
        k_tensor1<<<dim3((c.n + 2 * kTB - 1) / (2 * kTB), level + 1, B), kTB, 0, c.stream>>>(
            out, os, a.p[0], b.p[0], is, c.kt, level, accumulate ? 1 : 0);
    else
        k_tensor_sum<<<grid3(c.n, level + 1, B), kTB, 0, c.stream>>>(out, os, a, b, is, n, c.kt, level,
                                                                     accumulate ? 1 : 0);
    LAUNCH_CHECK(c);
}

void launch_pmult_sum(Ctx &c, uint64_t *out, size_t os, const PtrList &pt, const PtrList &ct, size_t is, int n,
                      uint32_t level, bool accumulate, uint32_t B)
{
    ProfScope ps(c, "pmult_sum",
                 8.0 * (level + 1) * c.n * ((double)n + B * (2.0 * n + 2.0 + (accumulate ? 2.0 : 0.0))));
    k_pmult_sum<<<grid3(c.n, level + 1, B), kTB, 0, c.stream>>>(out, os, pt, ct, is, n, c.kt, level,
                                                                accumulate ? 1 : 0);
    LAUNCH_CHECK(c);
}

void launch_diag_mac(Ctx &c, const std::vector<const uint64_t *> &cts, size_t is,
                     const std::vector<std::vector<const uint64_t *>> &pts, const std::vector<uint64_t *> &outs,
                     size_t os, uint32_t level, uint32_t B, uint32_t pk)
{
    MMFHE_REQUIRE(cts.size() <= (size_t)kDiagIn && outs.size() <= (size_t)kDiagMax && pts.size() == outs.size(),
                  MMFHE_E_LAYOUT, "diag_mac shape");
    MMFHE_REQUIRE(c.n % kDmTK == 0, MMFHE_E_PARAMS, "N must be a multiple of 32");
    DiagMacArgs a{};
    a.nc = (int)cts.size();
    a.no = (int)outs.size();
    a.is = is;
    a.os = os;
    a.level = level;
    a.L = c.L;
    a.pk = pk;
    a.B = B;
    double terms = 0;
    for (size_t i = 0; i < cts.size(); ++i) a.ct[i] = cts[i];
    for (size_t o = 0; o < outs.size(); ++o) {
        a.out[o] = outs[o];
        for (size_t i = 0; i < cts.size(); ++i) {
            a.pt[o][i] = pts[o][i];
            terms += pts[o][i] != nullptr;
        }
    }
    const double rows = level + 1 + pk;
    // algorithmic: babies read once, plaintexts once per launch, outputs written once
    ProfScope ps(c, "diag_mac", 8.0 * rows * c.n * (terms + B * 2.0 * (a.nc + a.no)), 2.0 * terms * rows * c.n * B);
    // plaintext-stationary staging (k_diag_mac) once a batch amortises the tile's plaintext words
    // (C4 complex K3, B = 13: 4.98 -> 4.15 ms, profiles/r02/c4prof_staged_r02ag.log); the L2-shared
    // variant for small batches (FC, B = 1).  MMFHE_DIAG_STAGED=1 / 0 forces one (A/B runs).
    static const int forced = [] {
        const char *e = getenv("MMFHE_DIAG_STAGED");
        return e ? (*e == '1' ? 1 : 0) : -1;
    }();
    // more than 16 baby steps: the staged kernel only (its 32-wide instantiation)
    const bool l2_variant = a.nc <= kDiagMax && (forced >= 0 ? forced == 0 : B < 4);
    if (l2_variant) {
        const dim3 g(((c.n + 255) / 256) * B, 2 * (level + 1 + pk));
        if (a.nc <= 4)
            k_diag_mac_l2<4><<<g, 256, 0, c.stream>>>(a, c.kt);
        else if (a.nc <= 8)
            k_diag_mac_l2<8><<<g, 256, 0, c.stream>>>(a, c.kt);
        else
            k_diag_mac_l2<16><<<g, 256, 0, c.stream>>>(a, c.kt);
        LAUNCH_CHECK(c);
        return;
    }
    static std::atomic<uint64_t> attr{0};
    once_per_device(attr, [] {
        const int mx = (int)(sizeof(uint64_t) * kDiagMax * kDiagIn * kDmTK);
        CUDA_CHECK(cudaFuncSetAttribute(k_diag_mac<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
        CUDA_CHECK(cudaFuncSetAttribute(k_diag_mac<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
        CUDA_CHECK(cudaFuncSetAttribute(k_diag_mac<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
        CUDA_CHECK(cudaFuncSetAttribute(k_diag_mac<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
    });
    const size_t smem = sizeof(uint64_t) * (size_t)a.no * a.nc * kDmTK;
    const dim3 g(c.n / kDmTK, level + 1 + pk);
    if (a.nc <= 4)
        k_diag_mac<4><<<g, 128, smem, c.stream>>>(a, c.kt);
    else if (a.nc <= 8)
        k_diag_mac<8><<<g, 128, smem, c.stream>>>(a, c.kt);
    else if (a.nc <= 16)
        k_diag_mac<16><<<g, 128, smem, c.stream>>>(a, c.kt);
    else
        k_diag_mac<32><<<g, 128, smem, c.stream>>>(a, c.kt);
    LAUNCH_CHECK(c);
}

void launch_k3_gauss_mac(Ctx &c, const std::vector<const uint64_t *> &xr, const std::vector<const uint64_t *> &xi,
                         size_t is, const std::vector<std::vector<const uint64_t *>> &pc,
                         const std::vector<std::vector<const uint64_t *>> &ps,
                         const std::vector<std::vector<const uint64_t *>> &pns, const std::vector<uint64_t *> &re,
                         const std::vector<uint64_t *> &im, size_t os, uint32_t level, uint32_t B, uint32_t pk)
{
    const int nb = (int)xr.size(), ng = (int)re.size();
    MMFHE_REQUIRE(nb <= kDiagMax && ng <= kDiagMax && xi.size() == xr.size() && im.size() == re.size(),
                  MMFHE_E_LAYOUT, "K3 MAC shape");
    K3MacArgs a{};
    a.nb = nb;
    a.ng = ng;
    a.is = is;
    a.os = os;
    a.level = level;
    a.L = c.L;
    a.pk = pk;
    a.B = B;
    double terms = 0;
    for (int s = 0; s < nb; ++s) {
        a.xr[s] = xr[s];
        a.xi[s] = xi[s];
    }
    for (int g = 0; g < ng; ++g) {
        a.re[g] = re[g];
        a.im[g] = im[g];
        for (int s = 0; s < nb; ++s) {
            a.pc[g][s] = pc[g][s];
            a.ps[g][s] = ps[g][s];
            a.pns[g][s] = pns[g][s];
            terms += pc[g][s] != nullptr;
        }
    }
    const double rows = level + 1 + pk;
    ProfScope ps_(c, "diag_mac", 8.0 * rows * c.n * (3 * terms + B * 2.0 * 2 * (nb + ng)), 2.0 * 3 * terms * rows * c.n * B);
    static std::atomic<uint64_t> attr{0};
    once_per_device(attr, [] {
        const int mx = (int)(sizeof(uint64_t) * 3 * kDiagMax * kDiagMax * kDmTK);
        CUDA_CHECK(cudaFuncSetAttribute(k_k3_gauss_mac<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
        CUDA_CHECK(cudaFuncSetAttribute(k_k3_gauss_mac<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
    });
    const size_t smem = sizeof(uint64_t) * 3 * (size_t)ng * nb * kDmTK;
    const dim3 g(c.n / kDmTK, level + 1 + pk);
    if (nb <= 8)
        k_k3_gauss_mac<8><<<g, MMFHE_K3_THREADS, smem, c.stream>>>(a, c.kt);
    else
        k_k3_gauss_mac<16><<<g, MMFHE_K3_THREADS, smem, c.stream>>>(a, c.kt);
    LAUNCH_CHECK(c);
}

void launch_lincomb_mat(Ctx &c, uint64_t *out, const uint64_t *in, uint32_t M, uint32_t J, uint32_t W, int lo0,
                        int lo_step, const TwPair *C, uint32_t level)
{
    MMFHE_REQUIRE(W <= 8192, MMFHE_E_SHAPE, "lincomb window too long");
    ProfScope ps(c, "lincomb_mat", 8.0 * 2.0 * (level + 1) * c.n * ((double)M + J),
                 2.0 * (level + 1) * c.n * (double)J * std::min<uint32_t>(W, M));
    k_lincomb_mat<<<grid3(c.n, level + 1, (J + kJG - 1) / kJG), kTB, 0, c.stream>>>(out, in, M, J, W, lo0, lo_step,
                                                                                   C, c.kt, level);
    LAUNCH_CHECK(c);
}

void launch_lincomb_sym(Ctx &c, uint64_t *out, const uint64_t *in, uint32_t M, uint32_t J, uint32_t W, int lo0,
                        const TwPair *T, uint32_t level)
{
    const size_t smem = sizeof(uint64_t) * ((kSymJT + W - 1) * kSymK + W / 2 + 1);
    MMFHE_REQUIRE(smem <= 200 * 1024, MMFHE_E_SHAPE, "FIR too long for the staged window");
    static std::atomic<uint64_t> attr{0};
    once_per_device(attr, [] {
        CUDA_CHECK(cudaFuncSetAttribute(k_lincomb_sym, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    });
    ProfScope ps(c, "lincomb_mat", 8.0 * 2.0 * (level + 1) * c.n * ((double)M + J),
                 2.0 * (level + 1) * c.n * (double)J * (W / 2 + (W & 1)));
    const dim3 grid(c.n / kSymK, 2 * (level + 1), (J + kSymJT - 1) / kSymJT);
    k_lincomb_sym<<<grid, kSymK * kSymSplit, smem, c.stream>>>(out, in, M, J, W, lo0, T, c.kt, level);
    LAUNCH_CHECK(c);
}

void launch_batch_sum(Ctx &c, uint64_t *out, const uint64_t *in, uint32_t B, uint32_t npolys, uint32_t level)
{
    const uint32_t rows = npolys * (level + 1);
    ProfScope ps(c, "batch_sum", 8.0 * rows * c.n * (B + 1.0));
    k_batch_sum<<<grid3(c.n, rows), kTB, 0, c.stream>>>(out, in, B, (size_t)rows * c.n, c.kt, level);
    LAUNCH_CHECK(c);
}

void launch_gather(Ctx &c, uint64_t *out, const PtrList &src, int n, size_t words)
{
    ProfScope ps(c, "gather", 16.0 * words * n);
    const size_t threads = (words + 1) / 2;
    k_gather<<<dim3((unsigned)((threads + kTB - 1) / kTB), n), kTB, 0, c.stream>>>(out, src, words);
    LAUNCH_CHECK(c);
}

// dst.p[b] (as writable) = in + b * words, b < n (16-byte aligned destinations)
__global__ void k_scatter(PtrList dst, const uint64_t *__restrict__ in, size_t words)
{
    const size_t i = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) * 2;
    if (i >= words) return;
    uint64_t *o = const_cast<uint64_t *>(dst.p[blockIdx.y]);
    const uint64_t *s = in + (size_t)blockIdx.y * words;
    if (i + 1 < words) {
        *(ulonglong2 *)(o + i) = *(const ulonglong2 *)(s + i);
    } else {
        o[i] = s[i];
    }
}

void launch_scatter(Ctx &c, const PtrList &dst, const uint64_t *in, int n, size_t words)
{
    ProfScope ps(c, "scatter", 16.0 * words * n);
    const size_t threads = (words + 1) / 2;
    k_scatter<<<dim3((unsigned)((threads + kTB - 1) / kTB), n), kTB, 0, c.stream>>>(dst, in, words);
    LAUNCH_CHECK(c);
}

void launch_hoisted_ip_pq(Ctx &c, const uint64_t *x, size_t xs, const uint64_t *y, size_t ys,
                          const std::vector<size_t> &off, const uint64_t *c0, size_t cs,
                          const std::vector<const uint64_t *> &keys, const std::vector<uint32_t> &ginv,
                          const std::vector<uint64_t *> &outs, size_t os, uint32_t level, uint32_t B)
{
    const auto &plans = c.modup[level];
    MMFHE_REQUIRE(keys.size() == outs.size() && keys.size() == ginv.size() && keys.size() <= (size_t)kDiagMax &&
                      plans.size() <= 4,
                  MMFHE_E_LAYOUT, "hoisted PQ inner product: <= 16 steps, <= 4 digits");
    HoistIPArgs a{};
    a.dnum = (uint32_t)plans.size();
    a.level = level;
    a.L = c.L;
    a.K = c.K;
    a.B = B;
    a.xs = xs;
    a.ys = ys;
    a.cs = cs;
    a.os = os;
    a.nsteps = (uint32_t)keys.size();
    for (size_t s = 0; s < keys.size(); ++s) {
        a.key[s] = keys[s];
        a.out[s] = outs[s];
        a.ginv[s] = ginv[s];
    }
    for (size_t j = 0; j < plans.size(); ++j) {
        a.y_off[j] = off[j] * c.n;
        a.lo[j] = plans[j].lo;
        a.hi[j] = plans[j].hi;
    }
    const double rows = level + 1 + c.K, S = (double)keys.size();
    // algorithmic: digit words and c0 once, every step's key once, every output once
    ProfScope ps(c, "key_ip_group", 8.0 * c.n * (rows * B * a.dnum + (level + 1.0) * B + S * rows * 2.0 * a.dnum +
                                          S * B * 2.0 * rows),
                 2.0 * a.dnum * rows * c.n * B * S);
    const size_t smem = sizeof(uint64_t) * (size_t)B * (a.dnum + 1) * kHTile;
    MMFHE_REQUIRE(smem <= 200 * 1024, MMFHE_E_SHAPE, "hoisted PQ inner product: batch too large for one tile");
    static std::atomic<uint64_t> attr{0};
    once_per_device(attr, [] {
        CUDA_CHECK(cudaFuncSetAttribute(k_hoisted_ip_pq<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        CUDA_CHECK(cudaFuncSetAttribute(k_hoisted_ip_pq<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    });
    const dim3 g(c.n / kHTile, level + 1 + c.K);
    if (MMFHE_D3 && a.dnum == 3)
        k_hoisted_ip_pq<3><<<g, kHTile, smem, c.stream>>>(x, y, c0, (const TwPair *)c.bconv_ptr(c.off_pd_pmod), c.kt, a);
    else
        k_hoisted_ip_pq<4><<<g, kHTile, smem, c.stream>>>(x, y, c0, (const TwPair *)c.bconv_ptr(c.off_pd_pmod), c.kt, a);
    LAUNCH_CHECK(c);
}

void launch_hoisted_rotsum_pq(Ctx &c, uint64_t *out, size_t os, const uint64_t *x, size_t xs, const uint64_t *y,
                              size_t ys, const std::vector<size_t> &off, const uint64_t *c0, size_t cs,
                              const std::vector<const uint64_t *> &keys, const std::vector<uint32_t> &g,
                              uint32_t level, uint32_t B)
{
    const auto &plans = c.modup[level];
    MMFHE_REQUIRE(keys.size() == g.size() && !keys.empty() && keys.size() <= (size_t)kRSteps && plans.size() <= 8,
                  MMFHE_E_LAYOUT, "hoisted PQ rotate-and-sum: 1..64 steps, <= 8 digits");
    HoistSumArgs a{};
    a.dnum = (uint32_t)plans.size();
    a.level = level;
    a.L = c.L;
    a.K = c.K;
    a.B = B;
    a.xs = xs;
    a.ys = ys;
    a.cs = cs;
    a.os = os;
    a.nsteps = (uint32_t)keys.size();
    for (size_t j = 0; j < plans.size(); ++j) {
        a.y_off[j] = off[j] * c.n;
        a.lo[j] = plans[j].lo;
        a.hi[j] = plans[j].hi;
    }
    for (size_t s = 0; s < keys.size(); ++s) {
        a.key[s] = keys[s];
        a.g[s] = g[s];
    }
    const double rows = level + 1 + c.K, S = (double)keys.size();
    // algorithmic: digit words, c1 and c0 once (read S times through L2), every step's key once, the sum once
    ProfScope ps(c, "key_ip_rotsum", 8.0 * c.n * (rows * B * a.dnum + 2.0 * (level + 1.0) * B + S * rows * 2.0 * a.dnum +
                                            B * 2.0 * rows),
                 2.0 * a.dnum * rows * c.n * B * S);
    const dim3 grid(c.n / kRTile, level + 1 + c.K, (B + kRItems - 1) / kRItems);
    const TwPair *pmod = (const TwPair *)c.bconv_ptr(c.off_pd_pmod);
    if (MMFHE_D3 && a.dnum == 3)  // PS3 / PS4 / PSV: exact digit count, 5 steps per 128-bit sum
        k_hoisted_rotsum_pq<3><<<grid, kRTile, 0, c.stream>>>(out, x, y, c0, pmod, c.kt, a);
    else if (a.dnum <= 4)
        k_hoisted_rotsum_pq<4><<<grid, kRTile, 0, c.stream>>>(out, x, y, c0, pmod, c.kt, a);
    else
        k_hoisted_rotsum_pq<8><<<grid, kRTile, 0, c.stream>>>(out, x, y, c0, pmod, c.kt, a);
    LAUNCH_CHECK(c);
}

void launch_conj_tensor(Ctx &c, uint64_t *t01, size_t t01s, uint64_t *t2, uint64_t *t3, size_t t23s,
                        const uint64_t *d, size_t ds, uint32_t level, uint32_t B, uint32_t g)
{
    ProfScope ps(c, "tensor_sum", 8.0 * (level + 1) * c.n * B * (2.0 + 4.0), 4.0 * (level + 1) * c.n * B);
    k_conj_tensor<<<grid3(c.n, level + 1, B), kTB, 0, c.stream>>>(t01, t01s, t2, t3, t23s, d, ds, c.kt, level, g);
    LAUNCH_CHECK(c);
}

void launch_pq_lift(Ctx &c, uint64_t *out, size_t os, size_t ops, const uint64_t *src, size_t ss, size_t sps,
                    uint32_t level, uint32_t npoly, uint32_t B, uint32_t g, bool accumulate)
{
    ProfScope ps(c, "pq_lift", 8.0 * npoly * (level + 1) * c.n * B * (accumulate ? 3.0 : 2.0));
    k_pq_lift<<<grid3(c.n, npoly * (level + 1), B), kTB, 0, c.stream>>>(
        out, os, ops, src, ss, sps, (const TwPair *)c.bconv_ptr(c.off_pd_pmod), c.kt, level + 1, g, accumulate ? 1 : 0);
    LAUNCH_CHECK(c);
}

void launch_add_plain(Ctx &c, uint64_t *c0, size_t s, const uint64_t *pt_mont, uint32_t level, uint32_t B)
{
    ProfScope ps(c, "add_plain", 8.0 * (level + 1) * c.n * (1.0 + 2.0 * B));
    k_add_plain<<<grid3(c.n, level + 1, B), kTB, 0, c.stream>>>(c0, s, pt_mont, c.kt);
    LAUNCH_CHECK(c);
}

}  // namespace mmfhe
