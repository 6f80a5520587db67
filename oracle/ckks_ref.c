/*
 * oracle/ckks_ref.c -- O-RNS: the plain CPU reference for the RNS-CKKS
 * arithmetic on the mmFHE hot path.  TEST INFRASTRUCTURE ONLY: only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
 * may load this library.  It shares no code, header or table with the CUDA
 * path (paper_2603_22437_b200/csrc).
 *
 * Everything here works on polynomials in COEFFICIENT form, stored limb-major
 * as uint64 arrays [n_limbs][N], one prime per limb.  Arithmetic is the
 * textbook one: (a*b) mod q through unsigned __int128 and '%'; ring products
 * through the textbook iterative negacyclic NTT (psi-twist, bit reversal,
 * radix-2 Cooley-Tukey).  No lazy reduction, no fusion, no precomputed
 * tables shared across calls.  Limbs (and base-conversion targets) are
 * independent residue computations, so their loops are spread over the host's
 * cores with OpenMP (`#pragma omp parallel for`): each limb's arithmetic is
 * exactly the sequential one, only different limbs run at the same time.
 *
 * Citations (PAPER.md line, section) -- the paper names these operations only
 * through its libraries ("RNS-CKKS backends"; HMult/HRot/rescale in the
 * HE primer P:416-421); the exact non-exact steps (rescale rounding, fast base
 * conversion without correction, hybrid key switching) follow the pinned
 * formulas of SURVEY.md §8(c)-5, restated at each function.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef unsigned __int128 u128;

static uint64_t mulmod(uint64_t a, uint64_t b, uint64_t q) { return (uint64_t)(((u128)a * b) % q); }
static uint64_t addmod(uint64_t a, uint64_t b, uint64_t q) { return (uint64_t)(((u128)a + b) % q); }
static uint64_t submod(uint64_t a, uint64_t b, uint64_t q) { return a >= b ? a - b : a + (q - b); }

static uint64_t powmod(uint64_t b, uint64_t e, uint64_t q)
{
    uint64_t r = 1 % q;
    b %= q;
    while (e) {
        if (e & 1) r = mulmod(r, b, q);
        b = mulmod(b, b, q);
        e >>= 1;
    }
    return r;
}

/* inverse by Fermat (q prime) */
static uint64_t invmod(uint64_t a, uint64_t q) { return powmod(a % q, q - 2, q); }

/* A primitive 2N-th root of unity mod q: psi = x^((q-1)/2N) for the smallest
 * x >= 2 with psi^N = -1 (then psi has order exactly 2N). */
uint64_t or_find_psi(uint64_t q, uint32_t n)
{
    uint64_t two_n = 2ull * n;
    if ((q - 1) % two_n) return 0;
    for (uint64_t x = 2; x < 1000000; ++x) {
        uint64_t psi = powmod(x, (q - 1) / two_n, q);
        if (powmod(psi, n, q) == q - 1) return psi;
    }
    return 0;
}

static void bit_reverse_permute(uint64_t *a, uint32_t n)
{
    for (uint32_t i = 1, j = 0; i < n; ++i) {
        uint32_t bit = n >> 1;
        for (; j & bit; bit >>= 1) j ^= bit;
        j ^= bit;
        if (i < j) { uint64_t t = a[i]; a[i] = a[j]; a[j] = t; }
    }
}

/* Cyclic radix-2 DIT transform with root w of order n (after bit reversal). */
static void cyclic_ntt(uint64_t *a, uint32_t n, uint64_t w, uint64_t q)
{
    bit_reverse_permute(a, n);
    for (uint32_t len = 2; len <= n; len <<= 1) {
        uint64_t wlen = powmod(w, n / len, q);
        for (uint32_t i = 0; i < n; i += len) {
            uint64_t wj = 1;
            for (uint32_t j = 0; j < len / 2; ++j) {
                uint64_t u = a[i + j];
                uint64_t v = mulmod(a[i + j + len / 2], wj, q);
                a[i + j] = addmod(u, v, q);
                a[i + j + len / 2] = submod(u, v, q);
                wj = mulmod(wj, wlen, q);
            }
        }
    }
}

/* Negacyclic NTT: A_k = a(psi^(2k+1)), k = 0..N-1 (natural order).
 * Twist a_i *= psi^i, then cyclic NTT with omega = psi^2. */
int or_ntt_forward(uint32_t n, uint64_t q, uint64_t *a)
{
    uint64_t psi = or_find_psi(q, n);
    if (!psi) return -1;
    uint64_t pw = 1;
    for (uint32_t i = 0; i < n; ++i) { a[i] = mulmod(a[i] % q, pw, q); pw = mulmod(pw, psi, q); }
    cyclic_ntt(a, n, mulmod(psi, psi, q), q);
    return 0;
}

/* Inverse of or_ntt_forward: cyclic inverse with omega^-1, times N^-1, untwist by psi^-i. */
int or_ntt_inverse(uint32_t n, uint64_t q, uint64_t *a)
{
    uint64_t psi = or_find_psi(q, n);
    if (!psi) return -1;
    uint64_t psi_inv = invmod(psi, q);
    cyclic_ntt(a, n, mulmod(psi_inv, psi_inv, q), q);
    uint64_t n_inv = invmod(n, q);
    uint64_t pw = n_inv;
    for (uint32_t i = 0; i < n; ++i) { a[i] = mulmod(a[i], pw, q); pw = mulmod(pw, psi_inv, q); }
    return 0;
}

/* out = a*b in Z_q[X]/(X^N+1), per limb: NTT, pointwise product, INTT. */
int or_poly_mul(uint32_t n, uint32_t n_limbs, const uint64_t *qs,
                const uint64_t *a, const uint64_t *b, uint64_t *out)
{
    int rc = 0;
#pragma omp parallel for schedule(dynamic, 1) reduction(| : rc)
    for (uint32_t l = 0; l < n_limbs; ++l) {
        uint64_t *ta = (uint64_t *)malloc(sizeof(uint64_t) * n);
        uint64_t *tb = (uint64_t *)malloc(sizeof(uint64_t) * n);
        uint64_t q = qs[l];
        memcpy(ta, a + (size_t)l * n, sizeof(uint64_t) * n);
        memcpy(tb, b + (size_t)l * n, sizeof(uint64_t) * n);
        rc |= or_ntt_forward(n, q, ta);
        rc |= or_ntt_forward(n, q, tb);
        for (uint32_t i = 0; i < n; ++i) ta[i] = mulmod(ta[i], tb[i], q);
        rc |= or_ntt_inverse(n, q, ta);
        memcpy(out + (size_t)l * n, ta, sizeof(uint64_t) * n);
        free(ta);
        free(tb);
    }
    return rc;
}

void or_add(uint32_t n, uint32_t n_limbs, const uint64_t *qs, const uint64_t *a, const uint64_t *b, uint64_t *out)
{
#pragma omp parallel for
    for (uint32_t l = 0; l < n_limbs; ++l)
        for (uint32_t i = 0; i < n; ++i) {
            size_t k = (size_t)l * n + i;
            out[k] = addmod(a[k], b[k], qs[l]);
        }
}

void or_sub(uint32_t n, uint32_t n_limbs, const uint64_t *qs, const uint64_t *a, const uint64_t *b, uint64_t *out)
{
#pragma omp parallel for
    for (uint32_t l = 0; l < n_limbs; ++l)
        for (uint32_t i = 0; i < n; ++i) {
            size_t k = (size_t)l * n + i;
            out[k] = submod(a[k], b[k], qs[l]);
        }
}

/* out_l = a_l * c_l mod q_l for one scalar residue c_l per limb. */
void or_scalar_mul(uint32_t n, uint32_t n_limbs, const uint64_t *qs, const uint64_t *a, const uint64_t *c, uint64_t *out)
{
#pragma omp parallel for
    for (uint32_t l = 0; l < n_limbs; ++l)
        for (uint32_t i = 0; i < n; ++i) {
            size_t k = (size_t)l * n + i;
            out[k] = mulmod(a[k], c[l], qs[l]);
        }
}

/* Galois automorphism sigma_g: a(X) -> a(X^g), g odd.  Coefficient i moves to
 * i*g mod 2N, negated when that lands in [N, 2N) because X^N = -1
 * (SURVEY §8(c)-4). */
void or_automorphism(uint32_t n, uint32_t n_limbs, const uint64_t *qs, const uint64_t *a, uint64_t g, uint64_t *out)
{
    uint64_t two_n = 2ull * n;
#pragma omp parallel for
    for (uint32_t l = 0; l < n_limbs; ++l) {
        const uint64_t *al = a + (size_t)l * n;
        uint64_t *ol = out + (size_t)l * n;
        for (uint32_t i = 0; i < n; ++i) {
            uint64_t j = ((uint64_t)i * g) % two_n;
            if (j < n) ol[j] = al[i];
            else ol[j - n] = submod(0, al[i], qs[l]);
        }
    }
}

/* Rescale by the last prime q_l (SURVEY §8(c)-5, round-half-up):
 *   h = floor(q_l/2),  t = [a_l + h]_{q_l},
 *   a'_i = (a_i + h - t) * q_l^{-1} mod q_i   for i < l.
 * a has l+1 limbs (q_0..q_l); out has l limbs. */
void or_rescale(uint32_t n, uint32_t l, const uint64_t *qs, const uint64_t *a, uint64_t *out)
{
    uint64_t ql = qs[l];
    uint64_t h = ql >> 1;
    const uint64_t *al = a + (size_t)l * n;
#pragma omp parallel for
    for (uint32_t i = 0; i < l; ++i) {
        uint64_t qi = qs[i];
        uint64_t ql_inv = invmod(ql % qi, qi);
        for (uint32_t k = 0; k < n; ++k) {
            uint64_t t = addmod(al[k], h, ql);
            uint64_t v = addmod(a[(size_t)i * n + k], h % qi, qi);
            v = submod(v, t % qi, qi);
            out[(size_t)i * n + k] = mulmod(v, ql_inv, qi);
        }
    }
}

/* Product of the primes mod m: prod_{i in S} s_i mod m. */
static uint64_t prod_mod(const uint64_t *s, uint32_t cnt, uint64_t m)
{
    uint64_t r = 1 % m;
    for (uint32_t i = 0; i < cnt; ++i) r = mulmod(r, s[i] % m, m);
    return r;
}

/* Fast base conversion (no correction) of x given mod the primes src[0..ns)
 * into each target prime t:
 *   y_t = sum_i [x_i * [S_hat_i^{-1}]_{s_i}]_{s_i} * [S_hat_i]_t  mod t,
 * S_hat_i = S / s_i.  (SURVEY §8(c)-5 ModUp / ModDown.) */
static void bconv(uint32_t n, const uint64_t *src, uint32_t ns, const uint64_t *x,
                  const uint64_t *dst, uint32_t nd, uint64_t *y)
{
    uint64_t *hat_inv = (uint64_t *)malloc(sizeof(uint64_t) * ns);
    uint64_t *others = (uint64_t *)malloc(sizeof(uint64_t) * (ns ? ns : 1));
    for (uint32_t i = 0; i < ns; ++i) {
        uint32_t c = 0;
        for (uint32_t k = 0; k < ns; ++k) if (k != i) others[c++] = src[k];
        hat_inv[i] = invmod(prod_mod(others, c, src[i]), src[i]);
    }
    free(others);
#pragma omp parallel for schedule(dynamic, 1)
    for (uint32_t d = 0; d < nd; ++d) {
        uint64_t *hat_t = (uint64_t *)malloc(sizeof(uint64_t) * ns);
        uint64_t *others = (uint64_t *)malloc(sizeof(uint64_t) * (ns ? ns : 1));
        uint64_t t = dst[d];
        for (uint32_t i = 0; i < ns; ++i) {
            uint32_t c = 0;
            for (uint32_t k = 0; k < ns; ++k) if (k != i) others[c++] = src[k];
            hat_t[i] = prod_mod(others, c, t);
        }
        for (uint32_t k = 0; k < n; ++k) {
            uint64_t acc = 0;
            for (uint32_t i = 0; i < ns; ++i) {
                uint64_t v = mulmod(x[(size_t)i * n + k], hat_inv[i], src[i]);
                acc = addmod(acc, mulmod(v % t, hat_t[i], t), t);
            }
            y[(size_t)d * n + k] = acc;
        }
        free(hat_t);
        free(others);
    }
    free(hat_inv);
}

/* ModUp of digit j at level l:
 * I_j = {j*alpha .. min(j*alpha+alpha, l+1)-1}.  Output basis is
 * q_0..q_l, p_0..p_{K-1} ([l+1+K][N]): limbs t in I_j copy x_t, every other
 * limb is the fast BConv of x restricted to I_j. */
void or_modup(uint32_t n, uint32_t l, const uint64_t *qs, uint32_t k_p, const uint64_t *ps,
              uint32_t alpha, uint32_t j, const uint64_t *x, uint64_t *out)
{
    uint32_t lo = j * alpha, hi = lo + alpha;
    if (hi > l + 1) hi = l + 1;
    uint32_t ns = hi - lo;
    uint32_t nb = l + 1 + k_p;
#pragma omp parallel for schedule(dynamic, 1)
    for (uint32_t t = 0; t < nb; ++t) {
        uint64_t pt = t <= l ? qs[t] : ps[t - l - 1];
        uint64_t *yt = out + (size_t)t * n;
        if (t >= lo && t < hi) {
            memcpy(yt, x + (size_t)t * n, sizeof(uint64_t) * n);
        } else {
            bconv(n, qs + lo, ns, x + (size_t)lo * n, &pt, 1, yt);
        }
    }
}

/* ModDown: c' over q_0..q_l, p_0..p_{K-1} ([l+1+K][N]):
 *   w_i = BConv_{P -> q_i}(c'_P),  out_i = (c'_i - w_i) * [P^{-1}]_{q_i}. */
void or_moddown(uint32_t n, uint32_t l, const uint64_t *qs, uint32_t k_p, const uint64_t *ps,
                const uint64_t *c, uint64_t *out)
{
    uint64_t *w = (uint64_t *)malloc(sizeof(uint64_t) * (size_t)(l + 1) * n);
    bconv(n, ps, k_p, c + (size_t)(l + 1) * n, qs, l + 1, w);
#pragma omp parallel for
    for (uint32_t i = 0; i <= l; ++i) {
        uint64_t qi = qs[i];
        uint64_t p_inv = invmod(prod_mod(ps, k_p, qi), qi);
        for (uint32_t k = 0; k < n; ++k) {
            size_t idx = (size_t)i * n + k;
            out[idx] = mulmod(submod(c[idx], w[idx], qi), p_inv, qi);
        }
    }
    free(w);
}

/* ModDown and rescale as ONE division (reading R31): c over q_0..q_l, p_0..p_{K-1} (coefficient form,
 * layout [l+1+K][N]: q rows then p rows) -> out over q_0..q_{l-1}:
 *   w = BConv_{p_0..p_{K-1}, q_l -> q_i}(c)  (fast base conversion, the sources' residues),
 *   out_i = (c_i - w_i) (P q_l)^{-1} mod q_i,  i < l.
 * (ModDown's formula with the special modulus P q_l: q_l is converted like a special prime.) */
void or_moddown_rescale(uint32_t n, uint32_t l, const uint64_t *qs, uint32_t k_p, const uint64_t *ps,
                        const uint64_t *c, uint64_t *out)
{
    uint32_t ns = k_p + 1;
    uint64_t *src = (uint64_t *)malloc(sizeof(uint64_t) * ns);
    uint64_t *x = (uint64_t *)malloc(sizeof(uint64_t) * (size_t)ns * n);
    uint64_t *w = (uint64_t *)malloc(sizeof(uint64_t) * (size_t)(l ? l : 1) * n);
    for (uint32_t k = 0; k < k_p; ++k) src[k] = ps[k];
    src[k_p] = qs[l];
    memcpy(x, c + (size_t)(l + 1) * n, sizeof(uint64_t) * (size_t)k_p * n);
    memcpy(x + (size_t)k_p * n, c + (size_t)l * n, sizeof(uint64_t) * n);
    bconv(n, src, ns, x, qs, l, w);
#pragma omp parallel for
    for (uint32_t i = 0; i < l; ++i) {
        uint64_t qi = qs[i];
        uint64_t m_inv = invmod(mulmod(prod_mod(ps, k_p, qi), qs[l] % qi, qi), qi);
        for (uint32_t k = 0; k < n; ++k) {
            size_t idx = (size_t)i * n + k;
            out[idx] = mulmod(submod(c[idx], w[idx], qi), m_inv, qi);
        }
    }
    free(src);
    free(x);
    free(w);
}

/* Hybrid key switching of x (coefficient form, level l) with the key
 *   evk[j] = (b_j, a_j),  j < dnum_L,  each over q_0..q_L, p_0..p_{K-1}
 * (layout [dnum_L][2][L+1+K][N]).  At level l the limbs q_{l+1..L} of the key
 * are dropped and dnum_l = ceil((l+1)/alpha) digits are used:
 *   y_j = ModUp_j(x);  c'_0 = sum_j y_j * b_j,  c'_1 = sum_j y_j * a_j  (over Q_l u P);
 *   (d0, d1) = (ModDown(c'_0), ModDown(c'_1)).
 * (SURVEY §8(c)-5 "Inner product", "ModDown".) */
int or_keyswitch(uint32_t n, uint32_t l, uint32_t big_l, const uint64_t *qs, uint32_t k_p,
                 const uint64_t *ps, uint32_t alpha, const uint64_t *x, const uint64_t *evk,
                 uint64_t *d0, uint64_t *d1)
{
    uint32_t nb = l + 1 + k_p;
    uint32_t nkey = big_l + 1 + k_p;
    uint32_t dnum = (l + 1 + alpha - 1) / alpha;
    uint64_t *basis = (uint64_t *)malloc(sizeof(uint64_t) * nb);
    for (uint32_t t = 0; t < nb; ++t) basis[t] = t <= l ? qs[t] : ps[t - l - 1];
    size_t pn = (size_t)nb * n;
    uint64_t *y = (uint64_t *)malloc(sizeof(uint64_t) * pn);
    uint64_t *kb = (uint64_t *)malloc(sizeof(uint64_t) * pn);
    uint64_t *ka = (uint64_t *)malloc(sizeof(uint64_t) * pn);
    uint64_t *acc0 = (uint64_t *)calloc(pn, sizeof(uint64_t));
    uint64_t *acc1 = (uint64_t *)calloc(pn, sizeof(uint64_t));
    uint64_t *prod = (uint64_t *)malloc(sizeof(uint64_t) * pn);
    int rc = 0;
    for (uint32_t j = 0; j < dnum; ++j) {
        or_modup(n, l, qs, k_p, ps, alpha, j, x, y);
        const uint64_t *bj = evk + ((size_t)j * 2 + 0) * nkey * n;
        const uint64_t *aj = evk + ((size_t)j * 2 + 1) * nkey * n;
        /* restrict the key to q_0..q_l, p_0..p_{K-1} */
        memcpy(kb, bj, sizeof(uint64_t) * (size_t)(l + 1) * n);
        memcpy(kb + (size_t)(l + 1) * n, bj + (size_t)(big_l + 1) * n, sizeof(uint64_t) * (size_t)k_p * n);
        memcpy(ka, aj, sizeof(uint64_t) * (size_t)(l + 1) * n);
        memcpy(ka + (size_t)(l + 1) * n, aj + (size_t)(big_l + 1) * n, sizeof(uint64_t) * (size_t)k_p * n);
        rc |= or_poly_mul(n, nb, basis, y, kb, prod);
        or_add(n, nb, basis, acc0, prod, acc0);
        rc |= or_poly_mul(n, nb, basis, y, ka, prod);
        or_add(n, nb, basis, acc1, prod, acc1);
    }
    or_moddown(n, l, qs, k_p, ps, acc0, d0);
    or_moddown(n, l, qs, k_p, ps, acc1, d1);
    free(basis); free(y); free(kb); free(ka); free(acc0); free(acc1); free(prod);
    return rc;
}
