// ops.h -- launchers of the RNS polynomial kernels (poly.cu).  All device
// buffers are limb-major [rows][N]; "pm" maps a row to its prime.
#pragma once
#include "context.h"

namespace mmfhe {

constexpr int kMaxTerms = 64;  // operands per fused-sum launch (chunked above)

struct PtrList {
    const uint64_t *p[kMaxTerms];
};

// out = a + b (sub=false) or a - b (sub=true), rows x N words.
void launch_addsub(Ctx &c, uint64_t *out, const uint64_t *a, const uint64_t *b, uint32_t rows, const PrimeMap &pm,
                   bool sub);
// x -> x * 2^64 mod q (Montgomery form), in place.
void launch_to_mont(Ctx &c, uint64_t *x, uint32_t rows, const PrimeMap &pm);
// NTT-domain automorphism sigma_g: out[j] = in[perm_g(j)] (all rows).
void launch_automorph(Ctx &c, uint64_t *out, const uint64_t *in, uint32_t rows, uint64_t g);
// ModUp base conversion of all digits at `level` from coefficient-form x [level+1][N] into
// y (digit j's n_tgt rows at y + off_j*N, coefficient form).
void launch_modup_bconv(Ctx &c, uint64_t *y, const uint64_t *x_coef, uint32_t level, const std::vector<size_t> &off);
// Key inner product: accQ [2][l+1][N], accP [2][K][N] = sum_j y_j (.) evk_j (Montgomery MAC).
void launch_key_ip(Ctx &c, uint64_t *accQ, uint64_t *accP, const uint64_t *x_ntt, const uint64_t *y,
                   const std::vector<size_t> &off, const uint64_t *key, uint32_t level);
// ModDown base conversion: w [2][l+1][N] = BConv_{P->Q}(zP [2][K][N], coefficient form).
void launch_moddown_bconv(Ctx &c, uint64_t *w, const uint64_t *zP, uint32_t level);
// out_p = (accQ_p - w_p) * P^{-1} (+ addend_p if given), p = 0, 1; NTT form.
void launch_moddown_final(Ctx &c, uint64_t *out0, uint64_t *out1, const uint64_t *accQ, const uint64_t *w,
                          const uint64_t *add0, const uint64_t *add1, uint32_t level);
// Rescale helper: v [2][l][N] = (t - h) mod q_i from t [2][N] (coefficient form mod q_l).
void launch_rescale_prep(Ctx &c, uint64_t *v, const uint64_t *t, uint32_t level);
// out [2][l][N] = (a_i - v_i) * q_l^{-1} mod q_i from a [2][l+1][N] (NTT form).
void launch_rescale_final(Ctx &c, uint64_t *out, const uint64_t *a, const uint64_t *v, uint32_t level);
// Fused tensor sum over <= kMaxTerms pairs: out [3][l+1][N] (+)= sum_p a_p (x) b_p.
void launch_tensor_sum(Ctx &c, uint64_t *out, const PtrList &a, const PtrList &b, int n, uint32_t level,
                       bool accumulate);
// out [2][l+1][N] (+)= sum_t pt_t (.) ct_t, pt in Montgomery form [l+1][N].
void launch_pmult_sum(Ctx &c, uint64_t *out, const PtrList &pt, const PtrList &ct, int n, uint32_t level,
                      bool accumulate);
// out [2][l+1][N] (+)= sum_t c_t ct_t with scalar constants consts[t][l+1] (Shoup pairs).
void launch_lincomb(Ctx &c, uint64_t *out, const PtrList &ct, const TwPair *consts, int n, uint32_t level,
                    bool accumulate);
// c0 [l+1][N] += pt (pt in Montgomery form).
void launch_add_plain(Ctx &c, uint64_t *c0, const uint64_t *pt_mont, uint32_t level);

}  // namespace mmfhe
