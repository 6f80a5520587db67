// ops.h -- launchers of the RNS polynomial kernels (poly.cu).
//
// All device buffers are limb-major [rows][N].  Batched launchers take B
// items laid out at a fixed item stride (in words); every kernel covers the
// whole batch in one launch so a key, plaintext or twiddle word fetched once
// serves B ciphertexts.
#pragma once
#include "context.h"

namespace mmfhe {

constexpr int kMaxTerms = 64;  // operands per fused-sum launch (chunked above)
constexpr int kDiagMax = 16;   // baby steps / outputs of one fused BSGS diagonal MAC
constexpr int kDiagIn = 32;    // baby steps of the plaintext-stationary (staged) diagonal MAC

struct PtrList {
    const uint64_t *p[kMaxTerms];
};

// out = a (+/-) b over `rows` rows (contiguous); pm maps row -> prime.
void launch_addsub(Ctx &c, uint64_t *out, const uint64_t *a, const uint64_t *b, uint32_t rows, const PrimeMap &pm,
                   bool sub);
// x -> x * 2^64 mod q (Montgomery form), in place.
void launch_to_mont(Ctx &c, uint64_t *x, uint32_t rows, const PrimeMap &pm);
// (The NTT-domain automorphism sigma_g has no kernel of its own: it is a gather fused into
// the INTT's first read (InvSrc), the key inner product and ModDown's addend.)

// ---- hybrid key switching (batched over B polynomials x_b, each [l+1][N])
// ModUp BConv of every digit: x_coef item stride xs; y item stride ys; digit j rows at y + off_j*N.
void launch_modup_bconv(Ctx &c, uint64_t *y, size_t ys, const uint64_t *x_coef, size_t xs, uint32_t level,
                        const std::vector<size_t> &off, uint32_t B);
// accQ [B][2][l+1][N], accP [B][2][K][N] = sum_j y_j (.) evk_j; each key word is loaded once for all B.
// gx / gy: the x (digit-own rows) / y reads go through sigma_g (NTT-domain gather; 1 = none).
// os: output item / poly strides of the Q and P rows (nullptr: compact accQ / accP as above).
struct IPOut {
    size_t qs, qp, ps, pp;
};
// ep: fused epilogue (double hoisting): poly 0 += add (item stride as, Q rows at r N, P rows at
// apbase + k N or none if apbase == ~0), read through sigma_ag, Q-row addends times [P]_{q_r}
// when pmod is set; with accumulate, both polys += the output's previous contents.
struct IPEpi {
    const uint64_t *add = nullptr;
    const uint64_t *add1 = nullptr;  // poly-1 addend on the Q rows, times [P]_{q_r} (R31's relinearisation lift)
    const TwPair *pmod = nullptr;
    size_t as = 0, apbase = ~(size_t)0;
    uint32_t ag = 1;
    int accumulate = 0;
};
void launch_key_ip(Ctx &c, uint64_t *accQ, uint64_t *accP, const uint64_t *x_ntt, size_t xs, const uint64_t *y,
                   size_t ys, const std::vector<size_t> &off, const uint64_t *key, uint32_t level, uint32_t B,
                   uint32_t gx = 1, uint32_t gy = 1, const IPOut *os = nullptr, const IPEpi *ep = nullptr);
// w [B*npoly][l+1][N] = BConv_{P->Q}(zP [B*npoly][K][N]) (coefficient form); with zq ([B*npoly][N], the
// q_l rows) the merged ModDown + rescale's conversion (R31): w [B*npoly][l][N] = BConv_{P u q_l -> Q_{l-1}}.
void launch_moddown_bconv(Ctx &c, uint64_t *w, const uint64_t *zP, uint32_t level, uint32_t B, uint32_t npoly = 2,
                          const uint64_t *zq = nullptr);
// A group of hoisted rotations left over Q_l u P in one launch (double hoisting's baby steps):
// outs[s] (PQ ciphertexts, item stride os) = (P sigma_s(c0) + IP0, IP1) of the digits of x / y
// through sigma_s, with ginv[s] the inverse Galois element of step s and keys[s] its evk.
void launch_hoisted_ip_pq(Ctx &c, const uint64_t *x, size_t xs, const uint64_t *y, size_t ys,
                          const std::vector<size_t> &off, const uint64_t *c0, size_t cs,
                          const std::vector<const uint64_t *> &keys, const std::vector<uint32_t> &ginv,
                          const std::vector<uint64_t *> &outs, size_t os, uint32_t level, uint32_t B);
// Double hoisting's first rotate-and-sum level in one pass: out (PQ ciphertexts, item stride os) =
// (P c0, P c1) + sum_s (P sigma_s(c0) + IP_s,0, IP_s,1), g[s] the Galois element of step s.
void launch_hoisted_rotsum_pq(Ctx &c, uint64_t *out, size_t os, const uint64_t *x, size_t xs, const uint64_t *y,
                              size_t ys, const std::vector<size_t> &off, const uint64_t *c0, size_t cs,
                              const std::vector<const uint64_t *> &keys, const std::vector<uint32_t> &g,
                              uint32_t level, uint32_t B);
// DESIGN R32: t01 (2-poly batch, item stride t01s) = (d0 s(d0), d1 s(d0)); t2 / t3 (single polys, item
// stride t23s) = d0 s(d1) / d1 s(d1); s = sigma_g, a gather in the NTT domain
void launch_conj_tensor(Ctx &c, uint64_t *t01, size_t t01s, uint64_t *t2, uint64_t *t3, size_t t23s,
                        const uint64_t *d, size_t ds, uint32_t level, uint32_t B, uint32_t g);
// double hoisting: Q rows of out (+)= [P]_{q_i} sigma_g(src) for npoly polys per
// item (out / src item strides os / ss, poly strides ops / sps): the identity baby step's P lift
// (the other PQ addends are the key inner product's fused epilogue, IPEpi)
void launch_pq_lift(Ctx &c, uint64_t *out, size_t os, size_t ops, const uint64_t *src, size_t ss, size_t sps,
                    uint32_t level, uint32_t npoly, uint32_t B, uint32_t g, bool accumulate);
// (ModDown's final step (accQ - w) P^{-1} + addends and the rescale's (a_i - v_i) q_l^{-1}
// run as the epilogue of the forward NTT's row pass: ntt_forward(..., RowEpi).)

// ---- fused sums (batched: operand item stride is, output item stride os)
// out (+)= sum_p a_p (x) b_p (3 polys), <= kMaxTerms pairs.
void launch_tensor_sum(Ctx &c, uint64_t *out, size_t os, const PtrList &a, const PtrList &b, size_t is, int n,
                       uint32_t level, bool accumulate, uint32_t B);
// out (+)= sum_t pt_t (.) ct_t; pt shared by the batch (Montgomery form).
void launch_pmult_sum(Ctx &c, uint64_t *out, size_t os, const PtrList &pt, const PtrList &ct, size_t is, int n,
                      uint32_t level, bool accumulate, uint32_t B);
// Fused BSGS inner sums (CK9): out_o (+0) = sum_c pts[o][c] (.) cts[c] for a batch of B
// (cts item stride is, outs item stride os); pts[o][c] may be null; <= kDiagIn inputs, <= kDiagMax outputs.
// pk = K: the operands are PQ ciphertexts / plaintexts (rows over Q_l u P, double hoisting).
void launch_diag_mac(Ctx &c, const std::vector<const uint64_t *> &cts, size_t is,
                     const std::vector<std::vector<const uint64_t *>> &pts, const std::vector<uint64_t *> &outs,
                     size_t os, uint32_t level, uint32_t B, uint32_t pk = 0);
// K3's inner sums with Gauss's three-product complex multiplication (babies xr[s], xi[s];
// plaintexts pc / ps / pns [g][s] (nullptr: no term); outputs re[g], im[g]): equal to the
// four-product sums bit for bit.
void launch_k3_gauss_mac(Ctx &c, const std::vector<const uint64_t *> &xr, const std::vector<const uint64_t *> &xi,
                         size_t is, const std::vector<std::vector<const uint64_t *>> &pc,
                         const std::vector<std::vector<const uint64_t *>> &ps,
                         const std::vector<std::vector<const uint64_t *>> &pns, const std::vector<uint64_t *> &re,
                         const std::vector<uint64_t *> &im, size_t os, uint32_t level, uint32_t B, uint32_t pk);
// Scalar "modular matrix product" over a batch of 2-poly cts (CK10):
//   out[j] = sum_{w < W} C[j][w] in[lo_j + w],  j < J,  lo_j = lo0 + j*lo_step,
// C given as (value, Montgomery form) pairs [J][W][l+1]; inputs outside [0, M) contribute nothing.
void launch_lincomb_mat(Ctx &c, uint64_t *out, const uint64_t *in, uint32_t M, uint32_t J, uint32_t W, int lo0,
                        int lo_step, const TwPair *C, uint32_t level);
// symmetric Toeplitz rows (every row the same taps, c_w == c_{W-1-w}); T: (value, Montgomery form) pairs [W][level+1]
void launch_lincomb_sym(Ctx &c, uint64_t *out, const uint64_t *in, uint32_t M, uint32_t J, uint32_t W, int lo0,
                        const TwPair *T, uint32_t level);
// out = sum_b in_b over a batch of B items of `words` words each (rows of level l).
void launch_batch_sum(Ctx &c, uint64_t *out, const uint64_t *in, uint32_t B, uint32_t npolys, uint32_t level);
// out[b] = copy of src.p[b] (n <= kMaxTerms items of `words` words each; device pointers,
// 16-byte aligned).
void launch_gather(Ctx &c, uint64_t *out, const PtrList &src, int n, size_t words);
// dst.p[b] (written through) = in + b*words, b < n <= kMaxTerms (16-byte aligned destinations).
void launch_scatter(Ctx &c, const PtrList &dst, const uint64_t *in, int n, size_t words);
// c0 of every item (item stride s) += pt (pt in Montgomery form).
void launch_add_plain(Ctx &c, uint64_t *c0, size_t s, const uint64_t *pt_mont, uint32_t level, uint32_t B);

}  // namespace mmfhe
