// eval.h -- the CKKS evaluator over batches of device ciphertexts (NTT form).
//
// Semantics follow the pinned operations of SURVEY §8(c)-4..6 (exact ring ops,
// round-half-up rescale, hybrid key switching without BConv correction,
// automorphism-first HRot, lazy relinearisation, exact scale bookkeeping).
// Every op works on a batch of B ciphertexts in one set of launches and records
// one logical op per item in the ctx trace (item order).
#pragma once
#include <complex>
#include <string>
#include <utility>
#include <vector>

#include "ops.h"

namespace mmfhe {

DCt make_ct(Ctx &c, uint32_t level, uint32_t npolys, uint32_t n_slots, double scale, uint32_t batch = 1);
DCt view_ct(const Ctx &c, const mmfhe_ct &ct, uint32_t npolys);  // non-owning device NTT-form view
DCt slice(const DCt &a, uint32_t start, uint32_t count);           // non-owning items [start, start+count)
DCt copy_ct(Ctx &c, const DCt &a);

// ABI boundary: coefficient/NTT form, host/device.  import_batch gathers
// cts[first + i*step], i < count, into one contiguous batch.
DCt import_ct(Ctx &c, const mmfhe_ct &in, uint32_t npolys);
DCt import_batch(Ctx &c, const mmfhe_ct *cts, size_t first, size_t step, size_t count);
void export_ct(Ctx &c, const DCt &in, mmfhe_ct &out);  // in.batch == 1
void export_pq(Ctx &c, const DCt &in, mmfhe_ct &out);  // a PQ ciphertext (in.batch == 1), library PQ layout
void export_batch(Ctx &c, const DCt &in, mmfhe_ct *outs);  // outs[0 .. in.batch)

// exact ops (batched)
DCt ev_addsub(Ctx &c, const DCt &a, const DCt &b, bool sub);
DCt ev_drop_to(Ctx &c, const DCt &a, uint32_t level);
DCt ev_tensor_sum(Ctx &c, const std::vector<std::pair<const DCt *, const DCt *>> &pairs);
DCt ev_pmult_sum(Ctx &c, const std::vector<std::pair<const DPlain *, const DCt *>> &terms);
// BSGS inner sums of every giant step in one pass over the baby steps:
// out[o] = sum_c pts[o][c] (.) cts[c] (pts[o][c] may be null); records one pmult_sum per output.
std::vector<DCt> ev_diag_mac(Ctx &c, const std::vector<const DCt *> &cts,
                             const std::vector<std::vector<const DPlain *>> &pts);
// K3's inner sums (re_g = sum_s pc xr_s + pns xi_s, im_g = sum_s ps xr_s + pc xi_s) by Gauss's
// three-product form: the same residues and trace as ev_diag_mac over the four-product rows,
// 3/4 of the MACs.  Output g is one batch of 2B items: re_g's B items, then im_g's.
std::vector<DCt> ev_k3_mac(Ctx &c, const std::vector<const DCt *> &xr, const std::vector<const DCt *> &xi,
                           const std::vector<std::vector<const DPlain *>> &pc,
                           const std::vector<std::vector<const DPlain *>> &ps,
                           const std::vector<std::vector<const DPlain *>> &pns);
// sum of all items of a batch (frame accumulation, depth 0)
DCt ev_batch_sum(Ctx &c, const DCt &a);
// S equal contiguous runs of a's items, each summed: item s of the result = sum of run s
DCt ev_batch_sum_runs(Ctx &c, const DCt &a, uint32_t S);
DCt ev_sum(Ctx &c, const std::vector<const DCt *> &cts);
DCt ev_add_plain(Ctx &c, const DCt &a, const DPlain &pt);
// Scalar linear maps over a batch (CK10): out[j] = sum_{w<W} coef[j][w] in[lo0 + j*lo_step + w]
// (inputs outside [0, M) contribute nothing); coef row-major [J][W]; exact scalar encoding at q_l.
DCt ev_lincomb_mat(Ctx &c, const DCt &in, uint32_t J, uint32_t W, int lo0, int lo_step,
                   const std::vector<double> &coef);

// key switching family (batched)
void ev_keyswitch(Ctx &c, const uint64_t *x_ntt, size_t xs, uint32_t level, uint32_t B, const DKey &key,
                  uint64_t *out, size_t os, const uint64_t *add0, const uint64_t *add1, size_t as);
DCt ev_relin(Ctx &c, const DCt &a3);
DCt ev_rotate(Ctx &c, const DCt &a, int32_t step);  // step MMFHE_STEP_CONJ: records "conj"
// Conj (DESIGN R28): every slot value conjugated (HRot with g = 2N - 1 and the conjugation key)
DCt ev_conjugate(Ctx &c, const DCt &a);
// sum over the m items of each of S sessions (all = [S][m] items) of x (x) x
DCt ev_square_sum_items(Ctx &c, const DCt &all, uint32_t m, uint32_t S);
// Hoisted HRot: one ModUp of c1 shared by every step; per step the
// ModUp'd digits are permuted by sigma_g, then IP + ModDown.  A separate op from
// ev_rotate (different residues, same decryption).
std::vector<DCt> ev_rotate_hoisted(Ctx &c, const DCt &a, const std::vector<int32_t> &steps);
DCt ev_rescale(Ctx &c, const DCt &a);
// a + HRot(a, step) in one key switch (the rotsum step)
DCt ev_rot_add(Ctx &c, const DCt &a, int32_t step);
// a + HRot(b, step) in one key switch (records "hrot" then "hadd")
DCt ev_rot_add(Ctx &c, const DCt &a, const DCt &b, int32_t step);
DCt ev_rotsum(Ctx &c, const DCt &a, uint32_t count, uint32_t stride);

// double-hoisted BSGS (SURVEY §8(c)-5 third op): ciphertexts over Q_l u P (DCt::pk = K)
DCt ev_lift_pq(Ctx &c, const DCt &a);                                                    // (P c0, P c1)
std::vector<DCt> ev_rotate_hoisted_pq(Ctx &c, const DCt &a, const std::vector<int32_t> &steps);  // no ModDown
// lift_pq(a) + sum of ev_rotate_hoisted_pq(a, steps) over Q_l u P in one pass (R27's first level; records
// the lift, the steps and the PQ additions it replaces)
DCt ev_rotsum_hoisted_pq(Ctx &c, const DCt &a, const std::vector<int32_t> &steps);
DCt ev_rotate_pq(Ctx &c, const DCt &a, int32_t step);  // ModDown(a1), sigma_g, key switch kept over Q_l u P
// acc += ev_rotate_pq(a, step), fused (the inner product accumulates into acc); records
// "hrot_pq" then "hadd_pq" per item
void ev_rotate_pq_acc(Ctx &c, DCt &acc, const DCt &a, int32_t step);
DCt ev_moddown_ct(Ctx &c, const DCt &a);               // both polys back to Q_l

// composites
inline DCt ev_relin_rescale(Ctx &c, const DCt &a3) { return ev_rescale(c, ev_relin(c, a3)); }
// DESIGN R31: relinearisation + rescale, and a PQ ciphertext's ModDown + rescale, as ONE division by
// P q_l (records "relin_rescale" / "moddown_rescale")
DCt ev_relin_rescale_merged(Ctx &c, const DCt &a3);
DCt ev_moddown_rescale_ct(Ctx &c, const DCt &a);
// DESIGN R32: d * Conj(d) relinearised with the conjugation and conjugate-product keys and rescaled by
// one division by P q_l (records "conj_mul_relin_rescale")
DCt ev_conj_mul_relin_rescale(Ctx &c, const DCt &d);
inline DCt ev_square_rescale(Ctx &c, const DCt &a) { return ev_relin_rescale(c, ev_tensor_sum(c, {{&a, &a}})); }

uint64_t galois_element(const Ctx &c, int32_t step, int32_t *normalised);
const DKey &find_gk(const Ctx &c, int32_t step_norm);
const DPlain &need_plain(const Ctx &c, const std::string &name, uint32_t level);

// key / plaintext stores
void load_key(Ctx &c, DKey &k, const uint64_t *words, size_t n_words, bool on_device);
// pq: coef holds [level+1+K][N] (q_0..q_level then p_0..p_{K-1}); stored as "name.pq@level"
void load_plain(Ctx &c, const std::string &name, uint32_t level, double scale, const uint64_t *coef,
                bool on_device, bool pq = false);
// host encoder (canonical embedding), csrc/encoder.cpp
std::vector<int64_t> encode_real(const Ctx &c, const std::vector<double> &v, double scale);
// complex slot values (DESIGN R28): the same canonical-embedding encoder, z_j and conj z_j
void encode_plain_c(Ctx &c, const std::string &name, const std::vector<std::complex<double>> &v, uint32_t level,
                    double scale, bool pq = false);
void encode_plain(Ctx &c, const std::string &name, const std::vector<double> &v, uint32_t level, double scale,
                  bool pq = false);
// exact round-half-away(v * q_scale) reduced mod m
uint64_t encode_scalar_mod(double v, uint64_t q_scale, uint64_t m);

}  // namespace mmfhe
