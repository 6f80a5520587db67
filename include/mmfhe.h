/*
 * mmfhe.h -- C-ABI of the B200-native mmFHE cloud-side library.
 *
 * The library evaluates the mmFHE kernel chains (PAPER.md §"Cloud-Side
 * Algorithms") over RNS-CKKS ciphertexts on one CUDA device.  It
 * follows the paper's problem statement: the cloud "receives ciphertexts and
 * public parameters", "selects and chains kernels ... according to the target
 * application" and "returns the encrypted result", holding
 * only the evaluation keys (rlk, gk; sk "never leaves the client").
 * The library therefore never takes a secret key, never decrypts and draws no
 * randomness: every call is a deterministic function of its inputs.
 *
 * Conventions (all entry points)
 *   - Every call returns mmfhe_status; nothing throws across the ABI.
 *     On error, mmfhe_last_error(ctx) holds a one-line message.
 *   - Polynomials are RNS residues, uint64 little-endian, limb-major:
 *     a ciphertext at level l is [2][l+1][N] (N = 2^log_n), residue of limb i
 *     modulo q_i, each in [0, q_i).
 *   - form = MMFHE_FORM_COEFF (0): coefficient representation -- the interchange
 *     format, identical to the client's.  form = MMFHE_FORM_EVAL (1): the
 *     library's internal NTT (evaluation) representation; its ordering is
 *     private (bit-reversed), only valid between calls of the same library.
 *   - on_device != 0: data is a CUDA device pointer on the ctx device (e.g. a
 *     torch tensor's data_ptr()); otherwise a host pointer (copies are done on
 *     the ctx stream, pinned host memory recommended).
 *   - Ciphertext buffers are CALLER-OWNED (inputs and outputs).  Keys and
 *     plaintext operands are copied into library-owned device memory and are
 *     freed by mmfhe_ctx_destroy.
 *   - Calls are asynchronous on the ctx stream (the one passed to
 *     mmfhe_ctx_create) unless stated; device outputs are valid after the
 *     caller synchronises that stream.  Host outputs are synchronous.
 *   - A ctx is not thread-safe; use one ctx per GPU / rank.
 *
 * Errors: depth exhausted -> MMFHE_E_DEPTH; missing Galois key
 * -> MMFHE_E_MISSING_KEY; layout/capacity -> MMFHE_E_LAYOUT; scale mismatch ->
 * MMFHE_E_SCALE; frame count / dimension mismatch -> MMFHE_E_SHAPE; unknown
 * plaintext operand -> MMFHE_E_MISSING_PLAIN.
 */
#ifndef MMFHE_H
#define MMFHE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    MMFHE_OK = 0,
    MMFHE_E_INVALID_ARG = 1,
    MMFHE_E_PARAMS = 2,
    MMFHE_E_DEPTH = 3,
    MMFHE_E_MISSING_KEY = 4,
    MMFHE_E_LAYOUT = 5,
    MMFHE_E_SCALE = 6,
    MMFHE_E_SHAPE = 7,
    MMFHE_E_CUDA = 8,
    MMFHE_E_OOM = 9,
    MMFHE_E_NCCL = 10,
    MMFHE_E_FORMAT = 11,
    MMFHE_E_MISSING_PLAIN = 12
} mmfhe_status;

enum { MMFHE_FORM_COEFF = 0, MMFHE_FORM_EVAL = 1 };

typedef struct mmfhe_ctx mmfhe_ctx; /* opaque */

/* CKKS parameters (P:433-454 Table tab:ckks_params; primes explicit).
 *   q[0..n_q)  : ciphertext modulus chain q_0..q_L (L = n_q - 1), each prime,
 *                = 1 mod 2N, < 2^60;
 *   p[0..n_p)  : special primes P = p_0...p_{K-1} of hybrid key switching;
 *   alpha      : limbs per key-switching digit, dnum(l) = ceil((l+1)/alpha);
 *   scale_bits : Delta = 2^scale_bits for fresh encodings. */
typedef struct {
    uint32_t log_n;
    uint32_t n_q;
    const uint64_t *q;
    uint32_t n_p;
    const uint64_t *p;
    uint32_t alpha;
    uint32_t scale_bits;
    uint32_t security; /* informational (e.g. 128) */
} mmfhe_params;

/* A ciphertext (or plaintext when n_polys == 1).  data points at
 * [n_polys][level+1][N] uint64; n_slots is the packing period n. */
typedef struct {
    uint32_t log_n;
    uint32_t level;
    uint32_t n_slots;
    uint32_t form;
    double scale;
    uint64_t *data;
    int32_t on_device;
    uint32_t n_polys; /* 2 for ciphertexts (0 is read as 2), 1 for plaintexts */
} mmfhe_ct;

/* Public chain parameters (R, D, A, F, gamma, P_phi,
 * Taylor order, filter taps, FC dims are public). */
typedef struct {
    uint32_t R, D, A, F;
    uint32_t gamma;        /* K2 sharpening exponent, power of two */
    uint32_t p_phi;        /* K4 mask exponent, power of two */
    uint32_t taylor_order; /* K7: 1 or 3 */
    uint32_t n_slots;      /* packing period n */
    uint32_t bsgs_baby;    /* K3 baby steps b (0: ceil(sqrt(2D-1))) */
    uint32_t hoist;        /* 1: rotations of one ciphertext by several amounts share one ModUp
                              (hoisted HRot: K3 / FC baby steps, K4's packed unpack);
                              2: double-hoisted BSGS for K3 and FC (baby steps kept over Q_l u P, diagonals
                              encoded over Q_l u P, each giant step ModDowns only its inner sum's c1 and
                              keeps its key switch over Q_l u P, one ModDown per output; K4's unpack as 1);
                              0: every rotation is a full HRot.  Different residues, same decryption */
    uint32_t frame_batch;  /* frames evaluated together per batched launch (0: all);
                              fixes the op order of the trace (op-major per batch) */
    uint32_t fc_dims[4];   /* n_in, h1, h2, h3 (padded logits) */
    uint32_t notch_width;  /* K6 zeroed bins around D/2 */
    uint32_t n_bands;      /* vital V2: number of FIR bands (<= 4) */
    uint32_t n_taps[4];    /* vital V2: taps per band (scalars "k5.b<i>") */
    uint32_t n_bins[4];    /* vital V2: narrowband DFT bins per band */
    uint32_t bins[4][64];  /* vital V2: bin indices k per band */
    double fs;             /* frame rate (Hz) */
    uint32_t vp_plus;      /* vital V2: 1 = sharpen P_k^2 and weighted frequency average in the cloud
                              (VP+): per band two outputs N_f = sum_k f_k P_k^2 and
                              D_f = sum_k P_k^2 (f_k = k fs / (F-1) Hz; the client reads
                              BPM = 60 N_f / D_f); depth +2.  0 = outputs P_k (client finishes) */
    uint32_t iq_pack;      /* vital V2 / K4: k >= 1 = i, q of 2^(k-1) frames packed into the slot
                              blocks of one ciphertext, one rotate-and-sum, unpacked (DESIGN R19):
                              per frame 2(2 - 2^(1-k)) + log2(R)/2^(k-1) rotations instead of
                              2 log2 R; needs 2^k R <= n, a multiple of 2^(k-1) frames per frame
                              batch (E_SHAPE) and the Galois keys for +-2^j R, j < k (listed by
                              mmfhe_chain_required_rotations); same decryption.  0 = canonical */
    uint32_t lanes;        /* gesture / k3 / K2b / K6 / FC chains: L = frames interleaved per ciphertext
                              (SIMD-dense packing, DESIGN R20); 0 or 1 = one frame per
                              ciphertext (the paper's layout).  Slot L*i + f holds element i of
                              frame f: every rotation amount is scaled by L, public vectors are
                              lane-repeated, frames' features are lane-summed at the start of the FC
                              head, logits sit in slots L*c.  Inputs: ceil(F/L) ciphertext pairs
                              (n_slots = L*n; unused lanes of the last pair zero); frame_batch then
                              counts ciphertext pairs.  L a power of two with L*n <= N/2 (E_SHAPE) */
    uint32_t fc_baby;      /* FC layers' BSGS baby steps b: min(fc_baby, h) (0: ceil(sqrt(h))) */
    uint32_t cplx;         /* gesture / k3_doppler_dft chains: 1 = complex slots (DESIGN R28, SURVEY
                              §8(f)-3): each input ciphertext carries z = v_re + j v_im (complex slot
                              values; the paper splits re and im into two ciphertexts), so
                              inputs are ONE ciphertext per frame (group): ceil(F/L) for chain gesture.
                              K3 multiplies complex diagonals of W (Eq. dft_kernel) -- one product per
                              diagonal instead of four -- and outputs d = d_re + j d_im; K1 computes
                              |d|^2 = d Conj(d) with the conjugation key (MMFHE_STEP_CONJ, listed by
                              mmfhe_chain_required_rotations).  Same depth; 0 = split re/im layout */
    uint32_t bsgs_aligned; /* K3 BSGS: 1 = giant offsets at multiples of b (G = b k, k = floor(-(D-1)/b) ..
                              floor((D-1)/b)), so the giant G = 0 needs no rotation (DESIGN R29; one giant
                              key switch fewer per input); 0 = the SURVEY §8(c)-7 split o = -(D-1) + g'b + s.
                              Different rotation keys and residues, same decryption */
    uint32_t rotsum_inner; /* hoist = 2: size a of every rotate-and-sum's double-hoisted first level (DESIGN
                              R27): one ModUp, a - 1 PQ steps summed in one pass, one ModDown, then log2(count/a)
                              rotate-and-add steps; a power of two <= 64 (0 = 8).  Its Galois keys j*stride,
                              j < a, are listed by mmfhe_chain_required_rotations; same decryption */
    uint32_t rotsum_hoist_all; /* hoist = 2: 1 = EVERY level of a rotate-and-sum double-hoisted (DESIGN R30):
                              levels of min(rotsum_inner, what is left) terms, each one ModUp + one-pass PQ
                              steps + one ModDown, no plain rotate-and-add key switches; 0 = R27 (first
                              level hoisted, then rotate-and-adds).  Same decryption */
    uint32_t ks_merge;     /* gesture / K3 / FC / vital V1, V2 chains: 1 = every relinearisation or double-hoisted ModDown that a
                              rescale follows runs as ONE division by P q_l (DESIGN R31: fast base conversion
                              from p_0..p_{K-1}, q_l, one forward NTT of the q_0..q_{l-1} rows fewer); records
                              "relin_rescale" / "moddown_rescale".  Other residues, same decryption */
    uint32_t k1_conj_fuse; /* cplx = 1 with ks_merge = 1: K1's d Conj(d) as ONE key switch (DESIGN R32): the inner
                              products of ModUp(d0 sigma(d1)) with the conjugation key and of ModUp(d1 sigma(d1))
                              with the conjugate-product key (MMFHE_STEP_CONJ_PROD, listed by
                              mmfhe_chain_required_rotations) share one division by P q_l; records
                              "conj_mul_relin_rescale".  Same decryption */
    uint32_t sessions;     /* gesture_features only: 0 / 1 = one session; S >= 2 = the inputs are S equal
                              contiguous runs (one per session, each the chain's usual input list), run
                              as ONE batch through the per-frame chain, one feature ciphertext per
                              session out (each the modular sum of its own frames: the residues of S
                              separate calls).  Needs frame_batch 0 (or >= the groups of all sessions) */
} mmfhe_chain_cfg;

/* ---- context ------------------------------------------------------------ */

/* Create a context on cuda_device using cuda_stream (a cudaStream_t, may be
 * NULL for the legacy default stream).  Precomputes NTT, base-conversion and
 * rescale tables for every prime.  MMFHE_E_PARAMS if a prime is not = 1 mod
 * 2N, not < 2^60, duplicated, or alpha/log_n out of range. */
mmfhe_status mmfhe_ctx_create(const mmfhe_params *params, int cuda_device, void *cuda_stream,
                              mmfhe_ctx **out);
mmfhe_status mmfhe_ctx_destroy(mmfhe_ctx *ctx);
const char *mmfhe_last_error(const mmfhe_ctx *ctx);
/* Bytes of device memory currently held by the ctx (keys, plains, pool). */
mmfhe_status mmfhe_ctx_memory(mmfhe_ctx *ctx, size_t *bytes);
/* Number of CUDA kernels this ctx has launched so far. */
mmfhe_status mmfhe_launch_count(mmfhe_ctx *ctx, uint64_t *count);

/* ---- keys ------------------------------------------------------- */

/* Rotation amounts (normalised to [0, N/2)) the chain needs; tells the
 * client which Galois keys to generate (SURVEY §8(d) key table).  Writes at
 * most cap entries, *n = total count (MMFHE_E_LAYOUT if cap too small). */
mmfhe_status mmfhe_chain_required_rotations(mmfhe_ctx *ctx, const char *chain, const mmfhe_chain_cfg *cfg,
                                            int32_t *steps, size_t cap, size_t *n);

/* Key id of the complex conjugation automorphism X -> X^(2N-1) (DESIGN R28): pass it as the
 * step of mmfhe_load_galois_key / mmfhe_client_keygen / mmfhe_serialize_key (and of the
 * HRot primitive, which then conjugates every slot).  It lies outside every normalised
 * rotation amount [0, N/2).  Its key is the key for sigma_{2N-1}(s); client keygen draws it
 * from PRNG key index 1 + N/2 (rotation k uses 1 + k). */
#define MMFHE_STEP_CONJ ((int32_t)(-2147483647 - 1))
/* Key id of the conjugate-product key (DESIGN R32): the key switching s * sigma_{2N-1}(s) to s, with
 * which K1's d * Conj(d) is relinearised in one step (cfg.k1_conj_fuse); client keygen draws it from
 * PRNG key index 2 + N/2.  Not a Galois key: the HRot primitive rejects it. */
#define MMFHE_STEP_CONJ_PROD ((int32_t)(-2147483647))

/* Evaluation keys in coefficient form, layout [dnum_L][2][L+1+K][N]
 * (b_j then a_j, limbs q_0..q_L then p_0..p_{K-1}); n_words must equal
 * dnum_L*2*(L+1+K)*N.  Relinearisation key = key for s^2; Galois key for
 * step k = key for sigma_g(s), g = 5^(k mod N/2) mod 2N.  Host or device
 * pointer (on_device). */
mmfhe_status mmfhe_load_relin_key(mmfhe_ctx *ctx, const uint64_t *words, size_t n_words, int on_device);
mmfhe_status mmfhe_load_galois_key(mmfhe_ctx *ctx, int32_t step, const uint64_t *words, size_t n_words,
                                   int on_device);

/* ---- public plaintext operands ------------------------------- */

/* Import a pre-encoded plaintext (n_polys = 1, form COEFF) under (name, level).
 * pt->scale is its scale (q_level for multiplicative operands). */
mmfhe_status mmfhe_load_plain(mmfhe_ctx *ctx, const char *name, const mmfhe_ct *pt);
/* The same for a plaintext over Q_level u P (double-hoisted BSGS diagonals):
 * pt->data holds [level+1+K][N] (q_0..q_level, then p_0..p_{K-1}); stored as "<name>.pq". */
mmfhe_status mmfhe_load_plain_pq(mmfhe_ctx *ctx, const char *name, const mmfhe_ct *pt);
/* Encode v[0..n) (period n, replicated to N/2 slots) at (level, scale) with the
 * library's own canonical-embedding encoder and store it under (name, level). */
mmfhe_status mmfhe_encode_plain(mmfhe_ctx *ctx, const char *name, const double *v, size_t n, uint32_t level,
                                double scale);
/* Encode every public operand a chain needs (K2 ramps, K3 diagonals, K6 mask,
 * FC diagonals and biases from fc weights, FIR taps, DFT coefficients) at the
 * levels the chain uses them, starting from entry level in_level.
 *   fc_w / fc_b: row-major weights of the FC layers (may be NULL for non-FC chains),
 *   fc_w[i] is fc_dims[i+1] x fc_dims[i] (rows beyond n_classes zero-padded by caller),
 *   taps[b]: FIR taps of band b (may be NULL for non-V2 chains). */
mmfhe_status mmfhe_prepare_chain(mmfhe_ctx *ctx, const char *chain, const mmfhe_chain_cfg *cfg, uint32_t in_level,
                                 const double *const *fc_w, const double *const *fc_b, const double *const *taps);
/* Scalar constants used by lincomb ops (K5 taps, VP+ DFT coefficients) are
 * encoded exactly: round-half-away(c * q_l). */
mmfhe_status mmfhe_load_scalars(mmfhe_ctx *ctx, const char *name, const double *v, size_t n);

/* ---- chains -------------------------------------------------- */

/* Chains: "k1_energy", "vitals_v1", "vitals_v2", "k3_doppler_dft",
 * "gesture_frame", "gesture_fc", "gesture" (frames + accumulate + FC), "gesture_features"
 * (frames + accumulate: the per-rank partial of a frame-sharded session), and the kernels
 * on their own ("used individually or composed"): "k2_soft_attention" (in: E;
 * out: N, D), "k2_doppler_soft_power" (in: K6 outputs Pm_t; out: f_t), "k4_soft_iq" (in:
 * re_t, im_t per frame; out: I_0..I_{F-1}, Q_0..Q_{F-1}), "k5_fir" (in: x_0..x_{F-1}; out:
 * per band b the filtered sequence with taps "k5.b<b>", band-major), "k5_fir_rot" (the
 * rotation-based FIR of P:205-206: every input one ciphertext holding a sequence in its
 * slots, zeros beyond; out: per band, per input, the filtered sequence in the same slots;
 * rotation keys -s and -g'b of the BSGS split of the longest band), "k6_notch" (in: P_t;
 * out: Pm_t), "k7_taylor_phase" (in: I_f,t, Q_f,t per frame; out: dphi_1..dphi_{F-1}),
 * "fc_forward" (in: features; out: logits; = gesture_fc).
 * in[0..n_in): input ciphertexts in the order the chain documents (DESIGN.md
 * §2): k1/vitals: re_0, im_0, re_1, im_1, ...; gesture*: v_re_t, v_im_t per frame.
 * Outputs: k1_energy one E per session; vitals_v1 (N, D); vitals_v2 the P_k of every
 * band's bins in band order, or with cfg.vp_plus (N_f, D_f) per band; k3_doppler_dft
 * per frame batch its d_re items then its d_im items; gesture_frame one f per frame;
 * gesture the logits; gesture_fc / fc_forward take one feature ciphertext per session and
 * run the head once over all of them as one batch (every op one launch over the sessions),
 * one logits ciphertext per session in input order.  Every output is valid in slot 0 (or the documented
 * slots); other slots may hold partial sums.
 * out: caller buffers; mmfhe_chain_plan tells their count and levels.  Outputs leave
 * through one batched INTT (coefficient form) per output batch.
 * MMFHE_E_SHAPE on a frame-count mismatch, MMFHE_E_DEPTH if in_level is too
 * low, MMFHE_E_MISSING_KEY / MMFHE_E_MISSING_PLAIN for absent operands.
 * Graph replay: when every input and output is device-resident and trace and
 * profile are off, the second call with the same chain, cfg, buffer addresses
 * and layouts is captured into a CUDA graph and later identical calls replay it
 * (same results, one graph launch; inputs are re-read each call).  Any key,
 * plaintext, scalar or prepare_chain load invalidates the captured graphs. */
mmfhe_status mmfhe_chain_plan(mmfhe_ctx *ctx, const char *chain, const mmfhe_chain_cfg *cfg, uint32_t in_level,
                              size_t n_in, uint32_t *out_levels, size_t cap, size_t *n_out);
mmfhe_status mmfhe_eval_chain(mmfhe_ctx *ctx, const char *chain, const mmfhe_chain_cfg *cfg, const mmfhe_ct *in,
                              size_t n_in, mmfhe_ct *out, size_t cap, size_t *n_out);

/* Asynchronous variant for serving loops: same arguments and results as
 * mmfhe_eval_chain, but host (ideally pinned) input/output buffers are handled
 * without blocking.  The inputs are uploaded on the context's copy stream into
 * one of two library-owned device staging slots (per chain and shape), the chain
 * runs on the ctx stream (graph replay applies), and the outputs are copied back
 * asynchronously; the call returns once everything is enqueued (output metadata
 * is already filled in).  Successive calls alternate slots, so the upload of
 * call i+1 overlaps the compute of call i.  The caller keeps every host buffer
 * alive and unmodified, and reads outputs only after mmfhe_ctx_sync.  All inputs
 * must share level, layout and form (MMFHE_E_LAYOUT otherwise).  Device-resident
 * arguments behave exactly like mmfhe_eval_chain. */
mmfhe_status mmfhe_eval_chain_async(mmfhe_ctx *ctx, const char *chain, const mmfhe_chain_cfg *cfg,
                                    const mmfhe_ct *in, size_t n_in, mmfhe_ct *out, size_t cap, size_t *n_out);
/* Wait for everything enqueued on the context (copy stream and ctx stream). */
mmfhe_status mmfhe_ctx_sync(mmfhe_ctx *ctx);

/* Sum of n partial ciphertexts mod q (cross-GPU frame accumulation after an
 * NCCL all-gather); all parts at one level and scale. */
mmfhe_status mmfhe_sum_partials(mmfhe_ctx *ctx, const mmfhe_ct *parts, size_t n, mmfhe_ct *out);

/* ---- primitives (tests, benches) -------------------------------------------
 * Inputs/outputs follow the mmfhe_ct conventions; out->data must hold the
 * result size.  Level/scale of out are written by the call. */

/* In-place forward / inverse NTT of rows [n_rows][N]; row r is taken mod
 * q_{prime_idx[r]} (indices into q_0..q_L, p_0..p_{K-1}). Device pointer. */
mmfhe_status mmfhe_ntt(mmfhe_ctx *ctx, uint64_t *d_rows, uint32_t n_rows, const uint32_t *prime_idx);
mmfhe_status mmfhe_intt(mmfhe_ctx *ctx, uint64_t *d_rows, uint32_t n_rows, const uint32_t *prime_idx);

mmfhe_status mmfhe_hadd(mmfhe_ctx *ctx, const mmfhe_ct *a, const mmfhe_ct *b, mmfhe_ct *out);
mmfhe_status mmfhe_hsub(mmfhe_ctx *ctx, const mmfhe_ct *a, const mmfhe_ct *b, mmfhe_ct *out);
/* out = a (.) pt, pt a plaintext previously loaded under (name, a->level). */
mmfhe_status mmfhe_pmult(mmfhe_ctx *ctx, const mmfhe_ct *a, const char *pt_name, mmfhe_ct *out);
/* HMult = tensor + relinearisation (no rescale). */
mmfhe_status mmfhe_hmult(mmfhe_ctx *ctx, const mmfhe_ct *a, const mmfhe_ct *b, mmfhe_ct *out);
/* Relinearise a 3-poly tensor ct (n_polys = 3). */
mmfhe_status mmfhe_relin(mmfhe_ctx *ctx, const mmfhe_ct *a3, mmfhe_ct *out);
/* HRot by step k: (sigma_g c0 + d0, d1), (d0, d1) = KS(sigma_g c1; gk_k). */
mmfhe_status mmfhe_hrot(mmfhe_ctx *ctx, const mmfhe_ct *a, int32_t step, mmfhe_ct *out);
/* Hoisted HRot: one ModUp of c1 shared by n_steps rotations (a
 * separate op -- sigma_g acts on the ModUp'd digits, residues differ from
 * mmfhe_hrot, decryption is the same rotation).  out[i] receives step i. */
mmfhe_status mmfhe_hrot_hoisted(mmfhe_ctx *ctx, const mmfhe_ct *a, const int32_t *steps, size_t n_steps,
                                mmfhe_ct *out);
/* Double hoisting's baby steps (DESIGN R22, SURVEY §8(c)-5 "a third op"): one ModUp of c1 shared
 * by n_steps rotations left over Q_level u P without ModDown, out[i] = (P sigma_g(c0) + IP_0,
 * IP_1) for step i (step 0: the P lift (P c0, P c1)).  Steps are grouped into one inner-product
 * launch per 16 (k_hoisted_ip_pq: the evaluation keys streamed once -- the path's evk-streaming
 * key-switch step).  Each out[i].data receives 2 (level+1+K) N words in the library's PQ layout:
 * poly 0 over q_0..q_level, poly 1 over q_0..q_level, poly 0 over p_0..p_{K-1}, poly 1 over
 * p_0..p_{K-1}; out[i].form selects coefficient or evaluation form, n_polys is set to 2. */
mmfhe_status mmfhe_hrot_hoisted_pq(mmfhe_ctx *ctx, const mmfhe_ct *a, const int32_t *steps, size_t n_steps,
                                   mmfhe_ct *out);
/* Rescale by q_level, round-half-up. */
mmfhe_status mmfhe_rescale(mmfhe_ctx *ctx, const mmfhe_ct *a, mmfhe_ct *out);
/* Hybrid key switching of one polynomial x (n_polys = 1, level l) with the
 * relinearisation key (step = 0) or the Galois key of `step`: out = (d0, d1). */
mmfhe_status mmfhe_keyswitch(mmfhe_ctx *ctx, const mmfhe_ct *x, int32_t step, int use_relin, mmfhe_ct *out);
/* Drop limbs to `level` (exact). */
mmfhe_status mmfhe_mod_switch(mmfhe_ctx *ctx, const mmfhe_ct *a, uint32_t level, mmfhe_ct *out);

/* ---- batched ops (throughput benches): n independent ciphertexts ---------- */
mmfhe_status mmfhe_hrot_batch(mmfhe_ctx *ctx, const mmfhe_ct *a, size_t n, int32_t step, mmfhe_ct *out);
mmfhe_status mmfhe_hmult_batch(mmfhe_ctx *ctx, const mmfhe_ct *a, const mmfhe_ct *b, size_t n, mmfhe_ct *out);

/* ---- serialisation ("versioned little-endian binary (magic, params
 * digest, per-prime residue arrays)"; keys are sent once and cached) ----
 * Blob layout, every field little-endian:
 *    0  char[8]  magic "MMFHEBLB"
 *    8  u32      version (1)
 *   12  u32      kind: MMFHE_SER_CT (ciphertext / plaintext), MMFHE_SER_RELIN_KEY,
 *                MMFHE_SER_GALOIS_KEY
 *   16  u64      params digest (mmfhe_params_digest: FNV-1a 64 over "mmfhe-params-v1",
 *                u32 log_n, u32 n_q, u64 q[n_q], u32 n_p, u64 p[n_p], u32 alpha, all LE)
 *   24  u32      log_n
 *   28  u32      level (ct) / L (key)
 *   32  u32      n_polys (ct) / dnum_L (key)
 *   36  u32      n_slots (ct) / K (key)
 *   40  f64      scale (ct) / 0
 *   48  i32      rotation step normalised to [0, N/2) (Galois key) / 0
 *   52  u32      n_rows: number of residue arrays
 *   56  u64      payload bytes = n_rows * N * 8
 *   64  u8[n_rows] prime index of each array (0..L: q_i, L+1..L+K: p_k), zero-padded to 8
 *   ..  u64[n_rows][N] residues in COEFFICIENT form, each < its prime
 * Arrays are in the ABI layouts: ct [n_polys][level+1], key [dnum][2][L+1+K].  Any other
 * magic, version, digest, size, prime order or an unreduced residue: MMFHE_E_FORMAT. */
enum { MMFHE_SER_CT = 0, MMFHE_SER_RELIN_KEY = 1, MMFHE_SER_GALOIS_KEY = 2 };
mmfhe_status mmfhe_params_digest(mmfhe_ctx *ctx, uint64_t *digest);
/* ct (host or device, coefficient or evaluation form; evaluation form is converted) into
 * buf[0..cap); *len = blob size (buf == NULL: size query only; cap too small: E_LAYOUT). */
mmfhe_status mmfhe_serialize_ct(mmfhe_ctx *ctx, const mmfhe_ct *ct, void *buf, size_t cap, size_t *len);
/* Blob -> caller buffer out->data (host or device per out->on_device, holding n_polys *
 * (level+1) * N words); writes out's level, scale, n_slots, n_polys, form = COEFF. */
mmfhe_status mmfhe_deserialize_ct(mmfhe_ctx *ctx, const void *buf, size_t len, mmfhe_ct *out);
/* Package client key words ([dnum][2][L+1+K][N] coefficient form, as mmfhe_load_*_key)
 * into a blob (the packaging only; the library never holds a secret key). */
mmfhe_status mmfhe_serialize_key(mmfhe_ctx *ctx, int kind, int32_t step, const uint64_t *words, size_t n_words,
                                 int on_device, void *buf, size_t cap, size_t *len);
/* Load a relinearisation or Galois key blob into the ctx's key store. */
mmfhe_status mmfhe_load_key_serialized(mmfhe_ctx *ctx, const void *buf, size_t len);

/* ---- the trusted client on the GPU ----------
 * For the sensor side only: these derive the secret key from `seed` on the device and never
 * hand it out; the cloud-side calls above never take it.  Randomness is the counter-based
 * SplitMix64 of synth/prng.py (client.cu states the streams), so outputs are bit-identical
 * to the reference client's.
 * mmfhe_client_keygen: pk [2][L+1][N] (b = e - a s, a), the relinearisation key (relin != 0,
 * key for s^2) and one Galois key per steps[i] (key for sigma_g(s), g = 5^(k mod N/2)), each
 * [dnum_L][2][L+1+K][N], coefficient form, written to host or device buffers (on_device).
 * mmfhe_client_encrypt: out[i] = (u b + e0 + pt_i, u a + e1) at pt_i's level with u ternary
 * and e0, e1 CBD(21) from the streams of ciphertext index first_index + i; pts are
 * coefficient-form plaintexts (n_polys = 1) sharing one level; pk as produced above. */
mmfhe_status mmfhe_client_keygen(mmfhe_ctx *ctx, uint64_t seed, const int32_t *steps, size_t n_steps, int relin,
                                 uint64_t *pk, uint64_t *rlk, uint64_t *gk, int on_device);
mmfhe_status mmfhe_client_encrypt(mmfhe_ctx *ctx, const uint64_t *pk, int pk_on_device, const mmfhe_ct *pts, size_t n,
                                  uint64_t seed, uint32_t first_index, mmfhe_ct *out);

/* ---- op trace (Theorem P:999-1006: data-oblivious execution) -------------- */
/* One logical op per line: "<op> <level> <arg>".  mmfhe_trace_clear resets. */
mmfhe_status mmfhe_trace_get(mmfhe_ctx *ctx, char *buf, size_t cap, size_t *len);
mmfhe_status mmfhe_trace_clear(mmfhe_ctx *ctx);
mmfhe_status mmfhe_trace_enable(mmfhe_ctx *ctx, int on);

/* ---- CUDA-graph replay of repeated mmfhe_eval_chain calls (default on) ----
 * on = 0 disables it and releases the captured graphs (their memory). */
mmfhe_status mmfhe_graph_enable(mmfhe_ctx *ctx, int on);
/* n_graphs: captured graphs held; replays: graph launches since ctx creation. */
mmfhe_status mmfhe_graph_stats(mmfhe_ctx *ctx, size_t *n_graphs, uint64_t *replays);

/* ---- kernel profile (bench roofline) ---------------------------------------
 * When on, CUDA events are recorded on the ctx stream around every kernel
 * launch.  mmfhe_profile_get synchronises the stream and returns one line per
 * kernel: "<kernel> <launches> <total_ms> <algorithmic_bytes>", then resets. */
mmfhe_status mmfhe_profile_enable(mmfhe_ctx *ctx, int on);
mmfhe_status mmfhe_profile_get(mmfhe_ctx *ctx, char *buf, size_t cap, size_t *len);

/* Integer roofline microbenchmark (synchronous): whole-GPU rate of one
 * register-resident operation, in operations per second.
 * kind 0: Harvey CT butterfly (lazy Shoup), 1: GS butterfly, 2: 64x64->128 MAC,
 * 3: fully reduced Shoup modular product, 4/5: CT/GS butterfly with the
 * truncated-quotient Shoup product (results in [0, 4q)).  Other kinds: E_INVALID_ARG. */
mmfhe_status mmfhe_microbench(mmfhe_ctx *ctx, int kind, double *ops_per_s);

#ifdef __cplusplus
}
#endif
#endif /* MMFHE_H */
