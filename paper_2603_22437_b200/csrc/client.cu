// client.cu -- the trusted client's key generation and encryption on the GPU (SURVEY §8(f)-4:
// "GPU keygen and encryption"; paper: 33 ms per ciphertext, 26.1 s per vital window on one
// core).  These entry points serve the CLIENT (the sensor
// side holds sk and encrypts); the cloud-side evaluator never calls them and never
// receives sk.  Randomness is the counter-based SplitMix64 of synth/prng.py (SURVEY §8(d)
// "PRNG": keyed by (seed, stream id), draw i a pure function of i), implemented here from
// its definition so that keys and ciphertexts are bit-identical to the oracle client's:
//   key(seed, sid) = mix64(mix64(seed) ^ sid),  draw_i = mix64(key + (i + 1) * GOLDEN);
//   uniform mod q: floor(draw * q / 2^64); ternary: draw mod 3 - 1;
//   CBD(21): popcount(draw & (2^21-1)) - popcount((draw >> 21) & (2^21-1)).
// Stream ids (synth/prng.py): SID_SECRET 1, SID_PK_A 2, SID_PK_E 3, SID_KS_A 2^32 + 64 key + j
// (limb t at draw offset t N), SID_KS_E 2^33 + 64 key + j, SID_ENC_U 3 2^32 + 4 index, ENC_E0 +1,
// ENC_E1 +2.  Key index 0 = relinearisation key (s' = s^2), 1 + k = Galois key of step k
// (s' = sigma_g(s)).  Formulas: pk = (e - a s, a); evk_j = (e_j - a_j s + P g_j s', a_j) with
// g_j = 1 mod q_i for q_i in digit j (full digits at level L) and 0 elsewhere (SURVEY §8(c)-5
// "Keys"); Enc(pt) = (u b + e0 + pt, u a + e1) at the plaintext's level.
#include "eval.h"
#include "modarith.cuh"

struct mmfhe_ctx : mmfhe::Ctx {
    using mmfhe::Ctx::Ctx;
};

using namespace mmfhe;

namespace {

constexpr uint64_t kGolden = 0x9E3779B97F4A7C15ull;
constexpr uint64_t kSidSecret = 1, kSidPkA = 2, kSidPkE = 3;
constexpr uint64_t kSidKsA = 1ull << 32, kSidKsE = 2ull << 32, kSidEncU = 3ull << 32;

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z)
{
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
__host__ __device__ __forceinline__ uint64_t stream_key(uint64_t seed, uint64_t sid) { return mix64(mix64(seed) ^ sid); }

enum Kind : int { kUniform = 0, kTernary = 1, kCbd = 2 };

// rows [B][R][N]: row r = item b * R + i, prime pm[i]; item b's stream id sid0 + b * sid_step.
// uniform: row i draws at offset i * N (limb t at offset t N, synth/prng.py); ternary / CBD: one
// value per coefficient (draw k), reduced into every row's prime.
struct SampleArgs {
    uint64_t seed, sid0, sid_step;
    uint32_t R;
    int kind;
    uint8_t prime[kMapCap];
};

__global__ void k_sample(uint64_t *__restrict__ out, SampleArgs a, KTables kt)
{
    const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= kt.n) return;
    const uint32_t i = blockIdx.y, b = blockIdx.z;
    const uint64_t q = kt.q[a.prime[i]];
    const uint64_t key = stream_key(a.seed, a.sid0 + (uint64_t)b * a.sid_step);
    const uint64_t idx = a.kind == kUniform ? (uint64_t)i * kt.n + k : k;
    const uint64_t x = mix64(key + (idx + 1) * kGolden);
    uint64_t v;
    if (a.kind == kUniform) {
        v = __umul64hi(x, q);
    } else {
        int64_t s;
        if (a.kind == kTernary) {
            s = (int64_t)(x % 3) - 1;
        } else {
            const uint64_t m = (1ull << 21) - 1;
            s = (int64_t)__popcll(x & m) - (int64_t)__popcll((x >> 21) & m);
        }
        v = s < 0 ? q - (uint64_t)(-s) : (uint64_t)s;
    }
    out[((size_t)b * a.R + i) * kt.n + k] = v;
}

// out = a (.) b (+ c) mod q over rows (NTT-domain products: two Montgomery reductions)
__global__ void k_mulmod_rows(uint64_t *__restrict__ out, size_t os, const uint64_t *__restrict__ a, size_t as,
                              const uint64_t *__restrict__ b, size_t bs, const uint64_t *__restrict__ c, size_t cs,
                              KTables kt, PrimeMap pm, int negate)
{
    const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= kt.n) return;
    const uint32_t i = blockIdx.y, item = blockIdx.z;
    const uint32_t p = pm.idx[i % pm.period];
    const uint64_t q = kt.q[p], qi = kt.qinv_neg[p];
    const size_t o = (size_t)i * kt.n + k;
    uint64_t v = mont_mul(mont_mul(a[item * as + o], b[item * bs + o], q, qi), kt.r2[p], q, qi);
    if (negate) v = v ? q - v : 0;
    if (c) v = add_mod(v, c[item * cs + o], q);
    out[item * os + o] = v;
}

// out += gadget_i s'_i: for rows i in [lo, hi) of each digit (rows = basis limbs)
__global__ void k_add_gadget(uint64_t *__restrict__ b_rows, const uint64_t *__restrict__ sp, KTables kt,
                             const TwPair *__restrict__ pmod, uint32_t lo, uint32_t hi)
{
    const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= kt.n) return;
    const uint32_t i = lo + blockIdx.y;
    if (i >= hi) return;
    const uint64_t q = kt.q[i];
    const size_t o = (size_t)i * kt.n + k;
    b_rows[o] = add_mod(b_rows[o], shoup(sp[o], pmod[i].w, pmod[i].wp, q), q);
}

__global__ void k_add_rows(uint64_t *__restrict__ out, size_t os, const uint64_t *__restrict__ a, size_t as,
                           KTables kt, PrimeMap pm)
{
    const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= kt.n) return;
    const uint32_t i = blockIdx.y, item = blockIdx.z;
    const uint64_t q = kt.q[pm.idx[i % pm.period]];
    const size_t o = (size_t)i * kt.n + k;
    uint64_t *d = out + item * os + o;
    *d = add_mod(*d, a[item * as + o], q);
}

dim3 g3(uint32_t n, uint32_t rows, uint32_t b) { return dim3((n + 255) / 256, rows, b); }

void sample(Ctx &c, uint64_t *out, const std::vector<uint32_t> &primes, uint32_t B, int kind, uint64_t seed,
            uint64_t sid0, uint64_t sid_step)
{
    SampleArgs a{};
    a.seed = seed;
    a.sid0 = sid0;
    a.sid_step = sid_step;
    a.R = (uint32_t)primes.size();
    a.kind = kind;
    MMFHE_REQUIRE(primes.size() <= (size_t)kMapCap, MMFHE_E_PARAMS, "too many limbs");
    for (size_t i = 0; i < primes.size(); ++i) a.prime[i] = (uint8_t)primes[i];
    k_sample<<<g3(c.n, a.R, B), 256, 0, c.stream>>>(out, a, c.kt);
    ++c.launches;
    CUDA_CHECK(cudaGetLastError());
}

void mulmod(Ctx &c, uint64_t *out, size_t os, const uint64_t *a, size_t as, const uint64_t *b, size_t bs,
            const uint64_t *add, size_t cs, const std::vector<uint32_t> &primes, uint32_t B, bool negate)
{
    const uint32_t R = (uint32_t)primes.size();
    k_mulmod_rows<<<g3(c.n, R, B), 256, 0, c.stream>>>(out, os, a, as, b, bs, add, cs, c.kt, make_map(primes),
                                                       negate ? 1 : 0);
    ++c.launches;
    CUDA_CHECK(cudaGetLastError());
}

void add_rows(Ctx &c, uint64_t *out, size_t os, const uint64_t *a, size_t as, const std::vector<uint32_t> &primes,
              uint32_t B)
{
    const uint32_t R = (uint32_t)primes.size();
    k_add_rows<<<g3(c.n, R, B), 256, 0, c.stream>>>(out, os, a, as, c.kt, make_map(primes));
    ++c.launches;
    CUDA_CHECK(cudaGetLastError());
}

std::vector<uint32_t> full_basis(const Ctx &c)
{
    std::vector<uint32_t> v;
    for (uint32_t i = 0; i < c.L + 1 + c.K; ++i) v.push_back(i);
    return v;
}

// s in NTT form over the full basis (rows L+1+K)
DBuf secret_ntt(Ctx &c, uint64_t seed)
{
    const std::vector<uint32_t> fb = full_basis(c);
    DBuf s(fb.size() * c.n, c.stream);
    sample(c, s.get(), fb, 1, kTernary, seed, kSidSecret, 0);
    ntt_forward(c, s.get(), (uint32_t)fb.size(), make_map(fb));
    return s;
}

// one evaluation key [dnum][2][L+1+K][N] in coefficient form, s' given in NTT form (full basis)
void make_evk(Ctx &c, uint64_t *out, const uint64_t *s_ntt, const uint64_t *sp_ntt, uint64_t seed, uint64_t key_index)
{
    const std::vector<uint32_t> fb = full_basis(c);
    const uint32_t R = (uint32_t)fb.size();
    const size_t rw = (size_t)R * c.n;
    const PrimeMap pm = make_map(fb);
    DBuf e(rw, c.stream), sp(rw, c.stream);
    CUDA_CHECK(cudaMemcpyAsync(sp.get(), sp_ntt, rw * 8, cudaMemcpyDeviceToDevice, c.stream));
    ntt_inverse(c, sp.get(), R, pm);  // s' in coefficient form (the gadget term is added there)
    for (uint32_t j = 0; j < c.dnum(c.L); ++j) {
        uint64_t *b = out + (size_t)(2 * j) * rw, *a = out + (size_t)(2 * j + 1) * rw;
        sample(c, a, fb, 1, kUniform, seed, kSidKsA + 64 * key_index + j, 0);
        sample(c, e.get(), fb, 1, kCbd, seed, kSidKsE + 64 * key_index + j, 0);
        // b = e - a s: NTT(a) (.) s, negated, INTT, + e
        DBuf at(rw, c.stream);
        CUDA_CHECK(cudaMemcpyAsync(at.get(), a, rw * 8, cudaMemcpyDeviceToDevice, c.stream));
        ntt_forward(c, at.get(), R, pm);
        mulmod(c, b, 0, at.get(), 0, s_ntt, 0, nullptr, 0, fb, 1, true);
        ntt_inverse(c, b, R, pm);
        add_rows(c, b, 0, e.get(), 0, fb, 1);
        const uint32_t lo = j * c.alpha, hi = std::min(lo + c.alpha, c.L + 1);
        k_add_gadget<<<g3(c.n, hi - lo, 1), 256, 0, c.stream>>>(b, sp.get(), c.kt,
                                                                 (const TwPair *)c.bconv_ptr(c.off_pd_pmod), lo, hi);
        ++c.launches;
        CUDA_CHECK(cudaGetLastError());
    }
}

thread_local std::string g_err;

mmfhe_status fail(mmfhe_ctx *c, mmfhe_status s, const char *msg)
{
    g_err = msg;
    if (c) c->last_error = msg;
    return s;
}

#define CL_BEGIN                                                                                  \
    try {                                                                                         \
        MMFHE_REQUIRE(ctx != nullptr, MMFHE_E_INVALID_ARG, "null ctx");                           \
        DeviceScope dev_scope_(ctx->device);                                                      \
        PoolScope pool_scope_(ctx->mem.pool);
#define CL_END                                                                                    \
    }                                                                                             \
    catch (const Error &e) { return fail(ctx, e.status, e.what()); }                              \
    catch (const std::exception &e) { return fail(ctx, MMFHE_E_CUDA, e.what()); }                 \
    return MMFHE_OK;

void copy_out(Ctx &c, uint64_t *dst, const uint64_t *src, size_t words, int on_device)
{
    CUDA_CHECK(cudaMemcpyAsync(dst, src, words * 8, on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost,
                               c.stream));
}

}  // namespace

extern "C" {

mmfhe_status mmfhe_client_keygen(mmfhe_ctx *ctx, uint64_t seed, const int32_t *steps, size_t n_steps, int relin,
                                 uint64_t *pk, uint64_t *rlk, uint64_t *gk, int on_device)
{
    CL_BEGIN
    MMFHE_REQUIRE(pk && (!relin || rlk) && (!n_steps || (steps && gk)), MMFHE_E_INVALID_ARG, "null argument");
    Ctx &c = *ctx;
    const std::vector<uint32_t> fb = full_basis(c);
    const uint32_t R = (uint32_t)fb.size(), RQ = c.L + 1;
    std::vector<uint32_t> qb;
    for (uint32_t i = 0; i < RQ; ++i) qb.push_back(i);
    DBuf s = secret_ntt(c, seed);  // rows q_0..q_L then p_0..p_{K-1}: the Q rows are s over Q
    // pk = (e - a s, a) over Q_L
    {
        DBuf d((size_t)2 * RQ * c.n, c.stream), at((size_t)RQ * c.n, c.stream), e((size_t)RQ * c.n, c.stream);
        uint64_t *b = d.get(), *a = d.get() + (size_t)RQ * c.n;
        sample(c, a, qb, 1, kUniform, seed, kSidPkA, 0);
        sample(c, e.get(), qb, 1, kCbd, seed, kSidPkE, 0);
        CUDA_CHECK(cudaMemcpyAsync(at.get(), a, (size_t)RQ * c.n * 8, cudaMemcpyDeviceToDevice, c.stream));
        ntt_forward(c, at.get(), RQ, make_map(qb));
        mulmod(c, b, 0, at.get(), 0, s.get(), 0, nullptr, 0, qb, 1, true);
        ntt_inverse(c, b, RQ, make_map(qb));
        add_rows(c, b, 0, e.get(), 0, qb, 1);
        copy_out(c, pk, d.get(), (size_t)2 * RQ * c.n, on_device);
    }
    const size_t kw = c.key_words();
    DBuf key(kw, c.stream), sp((size_t)R * c.n, c.stream);
    if (relin) {
        mulmod(c, sp.get(), 0, s.get(), 0, s.get(), 0, nullptr, 0, fb, 1, false);  // s^2 (NTT form)
        make_evk(c, key.get(), s.get(), sp.get(), seed, 0);
        copy_out(c, rlk, key.get(), kw, on_device);
    }
    for (size_t i = 0; i < n_steps; ++i) {
        int32_t k;
        const uint32_t g = (uint32_t)galois_element(c, steps[i], &k);
        MMFHE_REQUIRE(k != 0, MMFHE_E_INVALID_ARG, "Galois key for the identity rotation");
        if (k == MMFHE_STEP_CONJ_PROD) {  // s * sigma_{2N-1}(s) (DESIGN R32), PRNG key index 2 + N/2
            DBuf tmp((size_t)R * c.n, c.stream);
            const InvSrc src{s.get(), (size_t)R * c.n, c.n, R, (uint32_t)(2 * c.n - 1)};
            ntt_inverse(c, tmp.get(), R, make_map(fb), &src);
            ntt_forward(c, tmp.get(), R, make_map(fb));
            DBuf sp2((size_t)R * c.n, c.stream);
            mulmod(c, sp2.get(), 0, s.get(), 0, tmp.get(), 0, nullptr, 0, fb, 1, false);
            make_evk(c, key.get(), s.get(), sp2.get(), seed, 2 + (uint64_t)c.n / 2);
            copy_out(c, gk + i * kw, key.get(), kw, on_device);
            continue;
        }
        // sigma_g(s) in the NTT domain: the permutation of the inverse NTT's read (InvSrc) and back
        DBuf tmp((size_t)R * c.n, c.stream);
        const InvSrc src{s.get(), (size_t)R * c.n, c.n, R, g};
        ntt_inverse(c, tmp.get(), R, make_map(fb), &src);
        ntt_forward(c, tmp.get(), R, make_map(fb));
        // PRNG key index (oracle ckks.key_index): 1 + k for rotation k, 1 + N/2 for the conjugation
        make_evk(c, key.get(), s.get(), tmp.get(), seed, k == MMFHE_STEP_CONJ ? 1 + (uint64_t)c.n / 2 : 1 + (uint64_t)k);
        copy_out(c, gk + i * kw, key.get(), kw, on_device);
    }
    CUDA_CHECK(cudaStreamSynchronize(c.stream));
    CL_END
}

mmfhe_status mmfhe_client_encrypt(mmfhe_ctx *ctx, const uint64_t *pk, int pk_on_device, const mmfhe_ct *pts, size_t n,
                                  uint64_t seed, uint32_t first_index, mmfhe_ct *out)
{
    CL_BEGIN
    MMFHE_REQUIRE(pk && pts && out && n, MMFHE_E_INVALID_ARG, "null argument");
    Ctx &c = *ctx;
    const uint32_t l = pts[0].level, R = l + 1;
    for (size_t i = 0; i < n; ++i) {
        MMFHE_REQUIRE(pts[i].data && out[i].data && pts[i].level == l && pts[i].log_n == c.log_n &&
                          (pts[i].n_polys ? pts[i].n_polys : 2) == 1 && pts[i].form == MMFHE_FORM_COEFF,
                      MMFHE_E_LAYOUT, "plaintexts: one coefficient-form polynomial each, one level");
    }
    MMFHE_REQUIRE(l <= c.L, MMFHE_E_DEPTH, "level above the chain");
    std::vector<uint32_t> qb;
    for (uint32_t i = 0; i < R; ++i) qb.push_back(i);
    const PrimeMap pm = make_map(qb);
    const size_t rw = (size_t)R * c.n, Lw = (size_t)(c.L + 1) * c.n;
    const uint32_t B = (uint32_t)n;
    // pk limbs 0..l in NTT form
    DBuf pkd(2 * rw, c.stream);
    for (int p = 0; p < 2; ++p)
        CUDA_CHECK(cudaMemcpyAsync(pkd.get() + p * rw, pk + p * Lw, rw * 8,
                                   pk_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, c.stream));
    ntt_forward(c, pkd.get(), 2 * R, pm);
    // u (NTT form), e0, e1, pt for every item
    DBuf u(B * rw, c.stream), e0(B * rw, c.stream), e1(B * rw, c.stream), pt(B * rw, c.stream),
        ct((size_t)B * 2 * rw, c.stream);
    sample(c, u.get(), qb, B, kTernary, seed, kSidEncU + 4ull * first_index, 4);
    sample(c, e0.get(), qb, B, kCbd, seed, kSidEncU + 4ull * first_index + 1, 4);
    sample(c, e1.get(), qb, B, kCbd, seed, kSidEncU + 4ull * first_index + 2, 4);
    for (uint32_t b = 0; b < B; ++b)
        CUDA_CHECK(cudaMemcpyAsync(pt.get() + b * rw, pts[b].data, rw * 8,
                                   pts[b].on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, c.stream));
    ntt_forward(c, u.get(), B * R, pm);
    // c0 = INTT(u b) + e0 + pt, c1 = INTT(u a) + e1, items [B][2][l+1][N]
    for (int p = 0; p < 2; ++p)
        mulmod(c, ct.get() + p * rw, 2 * rw, u.get(), rw, pkd.get() + p * rw, 0, nullptr, 0, qb, B, false);
    ntt_inverse(c, ct.get(), B * 2 * R, pm);
    add_rows(c, ct.get(), 2 * rw, e0.get(), rw, qb, B);
    add_rows(c, ct.get(), 2 * rw, pt.get(), rw, qb, B);
    add_rows(c, ct.get() + rw, 2 * rw, e1.get(), rw, qb, B);
    for (uint32_t b = 0; b < B; ++b) {
        CUDA_CHECK(cudaMemcpyAsync(out[b].data, ct.get() + (size_t)b * 2 * rw, 2 * rw * 8,
                                   out[b].on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, c.stream));
        out[b].log_n = c.log_n;
        out[b].level = l;
        out[b].scale = pts[b].scale;
        out[b].n_slots = pts[b].n_slots;
        out[b].form = MMFHE_FORM_COEFF;
        out[b].n_polys = 2;
    }
    CUDA_CHECK(cudaStreamSynchronize(c.stream));
    CL_END
}

}  // extern "C"
