// serial.cpp -- versioned little-endian serialisation of ciphertexts, plaintexts and
// evaluation keys ("versioned little-endian binary (magic, params digest,
// per-prime residue arrays)"; SURVEY §5 checkpoint row: keys are "transmitted once at
// enrollment and cached on the cloud").  The byte layout is documented in
// include/mmfhe.h next to the entry points; every malformed blob is MMFHE_E_FORMAT.
#include <cstring>

#include "chains.h"

struct mmfhe_ctx : mmfhe::Ctx {
    using mmfhe::Ctx::Ctx;
};

using namespace mmfhe;

namespace {

constexpr char kMagic[8] = {'M', 'M', 'F', 'H', 'E', 'B', 'L', 'B'};
constexpr uint32_t kVersion = 1;
constexpr size_t kHeader = 64;

void put32(uint8_t *p, uint32_t v)
{
    for (int i = 0; i < 4; ++i) p[i] = (uint8_t)(v >> (8 * i));
}
void put64(uint8_t *p, uint64_t v)
{
    for (int i = 0; i < 8; ++i) p[i] = (uint8_t)(v >> (8 * i));
}
uint32_t get32(const uint8_t *p)
{
    uint32_t v = 0;
    for (int i = 0; i < 4; ++i) v |= (uint32_t)p[i] << (8 * i);
    return v;
}
uint64_t get64(const uint8_t *p)
{
    uint64_t v = 0;
    for (int i = 0; i < 8; ++i) v |= (uint64_t)p[i] << (8 * i);
    return v;
}

// FNV-1a 64 over "mmfhe-params-v1" || LE u32 log_n || u32 n_q || u64 q_i... || u32 n_p ||
// u64 p_k... || u32 alpha
uint64_t params_digest(const Ctx &c)
{
    std::vector<uint8_t> b;
    const char *tag = "mmfhe-params-v1";
    b.insert(b.end(), tag, tag + strlen(tag));
    auto w32 = [&](uint32_t v) {
        for (int i = 0; i < 4; ++i) b.push_back((uint8_t)(v >> (8 * i)));
    };
    auto w64 = [&](uint64_t v) {
        for (int i = 0; i < 8; ++i) b.push_back((uint8_t)(v >> (8 * i)));
    };
    w32(c.log_n);
    w32(c.L + 1);
    for (uint32_t i = 0; i <= c.L; ++i) w64(c.primes[i]);
    w32(c.K);
    for (uint32_t k = 0; k < c.K; ++k) w64(c.primes[c.L + 1 + k]);
    w32(c.alpha);
    uint64_t h = 0xcbf29ce484222325ull;
    for (uint8_t x : b) {
        h ^= x;
        h *= 0x100000001b3ull;
    }
    return h;
}

size_t rows_off(uint32_t n_rows) { return kHeader + ((n_rows + 7) / 8) * 8; }

struct Blob {
    uint32_t kind, log_n, level, n_polys, n_slots, n_rows;
    double scale;
    int32_t step;
    std::vector<uint8_t> prime;  // [n_rows]
    const uint8_t *res;          // [n_rows][N] little-endian u64
};

void write_blob(const Ctx &c, const Blob &h, const uint64_t *words, uint8_t *out)
{
    memset(out, 0, rows_off(h.n_rows));
    memcpy(out, kMagic, 8);
    put32(out + 8, kVersion);
    put32(out + 12, h.kind);
    put64(out + 16, params_digest(c));
    put32(out + 24, h.log_n);
    put32(out + 28, h.level);
    put32(out + 32, h.n_polys);
    put32(out + 36, h.n_slots);
    uint64_t sb;
    memcpy(&sb, &h.scale, 8);
    put64(out + 40, sb);
    put32(out + 48, (uint32_t)h.step);
    put32(out + 52, h.n_rows);
    put64(out + 56, (uint64_t)h.n_rows * c.n * 8);
    for (uint32_t r = 0; r < h.n_rows; ++r) out[kHeader + r] = h.prime[r];
    uint8_t *p = out + rows_off(h.n_rows);
    for (size_t i = 0; i < (size_t)h.n_rows * c.n; ++i) put64(p + 8 * i, words[i]);
}

Blob read_blob(const Ctx &c, const uint8_t *in, size_t len)
{
    MMFHE_REQUIRE(in && len >= kHeader, MMFHE_E_FORMAT, "blob shorter than its header");
    MMFHE_REQUIRE(memcmp(in, kMagic, 8) == 0, MMFHE_E_FORMAT, "bad magic");
    MMFHE_REQUIRE(get32(in + 8) == kVersion, MMFHE_E_FORMAT, "unsupported version " + std::to_string(get32(in + 8)));
    MMFHE_REQUIRE(get64(in + 16) == params_digest(c), MMFHE_E_FORMAT, "parameter digest differs from this ctx");
    Blob h;
    h.kind = get32(in + 12);
    h.log_n = get32(in + 24);
    h.level = get32(in + 28);
    h.n_polys = get32(in + 32);
    h.n_slots = get32(in + 36);
    const uint64_t sb = get64(in + 40);
    memcpy(&h.scale, &sb, 8);
    h.step = (int32_t)get32(in + 48);
    h.n_rows = get32(in + 52);
    MMFHE_REQUIRE(h.log_n == c.log_n, MMFHE_E_FORMAT, "ring dimension differs from this ctx");
    MMFHE_REQUIRE(h.n_rows >= 1 && h.n_rows <= 4096, MMFHE_E_FORMAT, "bad residue array count");
    MMFHE_REQUIRE(get64(in + 56) == (uint64_t)h.n_rows * c.n * 8, MMFHE_E_FORMAT, "payload size mismatch");
    MMFHE_REQUIRE(len == rows_off(h.n_rows) + (size_t)h.n_rows * c.n * 8, MMFHE_E_FORMAT, "blob length mismatch");
    h.prime.assign(in + kHeader, in + kHeader + h.n_rows);
    h.res = in + rows_off(h.n_rows);
    for (uint32_t r = 0; r < h.n_rows; ++r) {
        MMFHE_REQUIRE(h.prime[r] < c.primes.size(), MMFHE_E_FORMAT, "prime index out of range");
        const uint64_t q = c.primes[h.prime[r]];
        const uint8_t *p = h.res + (size_t)r * c.n * 8;
        for (uint32_t k = 0; k < c.n; ++k)
            MMFHE_REQUIRE(get64(p + 8 * k) < q, MMFHE_E_FORMAT, "residue not reduced mod its prime");
    }
    return h;
}

// residue rows of a ciphertext / plaintext: poly-major, limbs q_0..q_level
std::vector<uint8_t> ct_primes(uint32_t level, uint32_t n_polys)
{
    std::vector<uint8_t> v;
    for (uint32_t p = 0; p < n_polys; ++p)
        for (uint32_t i = 0; i <= level; ++i) v.push_back((uint8_t)i);
    return v;
}

// key rows: [dnum][2][L+1+K] over q_0..q_L, p_0..p_{K-1}
std::vector<uint8_t> key_primes(const Ctx &c)
{
    std::vector<uint8_t> v;
    for (uint32_t j = 0; j < c.dnum(c.L); ++j)
        for (int p = 0; p < 2; ++p)
            for (uint32_t i = 0; i < c.L + 1 + c.K; ++i) v.push_back((uint8_t)i);
    return v;
}

thread_local std::string g_err;

mmfhe_status fail(mmfhe_ctx *c, mmfhe_status s, const char *msg)
{
    g_err = msg;
    if (c) c->last_error = msg;
    return s;
}

#define SER_BEGIN                                                                                 \
    try {                                                                                         \
        MMFHE_REQUIRE(ctx != nullptr, MMFHE_E_INVALID_ARG, "null ctx");                           \
        DeviceScope dev_scope_(ctx->device);                                                      \
        PoolScope pool_scope_(ctx->mem.pool);
#define SER_END                                                                                   \
    }                                                                                             \
    catch (const Error &e) { return fail(ctx, e.status, e.what()); }                              \
    catch (const std::exception &e) { return fail(ctx, MMFHE_E_CUDA, e.what()); }                 \
    return MMFHE_OK;

}  // namespace

extern "C" {

mmfhe_status mmfhe_params_digest(mmfhe_ctx *ctx, uint64_t *digest)
{
    SER_BEGIN
    MMFHE_REQUIRE(digest, MMFHE_E_INVALID_ARG, "null argument");
    *digest = params_digest(*ctx);
    SER_END
}

mmfhe_status mmfhe_serialize_ct(mmfhe_ctx *ctx, const mmfhe_ct *ct, void *buf, size_t cap, size_t *len)
{
    SER_BEGIN
    MMFHE_REQUIRE(ct && len && ct->data, MMFHE_E_INVALID_ARG, "null argument");
    MMFHE_REQUIRE(ct->log_n == ctx->log_n && ct->level <= ctx->L, MMFHE_E_PARAMS, "ciphertext not of this ctx");
    MMFHE_REQUIRE(ct->form == MMFHE_FORM_COEFF || ct->form == MMFHE_FORM_EVAL, MMFHE_E_FORMAT, "bad form");
    const uint32_t np = ct->n_polys ? ct->n_polys : 2;
    Blob h{MMFHE_SER_CT, ctx->log_n, ct->level, np, ct->n_slots, np * (ct->level + 1), ct->scale, 0,
           ct_primes(ct->level, np), nullptr};
    const size_t words = (size_t)h.n_rows * ctx->n, total = rows_off(h.n_rows) + words * 8;
    *len = total;
    if (!buf) return MMFHE_OK;  // size query
    MMFHE_REQUIRE(cap >= total, MMFHE_E_LAYOUT, "buffer too small");
    std::vector<uint64_t> host(words);
    if (ct->form == MMFHE_FORM_EVAL) {
        // the interchange form is coefficient form: leave the library's NTT form first
        DCt x = import_ct(*ctx, *ct, np);  // an NTT-form copy
        DBuf coef(words, ctx->stream);
        const InvSrc src{x.data(), words, ctx->n, h.n_rows, 1};
        std::vector<uint32_t> pm;
        for (uint32_t i = 0; i <= ct->level; ++i) pm.push_back(i);
        ntt_inverse(*ctx, coef.get(), h.n_rows, make_map(pm), &src);
        CUDA_CHECK(cudaMemcpyAsync(host.data(), coef.get(), words * 8, cudaMemcpyDeviceToHost, ctx->stream));
        CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
    } else if (ct->on_device) {
        CUDA_CHECK(cudaMemcpyAsync(host.data(), ct->data, words * 8, cudaMemcpyDeviceToHost, ctx->stream));
        CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
    } else {
        memcpy(host.data(), ct->data, words * 8);
    }
    write_blob(*ctx, h, host.data(), (uint8_t *)buf);
    SER_END
}

mmfhe_status mmfhe_deserialize_ct(mmfhe_ctx *ctx, const void *buf, size_t len, mmfhe_ct *out)
{
    SER_BEGIN
    MMFHE_REQUIRE(buf && out && out->data, MMFHE_E_INVALID_ARG, "null argument");
    Blob h = read_blob(*ctx, (const uint8_t *)buf, len);
    MMFHE_REQUIRE(h.kind == MMFHE_SER_CT, MMFHE_E_FORMAT, "blob is not a ciphertext");
    MMFHE_REQUIRE(h.level <= ctx->L && h.n_polys >= 1 && h.n_polys <= 3 && h.n_rows == h.n_polys * (h.level + 1),
                  MMFHE_E_FORMAT, "ciphertext layout");
    MMFHE_REQUIRE(h.prime == ct_primes(h.level, h.n_polys), MMFHE_E_FORMAT, "ciphertext prime order");
    const size_t words = (size_t)h.n_rows * ctx->n;
    std::vector<uint64_t> host(words);
    for (size_t i = 0; i < words; ++i) host[i] = get64(h.res + 8 * i);
    if (out->on_device) {
        CUDA_CHECK(cudaMemcpyAsync(out->data, host.data(), words * 8, cudaMemcpyHostToDevice, ctx->stream));
        CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
    } else {
        memcpy(out->data, host.data(), words * 8);
    }
    out->log_n = h.log_n;
    out->level = h.level;
    out->n_polys = h.n_polys;
    out->n_slots = h.n_slots;
    out->scale = h.scale;
    out->form = MMFHE_FORM_COEFF;
    SER_END
}

mmfhe_status mmfhe_serialize_key(mmfhe_ctx *ctx, int kind, int32_t step, const uint64_t *words, size_t n_words,
                                 int on_device, void *buf, size_t cap, size_t *len)
{
    SER_BEGIN
    MMFHE_REQUIRE(words && len, MMFHE_E_INVALID_ARG, "null argument");
    MMFHE_REQUIRE(kind == MMFHE_SER_RELIN_KEY || kind == MMFHE_SER_GALOIS_KEY, MMFHE_E_INVALID_ARG, "bad key kind");
    MMFHE_REQUIRE(n_words == ctx->key_words(), MMFHE_E_LAYOUT, "key must hold dnum*2*(L+1+K)*N words");
    int32_t k = 0;
    if (kind == MMFHE_SER_GALOIS_KEY) galois_element(*ctx, step, &k);
    Blob h{(uint32_t)kind, ctx->log_n, ctx->L, ctx->dnum(ctx->L), ctx->K, (uint32_t)(n_words / ctx->n), 0.0, k,
           key_primes(*ctx), nullptr};
    const size_t total = rows_off(h.n_rows) + n_words * 8;
    *len = total;
    if (!buf) return MMFHE_OK;
    MMFHE_REQUIRE(cap >= total, MMFHE_E_LAYOUT, "buffer too small");
    std::vector<uint64_t> host(n_words);
    if (on_device) {
        CUDA_CHECK(cudaMemcpy(host.data(), words, n_words * 8, cudaMemcpyDeviceToHost));
    } else {
        memcpy(host.data(), words, n_words * 8);
    }
    write_blob(*ctx, h, host.data(), (uint8_t *)buf);
    SER_END
}

mmfhe_status mmfhe_load_key_serialized(mmfhe_ctx *ctx, const void *buf, size_t len)
{
    SER_BEGIN
    Blob h = read_blob(*ctx, (const uint8_t *)buf, len);
    MMFHE_REQUIRE(h.kind == MMFHE_SER_RELIN_KEY || h.kind == MMFHE_SER_GALOIS_KEY, MMFHE_E_FORMAT, "blob is not a key");
    MMFHE_REQUIRE(h.level == ctx->L && h.n_polys == ctx->dnum(ctx->L) && h.n_slots == ctx->K &&
                      (size_t)h.n_rows * ctx->n == ctx->key_words() && h.prime == key_primes(*ctx),
                  MMFHE_E_FORMAT, "key layout");
    std::vector<uint64_t> host((size_t)h.n_rows * ctx->n);
    for (size_t i = 0; i < host.size(); ++i) host[i] = get64(h.res + 8 * i);
    ctx->drop_graphs();
    ++ctx->state_gen;
    if (h.kind == MMFHE_SER_RELIN_KEY) {
        auto k = std::make_unique<DKey>();
        load_key(*ctx, *k, host.data(), host.size(), false);
        ctx->rlk = std::move(k);
    } else {
        int32_t k;
        galois_element(*ctx, h.step, &k);
        MMFHE_REQUIRE(k != 0, MMFHE_E_FORMAT, "Galois key for the identity rotation");
        auto key = std::make_unique<DKey>();
        load_key(*ctx, *key, host.data(), host.size(), false);
        ctx->gk[k] = std::move(key);
    }
    CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
    SER_END
}

}  // extern "C"
