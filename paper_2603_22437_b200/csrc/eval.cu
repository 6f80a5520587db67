// eval.cu -- host orchestration of the CKKS evaluator ops on the ctx stream.
#include <algorithm>
#include <cmath>

#include "eval.h"

namespace mmfhe {

namespace {
PrimeMap qmap(const Ctx &c, uint32_t level) { return make_map(c.q_basis(level)); }

void memcpy_d2d(Ctx &c, uint64_t *dst, const uint64_t *src, size_t words)
{
    CUDA_CHECK(cudaMemcpyAsync(dst, src, words * 8, cudaMemcpyDeviceToDevice, c.stream));
}
}  // namespace

DCt make_ct(Ctx &c, uint32_t level, uint32_t npolys, uint32_t n_slots, double scale)
{
    DCt r;
    r.buf = DBuf((size_t)npolys * (level + 1) * c.n, c.stream);
    r.level = level;
    r.npolys = npolys;
    r.n_slots = n_slots;
    r.scale = scale;
    return r;
}

DCt view_ct(const mmfhe_ct &ct, uint32_t npolys)
{
    DCt r;
    r.ext = ct.data;
    r.level = ct.level;
    r.npolys = npolys;
    r.n_slots = ct.n_slots;
    r.scale = ct.scale;
    return r;
}

DCt import_ct(Ctx &c, const mmfhe_ct &in, uint32_t npolys)
{
    MMFHE_REQUIRE(in.data != nullptr, MMFHE_E_INVALID_ARG, "null ciphertext data");
    MMFHE_REQUIRE(in.log_n == c.log_n, MMFHE_E_PARAMS, "ring dimension mismatch");
    MMFHE_REQUIRE(in.level <= c.L, MMFHE_E_DEPTH, "level above the chain");
    MMFHE_REQUIRE(in.form == MMFHE_FORM_COEFF || in.form == MMFHE_FORM_EVAL, MMFHE_E_FORMAT, "bad form");
    DCt r = make_ct(c, in.level, npolys, in.n_slots, in.scale);
    const size_t words = (size_t)npolys * (in.level + 1) * c.n;
    CUDA_CHECK(cudaMemcpyAsync(r.data(), in.data, words * 8,
                               in.on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, c.stream));
    if (in.form == MMFHE_FORM_COEFF)
        ntt_forward(c.kt, r.data(), npolys * (in.level + 1), qmap(c, in.level), c.stream, c.launches);
    return r;
}

void export_ct(Ctx &c, const DCt &in, mmfhe_ct &out)
{
    MMFHE_REQUIRE(out.data != nullptr, MMFHE_E_INVALID_ARG, "null output buffer");
    const uint32_t rows = in.npolys * (in.level + 1);
    const size_t words = (size_t)rows * c.n;
    out.log_n = c.log_n;
    out.level = in.level;
    out.scale = in.scale;
    out.n_slots = in.n_slots;
    out.n_polys = in.npolys;
    if (out.on_device) {
        memcpy_d2d(c, out.data, in.data(), words);
        if (out.form == MMFHE_FORM_COEFF) ntt_inverse(c.kt, out.data, rows, qmap(c, in.level), c.stream, c.launches);
    } else {
        DBuf tmp(words, c.stream);
        memcpy_d2d(c, tmp.get(), in.data(), words);
        if (out.form == MMFHE_FORM_COEFF) ntt_inverse(c.kt, tmp.get(), rows, qmap(c, in.level), c.stream, c.launches);
        CUDA_CHECK(cudaMemcpyAsync(out.data, tmp.get(), words * 8, cudaMemcpyDeviceToHost, c.stream));
        CUDA_CHECK(cudaStreamSynchronize(c.stream));
    }
}

// ------------------------------------------------------------------ exact ops
DCt ev_addsub(Ctx &c, const DCt &a, const DCt &b, bool sub)
{
    MMFHE_REQUIRE(a.level == b.level && a.npolys == b.npolys, MMFHE_E_LAYOUT, "hadd level/size mismatch");
    MMFHE_REQUIRE(a.scale == b.scale, MMFHE_E_SCALE, "hadd scale mismatch");
    c.rec(sub ? "hsub" : "hadd", a.level);
    DCt r = make_ct(c, a.level, a.npolys, a.n_slots, a.scale);
    launch_addsub(c, r.data(), a.data(), b.data(), a.npolys * (a.level + 1), qmap(c, a.level), sub);
    return r;
}

DCt ev_sum(Ctx &c, const std::vector<const DCt *> &cts)
{
    MMFHE_REQUIRE(!cts.empty(), MMFHE_E_INVALID_ARG, "empty sum");
    const DCt &a0 = *cts[0];
    DCt r = make_ct(c, a0.level, a0.npolys, a0.n_slots, a0.scale);
    memcpy_d2d(c, r.data(), a0.data(), (size_t)a0.npolys * (a0.level + 1) * c.n);
    for (size_t i = 1; i < cts.size(); ++i) {
        const DCt &b = *cts[i];
        MMFHE_REQUIRE(b.level == a0.level && b.npolys == a0.npolys, MMFHE_E_LAYOUT, "sum level mismatch");
        MMFHE_REQUIRE(b.scale == a0.scale, MMFHE_E_SCALE, "sum scale mismatch");
        c.rec("hadd", a0.level);
        launch_addsub(c, r.data(), r.data(), b.data(), a0.npolys * (a0.level + 1), qmap(c, a0.level), false);
    }
    return r;
}

DCt ev_drop_to(Ctx &c, const DCt &a, uint32_t level)
{
    MMFHE_REQUIRE(level <= a.level, MMFHE_E_DEPTH, "cannot raise a level");
    DCt r = make_ct(c, level, a.npolys, a.n_slots, a.scale);
    if (level != a.level) c.rec("modswitch", a.level, std::to_string(level));
    CUDA_CHECK(cudaMemcpy2DAsync(r.data(), (size_t)(level + 1) * c.n * 8, a.data(), (size_t)(a.level + 1) * c.n * 8,
                                 (size_t)(level + 1) * c.n * 8, a.npolys, cudaMemcpyDeviceToDevice, c.stream));
    return r;
}

DCt ev_tensor_sum(Ctx &c, const std::vector<std::pair<const DCt *, const DCt *>> &pairs)
{
    MMFHE_REQUIRE(!pairs.empty(), MMFHE_E_INVALID_ARG, "empty tensor sum");
    const DCt &a0 = *pairs[0].first;
    const double sc = a0.scale * pairs[0].second->scale;
    for (auto &pr : pairs) {
        MMFHE_REQUIRE(pr.first->level == a0.level && pr.second->level == a0.level, MMFHE_E_LAYOUT,
                      "tensor level mismatch");
        MMFHE_REQUIRE(pr.first->npolys == 2 && pr.second->npolys == 2, MMFHE_E_LAYOUT, "tensor needs 2-poly cts");
        MMFHE_REQUIRE(pr.first->scale * pr.second->scale == sc, MMFHE_E_SCALE, "tensor_sum scale mismatch");
    }
    c.rec("tensor_sum", a0.level, std::to_string(pairs.size()));
    DCt r = make_ct(c, a0.level, 3, a0.n_slots, sc);
    for (size_t s = 0; s < pairs.size(); s += kMaxTerms) {
        PtrList A{}, B{};
        int n = (int)std::min<size_t>(kMaxTerms, pairs.size() - s);
        for (int i = 0; i < n; ++i) {
            A.p[i] = pairs[s + i].first->data();
            B.p[i] = pairs[s + i].second->data();
        }
        launch_tensor_sum(c, r.data(), A, B, n, a0.level, s > 0);
    }
    return r;
}

DCt ev_pmult_sum(Ctx &c, const std::vector<std::pair<const DPlain *, const DCt *>> &terms)
{
    MMFHE_REQUIRE(!terms.empty(), MMFHE_E_INVALID_ARG, "empty pmult sum");
    const DCt &a0 = *terms[0].second;
    const double sc = a0.scale * terms[0].first->scale;
    for (auto &t : terms) {
        MMFHE_REQUIRE(t.second->level == a0.level && t.second->npolys == 2, MMFHE_E_LAYOUT, "pmult level mismatch");
        MMFHE_REQUIRE(t.first->level == a0.level, MMFHE_E_LAYOUT, "plaintext level mismatch");
        MMFHE_REQUIRE(t.second->scale * t.first->scale == sc, MMFHE_E_SCALE, "pmult_sum scale mismatch");
    }
    c.rec("pmult_sum", a0.level, std::to_string(terms.size()));
    DCt r = make_ct(c, a0.level, 2, a0.n_slots, sc);
    for (size_t s = 0; s < terms.size(); s += kMaxTerms) {
        PtrList P{}, C{};
        int n = (int)std::min<size_t>(kMaxTerms, terms.size() - s);
        for (int i = 0; i < n; ++i) {
            P.p[i] = terms[s + i].first->buf.get();
            C.p[i] = terms[s + i].second->data();
        }
        launch_pmult_sum(c, r.data(), P, C, n, a0.level, s > 0);
    }
    return r;
}

uint64_t encode_scalar_mod(double v, uint64_t q_scale, uint64_t m)
{
    // v = mant * 2^e exactly with |mant| < 2^53; x = v * q_scale = mant * q_scale * 2^e;
    // round half away from zero, exactly, in 128-bit integers.
    typedef unsigned __int128 u128;
    if (v == 0.0) return 0;
    MMFHE_REQUIRE(std::isfinite(v), MMFHE_E_INVALID_ARG, "non-finite scalar");
    int e;
    double f = std::frexp(std::fabs(v), &e);           // |v| = f * 2^e, f in [0.5, 1)
    uint64_t mant = (uint64_t)std::ldexp(f, 53);       // exact
    e -= 53;                                           // |v| = mant * 2^e
    u128 prod = (u128)mant * q_scale;                  // < 2^113
    u128 mag;
    if (e >= 0) {
        MMFHE_REQUIRE(e < 14, MMFHE_E_SCALE, "scalar constant overflows the encoding");
        mag = prod << e;
    } else if (-e >= 120) {
        mag = 0;
    } else {
        u128 half = (u128)1 << (-e - 1);
        mag = (prod + half) >> (-e);                   // ties away from zero (on |x|)
    }
    uint64_t r = (uint64_t)(mag % m);
    return (v < 0 && r) ? m - r : r;
}

DCt ev_lincomb(Ctx &c, const std::vector<const DCt *> &cts, const std::vector<double> &coefs)
{
    MMFHE_REQUIRE(!cts.empty() && cts.size() == coefs.size(), MMFHE_E_INVALID_ARG, "lincomb size");
    const DCt &a0 = *cts[0];
    for (auto *ct : cts)
        MMFHE_REQUIRE(ct->level == a0.level && ct->scale == a0.scale && ct->npolys == 2, MMFHE_E_SCALE,
                      "lincomb operands must share level and scale");
    c.rec("lincomb", a0.level, std::to_string(cts.size()));
    const uint32_t l = a0.level;
    const uint64_t ql = c.primes[l];
    // constant table [n][l+1] of Shoup pairs, cached by content
    std::string key = std::to_string(l) + ":";
    key.append((const char *)coefs.data(), coefs.size() * sizeof(double));
    auto it = c.const_cache.find(key);
    if (it == c.const_cache.end()) {
        std::vector<TwPair> tab(coefs.size() * (l + 1));
        for (size_t t = 0; t < coefs.size(); ++t)
            for (uint32_t i = 0; i <= l; ++i) {
                uint64_t v = encode_scalar_mod(coefs[t], ql, c.primes[i]);
                tab[t * (l + 1) + i] = {v, host::shoup(v, c.primes[i])};
            }
        DBuf b((tab.size() * sizeof(TwPair) + 7) / 8, c.stream);
        CUDA_CHECK(cudaMemcpyAsync(b.get(), tab.data(), tab.size() * sizeof(TwPair), cudaMemcpyHostToDevice,
                                   c.stream));
        CUDA_CHECK(cudaStreamSynchronize(c.stream));
        it = c.const_cache.emplace(key, std::move(b)).first;
    }
    const TwPair *consts = (const TwPair *)it->second.get();
    DCt r = make_ct(c, l, 2, a0.n_slots, a0.scale * (double)ql);
    for (size_t s = 0; s < cts.size(); s += kMaxTerms) {
        PtrList C{};
        int n = (int)std::min<size_t>(kMaxTerms, cts.size() - s);
        for (int i = 0; i < n; ++i) C.p[i] = cts[s + i]->data();
        launch_lincomb(c, r.data(), C, consts + s * (l + 1), n, l, s > 0);
    }
    return r;
}

DCt ev_add_plain(Ctx &c, const DCt &a, const DPlain &pt)
{
    MMFHE_REQUIRE(pt.level == a.level, MMFHE_E_LAYOUT, "plaintext level mismatch");
    MMFHE_REQUIRE(pt.scale == a.scale, MMFHE_E_SCALE, "add_plain scale mismatch");
    c.rec("add_plain", a.level);
    DCt r = make_ct(c, a.level, 2, a.n_slots, a.scale);
    memcpy_d2d(c, r.data(), a.data(), (size_t)2 * (a.level + 1) * c.n);
    launch_add_plain(c, r.data(), pt.buf.get(), a.level);
    return r;
}

// ------------------------------------------------------------------ key switching
void ev_keyswitch(Ctx &c, const uint64_t *x_ntt, uint32_t l, const DKey &key, uint64_t *out0, uint64_t *out1,
                  const uint64_t *add0, const uint64_t *add1)
{
    const size_t N = c.n;
    // 1. coefficient form of x
    DBuf xc((size_t)(l + 1) * N, c.stream);
    memcpy_d2d(c, xc.get(), x_ntt, (size_t)(l + 1) * N);
    ntt_inverse(c.kt, xc.get(), l + 1, qmap(c, l), c.stream, c.launches);
    // 2. ModUp: fast BConv of every digit, then NTT of the converted rows
    const auto &plans = c.modup[l];
    std::vector<size_t> off;
    std::vector<uint32_t> rowmap;
    const std::vector<uint32_t> basis = c.ext_basis(l);
    size_t T = 0;
    for (const auto &p : plans) {
        off.push_back(T);
        for (uint32_t r = 0; r < basis.size(); ++r)
            if (r < p.lo || r >= p.hi) rowmap.push_back(basis[r]);
        T += p.n_tgt;
    }
    DBuf y(T * N, c.stream);
    launch_modup_bconv(c, y.get(), xc.get(), l, off);
    ntt_forward(c.kt, y.get(), (uint32_t)T, make_map(rowmap), c.stream, c.launches);
    // 3. key inner product (evk streamed once)
    DBuf accQ((size_t)2 * (l + 1) * N, c.stream), accP((size_t)2 * c.K * N, c.stream);
    launch_key_ip(c, accQ.get(), accP.get(), x_ntt, y.get(), off, key.buf.get(), l);
    // 4. ModDown
    std::vector<uint32_t> pm;
    for (uint32_t k = 0; k < c.K; ++k) pm.push_back(c.L + 1 + k);
    ntt_inverse(c.kt, accP.get(), 2 * c.K, make_map(pm), c.stream, c.launches);
    DBuf w((size_t)2 * (l + 1) * N, c.stream);
    launch_moddown_bconv(c, w.get(), accP.get(), l);
    ntt_forward(c.kt, w.get(), 2 * (l + 1), qmap(c, l), c.stream, c.launches);
    launch_moddown_final(c, out0, out1, accQ.get(), w.get(), add0, add1, l);
}

DCt ev_relin(Ctx &c, const DCt &a3)
{
    MMFHE_REQUIRE(a3.npolys == 3, MMFHE_E_LAYOUT, "relin needs a 3-poly ciphertext");
    MMFHE_REQUIRE(c.rlk != nullptr, MMFHE_E_MISSING_KEY, "missing relinearisation key");
    c.rec("relin", a3.level);
    DCt r = make_ct(c, a3.level, 2, a3.n_slots, a3.scale);
    ev_keyswitch(c, a3.poly(2, c.n), a3.level, *c.rlk, r.poly(0, c.n), r.poly(1, c.n), a3.poly(0, c.n),
                 a3.poly(1, c.n));
    return r;
}

uint64_t galois_element(const Ctx &c, int32_t step, int32_t *normalised)
{
    const int64_t half = c.n / 2;
    int64_t k = ((int64_t)step % half + half) % half;
    if (normalised) *normalised = (int32_t)k;
    return host::pow(5, (uint64_t)k, 2ull * c.n);
}

const DKey &find_gk(const Ctx &c, int32_t k)
{
    auto it = c.gk.find(k);
    MMFHE_REQUIRE(it != c.gk.end(), MMFHE_E_MISSING_KEY, "missing Galois key for rotation " + std::to_string(k));
    return *it->second;
}

DCt ev_rotate(Ctx &c, const DCt &a, int32_t step)
{
    MMFHE_REQUIRE(a.npolys == 2, MMFHE_E_LAYOUT, "rotate needs a 2-poly ciphertext");
    int32_t k;
    const uint64_t g = galois_element(c, step, &k);
    DCt r = make_ct(c, a.level, 2, a.n_slots, a.scale);
    if (k == 0) {
        memcpy_d2d(c, r.data(), a.data(), (size_t)2 * (a.level + 1) * c.n);
        return r;
    }
    const DKey &key = find_gk(c, k);
    c.rec("hrot", a.level, std::to_string(k));
    DBuf sig((size_t)2 * (a.level + 1) * c.n, c.stream);
    launch_automorph(c, sig.get(), a.data(), 2 * (a.level + 1), g);
    const uint64_t *s0 = sig.get(), *s1 = sig.get() + (size_t)(a.level + 1) * c.n;
    ev_keyswitch(c, s1, a.level, key, r.poly(0, c.n), r.poly(1, c.n), s0, nullptr);
    return r;
}

DCt ev_rescale(Ctx &c, const DCt &a)
{
    MMFHE_REQUIRE(a.npolys == 2, MMFHE_E_LAYOUT, "rescale needs a 2-poly ciphertext");
    MMFHE_REQUIRE(a.level >= 1, MMFHE_E_DEPTH, "depth exhausted");
    const uint32_t l = a.level;
    c.rec("rescale", l);
    const size_t N = c.n;
    DBuf t(2 * N, c.stream);
    memcpy_d2d(c, t.get(), a.poly(0, c.n) + (size_t)l * N, N);
    memcpy_d2d(c, t.get() + N, a.poly(1, c.n) + (size_t)l * N, N);
    ntt_inverse(c.kt, t.get(), 2, make_map({l}), c.stream, c.launches);
    DBuf v((size_t)2 * l * N, c.stream);
    launch_rescale_prep(c, v.get(), t.get(), l);
    ntt_forward(c.kt, v.get(), 2 * l, qmap(c, l - 1), c.stream, c.launches);
    DCt r = make_ct(c, l - 1, 2, a.n_slots, a.scale / (double)c.primes[l]);
    launch_rescale_final(c, r.data(), a.data(), v.get(), l);
    return r;
}

DCt ev_rotsum(Ctx &c, const DCt &a, uint32_t count, uint32_t stride)
{
    DCt acc = make_ct(c, a.level, 2, a.n_slots, a.scale);
    memcpy_d2d(c, acc.data(), a.data(), (size_t)2 * (a.level + 1) * c.n);
    uint32_t step = stride;
    for (uint32_t n = 1; n < count; n *= 2, step *= 2) {
        DCt r = ev_rotate(c, acc, (int32_t)step);
        acc = ev_addsub(c, acc, r, false);
    }
    return acc;
}

// ------------------------------------------------------------------ stores
void load_key(Ctx &c, DKey &k, const uint64_t *words, size_t n_words, bool on_device)
{
    MMFHE_REQUIRE(n_words == c.key_words(), MMFHE_E_LAYOUT,
                  "key must hold dnum*2*(L+1+K)*N words (" + std::to_string(c.key_words()) + ")");
    k.buf = DBuf(n_words, c.stream);
    CUDA_CHECK(cudaMemcpyAsync(k.buf.get(), words, n_words * 8,
                               on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, c.stream));
    std::vector<uint32_t> all;
    for (uint32_t i = 0; i < c.L + 1 + c.K; ++i) all.push_back(i);
    const uint32_t rows = (uint32_t)(n_words / c.n);
    PrimeMap pm = make_map(all);
    ntt_forward(c.kt, k.buf.get(), rows, pm, c.stream, c.launches);
    launch_to_mont(c, k.buf.get(), rows, pm);
}

void load_plain(Ctx &c, const std::string &name, uint32_t level, double scale, const uint64_t *coef, bool on_device)
{
    MMFHE_REQUIRE(level <= c.L, MMFHE_E_DEPTH, "plaintext level above the chain");
    auto p = std::make_unique<DPlain>();
    p->level = level;
    p->scale = scale;
    const size_t words = (size_t)(level + 1) * c.n;
    p->buf = DBuf(words, c.stream);
    CUDA_CHECK(cudaMemcpyAsync(p->buf.get(), coef, words * 8,
                               on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, c.stream));
    PrimeMap pm = qmap(c, level);
    ntt_forward(c.kt, p->buf.get(), level + 1, pm, c.stream, c.launches);
    launch_to_mont(c, p->buf.get(), level + 1, pm);
    c.plains[plain_key(name, level)] = std::move(p);
}

const DPlain &need_plain(const Ctx &c, const std::string &name, uint32_t level)
{
    DPlain *p = c.find_plain(name, level);
    MMFHE_REQUIRE(p != nullptr, MMFHE_E_MISSING_PLAIN, "missing plaintext operand " + plain_key(name, level));
    return *p;
}

}  // namespace mmfhe
