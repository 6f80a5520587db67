// eval.cu -- host orchestration of the batched CKKS evaluator ops on the ctx stream.
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

void rec_n(Ctx &c, const char *op, uint32_t level, uint32_t times, const std::string &arg = "")
{
    for (uint32_t i = 0; i < times; ++i) c.rec(op, level, arg);
}
}  // namespace

DCt make_ct(Ctx &c, uint32_t level, uint32_t npolys, uint32_t n_slots, double scale, uint32_t batch)
{
    DCt r;
    r.n = c.n;
    r.level = level;
    r.npolys = npolys;
    r.n_slots = n_slots;
    r.scale = scale;
    r.batch = batch;
    r.buf = DBuf(r.item_words() * batch, c.stream);
    return r;
}

DCt view_ct(const Ctx &c, const mmfhe_ct &ct, uint32_t npolys)
{
    DCt r;
    r.ext = ct.data;
    r.n = c.n;
    r.level = ct.level;
    r.npolys = npolys;
    r.n_slots = ct.n_slots;
    r.scale = ct.scale;
    r.batch = 1;
    return r;
}

DCt slice(const DCt &a, uint32_t start, uint32_t count)
{
    MMFHE_REQUIRE(start + count <= a.batch, MMFHE_E_LAYOUT, "slice out of range");
    DCt r;
    r.ext = a.item(start);
    r.n = a.n;
    r.level = a.level;
    r.npolys = a.npolys;
    r.n_slots = a.n_slots;
    r.scale = a.scale;
    r.batch = count;
    return r;
}

DCt copy_ct(Ctx &c, const DCt &a)
{
    DCt r = make_ct(c, a.level, a.npolys, a.n_slots, a.scale, a.batch);
    memcpy_d2d(c, r.data(), a.data(), a.item_words() * a.batch);
    return r;
}

DCt import_batch(Ctx &c, const mmfhe_ct *cts, size_t first, size_t step, size_t count)
{
    MMFHE_REQUIRE(count >= 1, MMFHE_E_SHAPE, "empty batch");
    const mmfhe_ct &c0 = cts[first];
    for (size_t i = 0; i < count; ++i) {
        const mmfhe_ct &x = cts[first + i * step];
        MMFHE_REQUIRE(x.data != nullptr, MMFHE_E_INVALID_ARG, "null ciphertext data");
        MMFHE_REQUIRE(x.log_n == c.log_n, MMFHE_E_PARAMS, "ring dimension mismatch");
        MMFHE_REQUIRE(x.level <= c.L, MMFHE_E_DEPTH, "level above the chain");
        MMFHE_REQUIRE(x.form == c0.form && (x.form == MMFHE_FORM_COEFF || x.form == MMFHE_FORM_EVAL),
                      MMFHE_E_FORMAT, "bad or mixed form");
        MMFHE_REQUIRE(x.level == c0.level && x.scale == c0.scale, MMFHE_E_SCALE, "inputs must share level and scale");
        MMFHE_REQUIRE((x.n_polys ? x.n_polys : 2) == 2, MMFHE_E_LAYOUT, "chain inputs are 2-poly ciphertexts");
    }
    DCt r = make_ct(c, c0.level, 2, c0.n_slots, c0.scale, (uint32_t)count);
    const size_t words = r.item_words();
    bool all_dev = true;
    for (size_t i = 0; i < count; ++i)
        all_dev = all_dev && cts[first + i * step].on_device && ((uintptr_t)cts[first + i * step].data % 16 == 0);
    if (all_dev && c0.form == MMFHE_FORM_EVAL) {
        // device NTT-form items already back to back: use them in place (like input_ct)
        bool contig = true;
        for (size_t i = 1; i < count && contig; ++i)
            contig = cts[first + i * step].data == (const uint64_t *)c0.data + i * words;
        if (contig) {
            DCt v = view_ct(c, c0, 2);
            v.batch = (uint32_t)count;
            return v;
        }
    }
    if (all_dev && c0.form == MMFHE_FORM_COEFF && 2 * (c0.level + 1) <= (uint32_t)kMapCap) {
        // uniformly strided device items: the NTT's col pass reads them in place (the
        // fused-source Barrett step is the identity on residues < q), no gather copy
        const ptrdiff_t S = count > 1 ? cts[first + step].data - c0.data : (ptrdiff_t)words;
        bool uniform = S >= (ptrdiff_t)words;
        for (size_t i = 2; i < count && uniform; ++i) uniform = cts[first + i * step].data == c0.data + i * S;
        if (uniform) {
            ColSrc src{};
            src.x = c0.data;
            src.xs = (size_t)S;
            src.period = 2 * (c0.level + 1);
            std::vector<uint32_t> pm;
            for (uint32_t t = 0; t < src.period; ++t) {
                src.src[t] = (uint8_t)t;
                pm.push_back(t % (c0.level + 1));
            }
            ntt_forward(c, r.data(), r.rows(), make_map(pm), &src);
            return r;
        }
    }
    if (all_dev) {  // one gather launch per 64 device items
        for (size_t s = 0; s < count; s += kMaxTerms) {
            PtrList P{};
            const int n = (int)std::min<size_t>(kMaxTerms, count - s);
            for (int i = 0; i < n; ++i) P.p[i] = cts[first + (s + i) * step].data;
            launch_gather(c, r.item((uint32_t)s), P, n, words);
        }
    } else {
        for (size_t i = 0; i < count; ++i) {
            const mmfhe_ct &x = cts[first + i * step];
            CUDA_CHECK(cudaMemcpyAsync(r.item((uint32_t)i), x.data, words * 8,
                                       x.on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, c.stream));
        }
    }
    if (c0.form == MMFHE_FORM_COEFF) ntt_forward(c, r.data(), r.rows(), qmap(c, c0.level));
    return r;
}

DCt import_ct(Ctx &c, const mmfhe_ct &in, uint32_t npolys)
{
    MMFHE_REQUIRE(in.data != nullptr, MMFHE_E_INVALID_ARG, "null ciphertext data");
    MMFHE_REQUIRE(in.log_n == c.log_n, MMFHE_E_PARAMS, "ring dimension mismatch");
    MMFHE_REQUIRE(in.level <= c.L, MMFHE_E_DEPTH, "level above the chain");
    MMFHE_REQUIRE(in.form == MMFHE_FORM_COEFF || in.form == MMFHE_FORM_EVAL, MMFHE_E_FORMAT, "bad form");
    DCt r = make_ct(c, in.level, npolys, in.n_slots, in.scale);
    CUDA_CHECK(cudaMemcpyAsync(r.data(), in.data, r.item_words() * 8,
                               in.on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, c.stream));
    if (in.form == MMFHE_FORM_COEFF) ntt_forward(c, r.data(), r.rows(), qmap(c, in.level));
    return r;
}

void export_ct(Ctx &c, const DCt &in, mmfhe_ct &out)
{
    MMFHE_REQUIRE(out.data != nullptr, MMFHE_E_INVALID_ARG, "null output buffer");
    MMFHE_REQUIRE(in.batch == 1, MMFHE_E_LAYOUT, "export one ciphertext at a time");
    const uint32_t rows = in.rows();
    const size_t words = in.item_words();
    out.log_n = c.log_n;
    out.level = in.level;
    out.scale = in.scale;
    out.n_slots = in.n_slots;
    out.n_polys = in.npolys;
    // coefficient form: out-of-place INTT straight from the library's buffer
    const InvSrc src{in.data(), words, c.n, rows, 1};
    if (out.on_device) {
        if (out.form == MMFHE_FORM_COEFF)
            ntt_inverse(c, out.data, rows, qmap(c, in.level), &src);
        else
            memcpy_d2d(c, out.data, in.data(), words);
    } else {
        DBuf tmp(words, c.stream);
        if (out.form == MMFHE_FORM_COEFF)
            ntt_inverse(c, tmp.get(), rows, qmap(c, in.level), &src);
        else
            memcpy_d2d(c, tmp.get(), in.data(), words);
        CUDA_CHECK(cudaMemcpyAsync(out.data, tmp.get(), words * 8, cudaMemcpyDeviceToHost, c.stream));
        CUDA_CHECK(cudaStreamSynchronize(c.stream));
    }
}

PrimeMap pq_item_map(const Ctx &c, uint32_t l);

void export_pq(Ctx &c, const DCt &in, mmfhe_ct &out)
{
    MMFHE_REQUIRE(out.data != nullptr, MMFHE_E_INVALID_ARG, "null output buffer");
    MMFHE_REQUIRE(in.batch == 1 && in.pk == c.K && in.npolys == 2, MMFHE_E_LAYOUT, "export one PQ ciphertext");
    const uint32_t rows = in.rows();
    const size_t words = in.item_words();
    out.log_n = c.log_n;
    out.level = in.level;
    out.scale = in.scale;
    out.n_slots = in.n_slots;
    out.n_polys = 2;
    const InvSrc src{in.data(), words, c.n, rows, 1};
    uint64_t *dst = out.data;
    DBuf tmp;
    if (!out.on_device) {
        tmp = DBuf(words, c.stream);
        dst = tmp.get();
    }
    if (out.form == MMFHE_FORM_COEFF)
        ntt_inverse(c, dst, rows, pq_item_map(c, in.level), &src);
    else
        memcpy_d2d(c, dst, in.data(), words);
    if (!out.on_device) {
        CUDA_CHECK(cudaMemcpyAsync(out.data, dst, words * 8, cudaMemcpyDeviceToHost, c.stream));
        CUDA_CHECK(cudaStreamSynchronize(c.stream));
    }
}

// Every item of a batch to its own output: one out-of-place INTT of the whole batch into a
// staging buffer (coefficient-form outputs), then one scatter launch per 64 device outputs
// or one D2H copy per host output -- instead of two INTT launches per ciphertext.
void export_batch(Ctx &c, const DCt &in, mmfhe_ct *outs)
{
    const uint32_t B = in.batch;
    bool uniform = B > 1;
    for (uint32_t b = 0; uniform && b < B; ++b) {
        const mmfhe_ct &o = outs[b];
        uniform = o.data != nullptr && o.form == outs[0].form && o.on_device == outs[0].on_device &&
                  (!o.on_device || ((uintptr_t)o.data & 15) == 0);
    }
    if (!uniform) {
        for (uint32_t b = 0; b < B; ++b) export_ct(c, slice(in, b, 1), outs[b]);
        return;
    }
    const size_t words = in.item_words();
    const uint32_t rows = in.rows() / B;  // per item
    const uint64_t *src = in.data();
    DBuf tmp;
    if (outs[0].form == MMFHE_FORM_COEFF) {
        tmp = DBuf(words * B, c.stream);
        const InvSrc is{in.data(), words, c.n, rows, 1};
        ntt_inverse(c, tmp.get(), rows * B, qmap(c, in.level), &is);
        src = tmp.get();
    }
    for (uint32_t b = 0; b < B; ++b) {
        mmfhe_ct &o = outs[b];
        o.log_n = c.log_n;
        o.level = in.level;
        o.scale = in.scale;
        o.n_slots = in.n_slots;
        o.n_polys = in.npolys;
    }
    if (outs[0].on_device) {
        for (uint32_t b0 = 0; b0 < B; b0 += kMaxTerms) {
            const int n = (int)std::min<uint32_t>(kMaxTerms, B - b0);
            PtrList dst{};
            for (int i = 0; i < n; ++i) dst.p[i] = outs[b0 + i].data;
            launch_scatter(c, dst, src + (size_t)b0 * words, n, words);
        }
    } else {
        for (uint32_t b = 0; b < B; ++b)
            CUDA_CHECK(cudaMemcpyAsync(outs[b].data, src + (size_t)b * words, words * 8, cudaMemcpyDeviceToHost,
                                       c.stream));
        CUDA_CHECK(cudaStreamSynchronize(c.stream));
    }
}

// ------------------------------------------------------------------ exact ops
DCt make_pq(Ctx &c, uint32_t level, uint32_t n_slots, double scale, uint32_t batch);
PrimeMap pq_item_map(const Ctx &c, uint32_t l);

DCt ev_addsub(Ctx &c, const DCt &a, const DCt &b, bool sub)
{
    MMFHE_REQUIRE(a.level == b.level && a.npolys == b.npolys && a.batch == b.batch && a.pk == b.pk, MMFHE_E_LAYOUT,
                  "hadd level/size mismatch");
    MMFHE_REQUIRE(a.scale == b.scale, MMFHE_E_SCALE, "hadd scale mismatch");
    if (a.pk) {  // PQ ciphertexts (double hoisting)
        MMFHE_REQUIRE(!sub && a.npolys == 2, MMFHE_E_LAYOUT, "PQ ciphertexts: 2-poly sums only");
        rec_n(c, "hadd_pq", a.level, a.batch);
        DCt r = make_pq(c, a.level, a.n_slots, a.scale, a.batch);
        launch_addsub(c, r.data(), a.data(), b.data(), a.rows(), pq_item_map(c, a.level), false);
        return r;
    }
    rec_n(c, sub ? "hsub" : "hadd", a.level, a.batch);
    DCt r = make_ct(c, a.level, a.npolys, a.n_slots, a.scale, a.batch);
    launch_addsub(c, r.data(), a.data(), b.data(), a.rows(), qmap(c, a.level), sub);
    return r;
}

DCt ev_sum(Ctx &c, const std::vector<const DCt *> &cts)
{
    MMFHE_REQUIRE(!cts.empty(), MMFHE_E_INVALID_ARG, "empty sum");
    const DCt &a0 = *cts[0];
    DCt r = copy_ct(c, a0);
    for (size_t i = 1; i < cts.size(); ++i) {
        const DCt &b = *cts[i];
        MMFHE_REQUIRE(b.level == a0.level && b.npolys == a0.npolys && b.batch == a0.batch, MMFHE_E_LAYOUT,
                      "sum level mismatch");
        MMFHE_REQUIRE(b.scale == a0.scale, MMFHE_E_SCALE, "sum scale mismatch");
        rec_n(c, "hadd", a0.level, a0.batch);
        launch_addsub(c, r.data(), r.data(), b.data(), a0.rows(), qmap(c, a0.level), false);
    }
    return r;
}

DCt ev_batch_sum(Ctx &c, const DCt &a)
{
    rec_n(c, "hadd", a.level, a.batch - 1);
    DCt r = make_ct(c, a.level, a.npolys, a.n_slots, a.scale, 1);
    launch_batch_sum(c, r.data(), a.data(), a.batch, a.npolys, a.level);
    return r;
}

DCt ev_batch_sum_runs(Ctx &c, const DCt &a, uint32_t S)
{
    MMFHE_REQUIRE(S >= 1 && a.batch % S == 0, MMFHE_E_SHAPE, "batch does not split into equal runs");
    const uint32_t g = a.batch / S;
    for (uint32_t s = 0; s < S; ++s) rec_n(c, "hadd", a.level, g - 1);
    DCt r = make_ct(c, a.level, a.npolys, a.n_slots, a.scale, S);
    for (uint32_t s = 0; s < S; ++s)
        launch_batch_sum(c, r.data() + (size_t)s * r.item_words(), a.data() + (size_t)s * g * a.item_words(), g,
                         a.npolys, a.level);
    return r;
}

DCt ev_drop_to(Ctx &c, const DCt &a, uint32_t level)
{
    MMFHE_REQUIRE(level <= a.level, MMFHE_E_DEPTH, "cannot raise a level");
    DCt r = make_ct(c, level, a.npolys, a.n_slots, a.scale, a.batch);
    if (level != a.level) rec_n(c, "modswitch", a.level, a.batch, std::to_string(level));
    CUDA_CHECK(cudaMemcpy2DAsync(r.data(), r.poly_words() * 8, a.data(), a.poly_words() * 8, r.poly_words() * 8,
                                 (size_t)a.npolys * a.batch, cudaMemcpyDeviceToDevice, c.stream));
    return r;
}

DCt ev_tensor_sum(Ctx &c, const std::vector<std::pair<const DCt *, const DCt *>> &pairs)
{
    MMFHE_REQUIRE(!pairs.empty(), MMFHE_E_INVALID_ARG, "empty tensor sum");
    const DCt &a0 = *pairs[0].first;
    const double sc = a0.scale * pairs[0].second->scale;
    for (auto &pr : pairs) {
        for (const DCt *x : {pr.first, pr.second}) {
            MMFHE_REQUIRE(x->level == a0.level && x->batch == a0.batch, MMFHE_E_LAYOUT, "tensor level/batch mismatch");
            MMFHE_REQUIRE(x->npolys == 2, MMFHE_E_LAYOUT, "tensor needs 2-poly cts");
        }
        MMFHE_REQUIRE(pr.first->scale * pr.second->scale == sc, MMFHE_E_SCALE, "tensor_sum scale mismatch");
    }
    rec_n(c, "tensor_sum", a0.level, a0.batch, std::to_string(pairs.size()));
    DCt r = make_ct(c, a0.level, 3, a0.n_slots, sc, a0.batch);
    for (size_t s = 0; s < pairs.size(); s += kMaxTerms) {
        PtrList A{}, B{};
        int n = (int)std::min<size_t>(kMaxTerms, pairs.size() - s);
        for (int i = 0; i < n; ++i) {
            A.p[i] = pairs[s + i].first->data();
            B.p[i] = pairs[s + i].second->data();
        }
        launch_tensor_sum(c, r.data(), r.item_words(), A, B, a0.item_words(), n, a0.level, s > 0, a0.batch);
    }
    return r;
}

// K1 over session-major inputs: all = [S][m] contiguous items; out_s = sum_{t<m} x_{s,t} (x) x_{s,t}
// (the same op and trace as ev_tensor_sum over the m per-frame batches of S sessions, without
// gathering those batches: operand t is at item offset t with item stride m)
DCt ev_square_sum_items(Ctx &c, const DCt &all, uint32_t m, uint32_t S)
{
    MMFHE_REQUIRE(all.npolys == 2 && m >= 1 && all.batch == m * S, MMFHE_E_LAYOUT, "square sum layout");
    rec_n(c, "tensor_sum", all.level, S, std::to_string(m));
    DCt r = make_ct(c, all.level, 3, all.n_slots, all.scale * all.scale, S);
    for (uint32_t s0 = 0; s0 < m; s0 += kMaxTerms) {
        PtrList A{};
        const int n = (int)std::min<uint32_t>(kMaxTerms, m - s0);
        for (int i = 0; i < n; ++i) A.p[i] = all.item(s0 + i);
        launch_tensor_sum(c, r.data(), r.item_words(), A, A, (size_t)m * all.item_words(), n, all.level, s0 > 0, S);
    }
    return r;
}

DCt ev_pmult_sum(Ctx &c, const std::vector<std::pair<const DPlain *, const DCt *>> &terms)
{
    MMFHE_REQUIRE(!terms.empty(), MMFHE_E_INVALID_ARG, "empty pmult sum");
    const DCt &a0 = *terms[0].second;
    const double sc = a0.scale * terms[0].first->scale;
    for (auto &t : terms) {
        MMFHE_REQUIRE(t.second->level == a0.level && t.second->npolys == 2 && t.second->batch == a0.batch,
                      MMFHE_E_LAYOUT, "pmult level/batch mismatch");
        MMFHE_REQUIRE(t.first->level == a0.level, MMFHE_E_LAYOUT, "plaintext level mismatch");
        MMFHE_REQUIRE(t.second->scale * t.first->scale == sc, MMFHE_E_SCALE, "pmult_sum scale mismatch");
    }
    rec_n(c, "pmult_sum", a0.level, a0.batch, std::to_string(terms.size()));
    DCt r = make_ct(c, a0.level, 2, a0.n_slots, sc, a0.batch);
    for (size_t s = 0; s < terms.size(); s += kMaxTerms) {
        PtrList P{}, C{};
        int n = (int)std::min<size_t>(kMaxTerms, terms.size() - s);
        for (int i = 0; i < n; ++i) {
            P.p[i] = terms[s + i].first->buf.get();
            C.p[i] = terms[s + i].second->data();
        }
        launch_pmult_sum(c, r.data(), r.item_words(), P, C, a0.item_words(), n, a0.level, s > 0, a0.batch);
    }
    return r;
}

std::vector<DCt> ev_diag_mac(Ctx &c, const std::vector<const DCt *> &cts,
                             const std::vector<std::vector<const DPlain *>> &pts)
{
    MMFHE_REQUIRE(!cts.empty() && !pts.empty(), MMFHE_E_INVALID_ARG, "empty diagonal MAC");
    const DCt &a0 = *cts[0];
    for (auto *x : cts)
        MMFHE_REQUIRE(x->level == a0.level && x->batch == a0.batch && x->npolys == 2 && x->scale == a0.scale &&
                          x->pk == a0.pk,
                      MMFHE_E_LAYOUT, "diag MAC operands must share level, batch, basis and scale");
    std::vector<DCt> out;
    const bool fused = cts.size() <= (size_t)kDiagIn && pts.size() <= (size_t)kDiagMax;
    MMFHE_REQUIRE(fused || !a0.pk, MMFHE_E_LAYOUT, "PQ diagonal MAC: at most 32 baby steps and 16 outputs");
    std::vector<const uint64_t *> ctp;
    for (auto *x : cts) ctp.push_back(x->data());
    std::vector<std::vector<const uint64_t *>> ptp;
    std::vector<uint64_t *> outp;
    for (const auto &row : pts) {
        MMFHE_REQUIRE(row.size() == cts.size(), MMFHE_E_LAYOUT, "diag MAC row size");
        double sc = 0;
        int cnt = 0;
        std::vector<const uint64_t *> rp;
        std::vector<std::pair<const DPlain *, const DCt *>> terms;
        for (size_t i = 0; i < row.size(); ++i) {
            const DPlain *p = row[i];
            rp.push_back(p ? p->buf.get() : nullptr);
            if (!p) continue;
            MMFHE_REQUIRE(p->level == a0.level && p->pk == a0.pk, MMFHE_E_LAYOUT, "plaintext level / basis mismatch");
            const double s = a0.scale * p->scale;
            MMFHE_REQUIRE(cnt == 0 || s == sc, MMFHE_E_SCALE, "diag MAC scale mismatch");
            sc = s;
            ++cnt;
            terms.push_back({p, cts[i]});
        }
        MMFHE_REQUIRE(cnt > 0, MMFHE_E_INVALID_ARG, "diag MAC output without terms");
        if (!fused) {  // more than kDiagMax babies or outputs: one plaintext inner product per output
            out.push_back(ev_pmult_sum(c, terms));
            continue;
        }
        rec_n(c, a0.pk ? "pmult_sum_pq" : "pmult_sum", a0.level, a0.batch, std::to_string(cnt));
        out.push_back(a0.pk ? make_pq(c, a0.level, a0.n_slots, sc, a0.batch)
                            : make_ct(c, a0.level, 2, a0.n_slots, sc, a0.batch));
        ptp.push_back(rp);
        outp.push_back(out.back().data());
    }
    if (fused)
        launch_diag_mac(c, ctp, a0.item_words(), ptp, outp, out[0].item_words(), a0.level, a0.batch, a0.pk);
    return out;
}

std::vector<DCt> ev_k3_mac(Ctx &c, const std::vector<const DCt *> &xr, const std::vector<const DCt *> &xi,
                           const std::vector<std::vector<const DPlain *>> &pc,
                           const std::vector<std::vector<const DPlain *>> &ps,
                           const std::vector<std::vector<const DPlain *>> &pns)
{
    MMFHE_REQUIRE(!xr.empty() && xr.size() == xi.size() && !pc.empty(), MMFHE_E_INVALID_ARG, "empty K3 MAC");
    const DCt &a0 = *xr[0];
    std::vector<const uint64_t *> r, i;
    for (size_t s = 0; s < xr.size(); ++s) {
        for (const DCt *x : {xr[s], xi[s]})
            MMFHE_REQUIRE(x->level == a0.level && x->batch == a0.batch && x->npolys == 2 && x->scale == a0.scale &&
                              x->pk == a0.pk,
                          MMFHE_E_LAYOUT, "K3 MAC operands must share level, batch, basis and scale");
        r.push_back(xr[s]->data());
        i.push_back(xi[s]->data());
    }
    std::vector<std::vector<const uint64_t *>> C(pc.size()), S(pc.size()), NS(pc.size());
    std::vector<DCt> out;
    std::vector<uint64_t *> re, im;
    for (size_t g = 0; g < pc.size(); ++g) {
        double sc = 0;
        int cnt = 0;
        for (size_t s = 0; s < xr.size(); ++s) {
            const DPlain *p = pc[g][s];
            C[g].push_back(p ? p->buf.get() : nullptr);
            S[g].push_back(p ? ps[g][s]->buf.get() : nullptr);
            NS[g].push_back(p ? pns[g][s]->buf.get() : nullptr);
            if (!p) continue;
            for (const DPlain *x : {pc[g][s], ps[g][s], pns[g][s]})
                MMFHE_REQUIRE(x->level == a0.level && x->pk == a0.pk && x->scale == p->scale, MMFHE_E_LAYOUT,
                              "plaintext level / basis / scale mismatch");
            const double v = a0.scale * p->scale;
            MMFHE_REQUIRE(cnt == 0 || v == sc, MMFHE_E_SCALE, "K3 MAC scale mismatch");
            sc = v;
            cnt += 2;
        }
        MMFHE_REQUIRE(cnt > 0, MMFHE_E_INVALID_ARG, "giant step without terms");
        for (int part = 0; part < 2; ++part)
            rec_n(c, a0.pk ? "pmult_sum_pq" : "pmult_sum", a0.level, a0.batch, std::to_string(cnt));
        // one 2B batch per giant: its d_re items, then its d_im items (the giant rotations of
        // both then run as one launch set sharing the key)
        out.push_back(a0.pk ? make_pq(c, a0.level, a0.n_slots, sc, 2 * a0.batch)
                            : make_ct(c, a0.level, 2, a0.n_slots, sc, 2 * a0.batch));
        re.push_back(out.back().data());
        im.push_back(out.back().item(a0.batch));
    }
    launch_k3_gauss_mac(c, r, i, a0.item_words(), C, S, NS, re, im, out[0].item_words(), a0.level, a0.batch, a0.pk);
    return out;
}

uint64_t encode_scalar_mod(double v, uint64_t q_scale, uint64_t m)
{
    // v = mant * 2^e exactly with mant < 2^53; |x| = mant * q_scale * 2^e rounded
    // half away from zero, exactly, in 128-bit integers.
    typedef unsigned __int128 u128;
    if (v == 0.0) return 0;
    MMFHE_REQUIRE(std::isfinite(v), MMFHE_E_INVALID_ARG, "non-finite scalar");
    int e;
    double f = std::frexp(std::fabs(v), &e);  // |v| = f * 2^e, f in [0.5, 1)
    uint64_t mant = (uint64_t)std::ldexp(f, 53);
    e -= 53;
    u128 prod = (u128)mant * q_scale;  // < 2^113
    u128 mag;
    if (e >= 0) {
        MMFHE_REQUIRE(e < 14, MMFHE_E_SCALE, "scalar constant overflows the encoding");
        mag = prod << e;
    } else if (-e >= 120) {
        mag = 0;
    } else {
        u128 half = (u128)1 << (-e - 1);
        mag = (prod + half) >> (-e);
    }
    uint64_t r = (uint64_t)(mag % m);
    return (v < 0 && r) ? m - r : r;
}

DCt ev_lincomb_mat(Ctx &c, const DCt &in, uint32_t J, uint32_t W, int lo0, int lo_step,
                   const std::vector<double> &coef)
{
    MMFHE_REQUIRE(in.npolys == 2 && J >= 1 && W >= 1 && coef.size() == (size_t)J * W, MMFHE_E_SHAPE,
                  "lincomb matrix shape");
    const uint32_t l = in.level, M = in.batch;
    const uint64_t ql = c.primes[l];
    for (uint32_t j = 0; j < J; ++j) {
        int cnt = 0;
        for (uint32_t w = 0; w < W; ++w) {
            const int i = lo0 + (int)j * lo_step + (int)w;
            cnt += (i >= 0 && i < (int)M);
        }
        MMFHE_REQUIRE(cnt > 0, MMFHE_E_SHAPE, "lincomb output without inputs");
        c.rec("lincomb", l, std::to_string(cnt));
    }
    std::string key = "mat:" + std::to_string(l) + ":" + std::to_string(J) + ":" + std::to_string(W) + ":";
    key.append((const char *)coef.data(), coef.size() * sizeof(double));
    auto it = c.const_cache.find(key);
    if (it == c.const_cache.end()) {
        std::vector<TwPair> tab(coef.size() * (l + 1));
        for (size_t t = 0; t < coef.size(); ++t)
            for (uint32_t i = 0; i <= l; ++i) {
                // (value, Montgomery form): the lincomb kernels multiply-accumulate in 128 bits
                const uint64_t v = encode_scalar_mod(coef[t], ql, c.primes[i]);
                tab[t * (l + 1) + i] = {v, host::to_mont(v, c.primes[i])};
            }
        DBuf b((tab.size() * sizeof(TwPair) + 7) / 8, c.stream);
        CUDA_CHECK(cudaMemcpyAsync(b.get(), tab.data(), tab.size() * sizeof(TwPair), cudaMemcpyHostToDevice,
                                   c.stream));
        CUDA_CHECK(cudaStreamSynchronize(c.stream));
        it = c.const_cache.emplace(key, std::move(b)).first;
    }
    DCt r = make_ct(c, l, 2, in.n_slots, in.scale * (double)ql, J);
    // Toeplitz rows with one symmetric tap vector (linear-phase FIR): equal doubles encode to
    // equal residues, so pairing the mirrored inputs before the product is exact
    bool sym = lo_step == 1 && W >= 2 && W <= 129;
    for (uint32_t w = 0; sym && w < W; ++w) sym = coef[w] == coef[W - 1 - w];
    for (size_t t = W; sym && t < coef.size(); ++t) sym = coef[t] == coef[t % W];
    if (sym)
        launch_lincomb_sym(c, r.data(), in.data(), M, J, W, lo0, (const TwPair *)it->second.get(), l);
    else
        launch_lincomb_mat(c, r.data(), in.data(), M, J, W, lo0, lo_step, (const TwPair *)it->second.get(), l);
    return r;
}

DCt ev_add_plain(Ctx &c, const DCt &a, const DPlain &pt)
{
    MMFHE_REQUIRE(pt.level == a.level && a.npolys == 2, MMFHE_E_LAYOUT, "plaintext level mismatch");
    MMFHE_REQUIRE(pt.scale == a.scale, MMFHE_E_SCALE, "add_plain scale mismatch");
    rec_n(c, "add_plain", a.level, a.batch);
    DCt r = copy_ct(c, a);
    launch_add_plain(c, r.data(), r.item_words(), pt.buf.get(), a.level, a.batch);
    return r;
}

// ------------------------------------------------------------------ key switching
namespace {
// ModUp of B polynomials x_b (NTT form, item stride xs): y [B][T][N] in NTT form,
// digit j's n_tgt rows at offset off[j] (rows inside I_j are x itself and not stored).
struct ModUpOut {
    DBuf y;
    std::vector<size_t> off;
    std::vector<uint32_t> rowmap;
    size_t T = 0;
};

// g != 1: ModUp of sigma_g(x) (the rotation's permutation fused into the INTT's first read).
ModUpOut ks_modup(Ctx &c, const uint64_t *x_ntt, size_t xs, uint32_t l, uint32_t B, uint32_t g = 1)
{
    const size_t N = c.n;
    const size_t lw = (size_t)(l + 1) * N;
    ModUpOut m;
    // coefficient form of every x_b (or sigma_g(x_b)): out-of-place INTT, no staging copy
    DBuf xc(B * lw, c.stream);
    const InvSrc src{x_ntt, xs, N, l + 1, g};
    ntt_inverse(c, xc.get(), B * (l + 1), qmap(c, l), &src);
    // fast BConv of every digit, then NTT of the converted rows
    const auto &plans = c.modup[l];
    const std::vector<uint32_t> basis = c.ext_basis(l);
    for (const auto &p : plans) {
        m.off.push_back(m.T);
        for (uint32_t r = 0; r < basis.size(); ++r)
            if (r < p.lo || r >= p.hi) m.rowmap.push_back(basis[r]);
        m.T += p.n_tgt;
    }
    m.y = DBuf(B * m.T * N, c.stream);
    bool single = m.T <= (size_t)kMapCap;
    for (const auto &p : plans) single = single && p.hi - p.lo == 1;
    if (single) {
        // single-limb digits: BConv is y = x_j mod q_t, fused into the NTT's first read
        ColSrc src{};
        src.x = xc.get();
        src.xs = lw;
        src.period = (uint32_t)m.T;
        size_t t = 0;
        for (const auto &p : plans)
            for (uint32_t i = 0; i < p.n_tgt; ++i) {
                // x_j < q_j < 2 q_t: already a valid NTT input, no reduction on load
                if (c.primes[p.lo] < 2 * c.primes[m.rowmap[t]]) src.below2q[t >> 5] |= 1u << (t & 31);
                src.src[t++] = (uint8_t)p.lo;
            }
        ntt_forward(c, m.y.get(), (uint32_t)(B * m.T), make_map(m.rowmap), &src);
    } else {
        launch_modup_bconv(c, m.y.get(), m.T * N, xc.get(), lw, l, m.off, B);
        ntt_forward(c, m.y.get(), (uint32_t)(B * m.T), make_map(m.rowmap));
    }
    return m;
}

// ModDown of npoly polynomials per item, NTT form in and out:
//   out = (X - NTT(BConv_{P->Q}(INTT(Pr)))) P^{-1} (+ addends)
// X: the Q rows (item stride xs, poly stride xps); Pr: the P rows (item stride prs, the
// item's npoly*K rows contiguous).  The final step (X - w) P^{-1} + addends is the epilogue
// of w's forward NTT row pass: w never goes to HBM.  Poly 0's addend add0 is read through
// sigma_g0 (NTT-domain gather; 1 = none); add2 is a second, unpermuted poly-0 addend.
void moddown(Ctx &c, const uint64_t *X, size_t xs, size_t xps, const uint64_t *Pr, size_t prs, uint32_t l, uint32_t B,
             uint32_t npoly, uint64_t *out, size_t os, size_t ops, const uint64_t *add0 = nullptr,
             const uint64_t *add1 = nullptr, size_t as = 0, uint32_t g0 = 1, const uint64_t *add2 = nullptr)
{
    const size_t N = c.n;
    std::vector<uint32_t> pm;
    for (uint32_t k = 0; k < c.K; ++k) pm.push_back(c.L + 1 + k);
    DBuf zP((size_t)B * npoly * c.K * N, c.stream);
    const InvSrc isrc{Pr, prs, N, npoly * c.K, 1};
    ntt_inverse(c, zP.get(), B * npoly * c.K, make_map(pm), &isrc);
    RowEpi ep{};
    ep.out = out;
    ep.X = X;
    ep.mul = (const TwPair *)c.bconv_ptr(c.off_pd_pinv);
    ep.add0 = add0;
    ep.add1 = add1;
    ep.add2 = add2;
    ep.os = os;
    ep.ops = ops;
    ep.xs = xs;
    ep.xps = xps;
    ep.as = as;
    ep.per = l + 1;
    ep.g0 = g0;
    ep.npoly = npoly;
    DBuf w((size_t)B * npoly * (l + 1) * N, c.stream);
    if (c.K == 1 && l + 1 <= (uint32_t)kMapCap) {
        // one special prime: BConv_{P->Q} is w_i = zP mod q_i, fused into the NTT's first read
        ColSrc src{};
        src.x = zP.get();
        src.xs = N;  // one P row per (item, poly)
        src.period = l + 1;
        for (uint32_t i = 0; i <= l; ++i)
            if (c.primes[c.L + 1] < 2 * c.primes[i]) src.below2q[i >> 5] |= 1u << (i & 31);
        ntt_forward(c, w.get(), B * npoly * (l + 1), qmap(c, l), &src, &ep);
    } else {
        launch_moddown_bconv(c, w.get(), zP.get(), l, B, npoly);
        ntt_forward(c, w.get(), B * npoly * (l + 1), qmap(c, l), nullptr, &ep);
    }
}

// Key inner product (each evk word fetched once per batch split) + ModDown.  The x / y
// reads of the inner product go through sigma_gx / sigma_gy and poly 0's addend through
// sigma_g0 (NTT-domain gathers fused into the kernels; 1 = none); add2 is a second,
// unpermuted poly-0 addend.
void ks_ip_moddown(Ctx &c, const uint64_t *x_ntt, size_t xs, const uint64_t *y, const ModUpOut &m, uint32_t l,
                   uint32_t B, const DKey &key, uint64_t *out, size_t os, const uint64_t *add0,
                   const uint64_t *add1, size_t as, uint32_t gx = 1, uint32_t gy = 1, uint32_t g0 = 1,
                   const uint64_t *add2 = nullptr)
{
    const size_t N = c.n;
    const size_t lw = (size_t)(l + 1) * N;
    DBuf accQ(B * 2 * lw, c.stream), accP(B * 2 * c.K * N, c.stream);
    launch_key_ip(c, accQ.get(), accP.get(), x_ntt, xs, y, m.T * N, m.off, key.buf.get(), l, B, gx, gy);
    moddown(c, accQ.get(), 2 * lw, lw, accP.get(), 2 * c.K * N, l, B, 2, out, os, lw, add0, add1, as, g0, add2);
}
}  // namespace

// PQ ciphertext batch (double hoisting): [2][l+1] Q rows then [2][K] P rows per item
DCt make_pq(Ctx &c, uint32_t level, uint32_t n_slots, double scale, uint32_t batch)
{
    DCt r;
    r.n = c.n;
    r.level = level;
    r.npolys = 2;
    r.pk = c.K;
    r.n_slots = n_slots;
    r.scale = scale;
    r.batch = batch;
    r.buf = DBuf(r.item_words() * batch, c.stream);
    return r;
}

// row -> prime map of one PQ item: Q rows of both polys, then P rows of both polys
PrimeMap pq_item_map(const Ctx &c, uint32_t l)
{
    std::vector<uint32_t> v;
    for (int p = 0; p < 2; ++p)
        for (uint32_t i = 0; i <= l; ++i) v.push_back(i);
    for (int p = 0; p < 2; ++p)
        for (uint32_t k = 0; k < c.K; ++k) v.push_back(c.L + 1 + k);
    return make_map(v);
}

void ev_keyswitch(Ctx &c, const uint64_t *x_ntt, size_t xs, uint32_t l, uint32_t B, const DKey &key,
                  uint64_t *out, size_t os, const uint64_t *add0, const uint64_t *add1, size_t as)
{
    ModUpOut m = ks_modup(c, x_ntt, xs, l, B);
    ks_ip_moddown(c, x_ntt, xs, m.y.get(), m, l, B, key, out, os, add0, add1, as);
}

std::vector<DCt> ev_rotate_hoisted(Ctx &c, const DCt &a, const std::vector<int32_t> &steps)
{
    MMFHE_REQUIRE(a.npolys == 2, MMFHE_E_LAYOUT, "rotate needs a 2-poly ciphertext");
    const uint32_t l = a.level, B = a.batch;
    std::vector<DCt> out;
    bool need = false;
    for (int32_t s : steps) {
        int32_t k;
        galois_element(c, s, &k);
        if (k) {
            find_gk(c, k);  // fail before any work on a missing key
            need = true;
        }
    }
    ModUpOut m;
    if (need) m = ks_modup(c, a.poly(1), a.item_words(), l, B);
    for (int32_t s : steps) {
        int32_t k;
        const uint64_t g = galois_element(c, s, &k);
        if (k == 0) {
            out.push_back(copy_ct(c, a));
            continue;
        }
        const DKey &key = find_gk(c, k);
        rec_n(c, "hrot_hoisted", l, B, std::to_string(k));
        // sigma_g on (c0, c1) and on the ModUp'd digits is an NTT-domain permutation of
        // every row: applied inside the inner product's reads and ModDown's addend
        DCt r = make_ct(c, l, 2, a.n_slots, a.scale, B);
        const uint32_t g32 = (uint32_t)g;
        ks_ip_moddown(c, a.poly(1), a.item_words(), m.y.get(), m, l, B, key, r.data(), r.item_words(), a.data(),
                      nullptr, a.item_words(), g32, g32, g32);
        out.push_back(std::move(r));
    }
    return out;
}

DCt ev_relin(Ctx &c, const DCt &a3)
{
    MMFHE_REQUIRE(a3.npolys == 3, MMFHE_E_LAYOUT, "relin needs a 3-poly ciphertext");
    MMFHE_REQUIRE(c.rlk != nullptr, MMFHE_E_MISSING_KEY, "missing relinearisation key");
    rec_n(c, "relin", a3.level, a3.batch);
    DCt r = make_ct(c, a3.level, 2, a3.n_slots, a3.scale, a3.batch);
    ev_keyswitch(c, a3.poly(2), a3.item_words(), a3.level, a3.batch, *c.rlk, r.data(), r.item_words(), a3.data(),
                 a3.poly(1), a3.item_words());
    return r;
}

uint64_t galois_element(const Ctx &c, int32_t step, int32_t *normalised)
{
    if (step == MMFHE_STEP_CONJ) {  // complex conjugation of every slot (DESIGN R28)
        if (normalised) *normalised = MMFHE_STEP_CONJ;
        return 2ull * c.n - 1;
    }
    if (step == MMFHE_STEP_CONJ_PROD) {  // the conjugate-product key (R32): an id, no Galois element
        if (normalised) *normalised = MMFHE_STEP_CONJ_PROD;
        return 0;
    }
    const int64_t half = c.n / 2;
    int64_t k = ((int64_t)step % half + half) % half;
    if (normalised) *normalised = (int32_t)k;
    return host::pow(5, (uint64_t)k, 2ull * c.n);
}

const DKey &find_gk(const Ctx &c, int32_t k)
{
    auto it = c.gk.find(k);
    MMFHE_REQUIRE(it != c.gk.end(), MMFHE_E_MISSING_KEY,
                  k == MMFHE_STEP_CONJ        ? std::string("missing conjugation key")
                  : k == MMFHE_STEP_CONJ_PROD ? std::string("missing conjugate-product key")
                                              : "missing Galois key for rotation " + std::to_string(k));
    return *it->second;
}

namespace {
// HRot's algorithm for Galois element g (a rotation, or the conjugation)
DCt automorphism_ks(Ctx &c, const DCt &a, uint64_t g, const DKey &key)
{
    DCt r = make_ct(c, a.level, 2, a.n_slots, a.scale, a.batch);
    // sigma_g fused: into the INTT's first read (c1), the inner product's reads of the
    // digit-own rows (sigma_g c1) and ModDown's addend (sigma_g c0)
    const uint32_t g32 = (uint32_t)g;
    ModUpOut m = ks_modup(c, a.poly(1), a.item_words(), a.level, a.batch, g32);
    ks_ip_moddown(c, a.poly(1), a.item_words(), m.y.get(), m, a.level, a.batch, key, r.data(), r.item_words(),
                  a.data(), nullptr, a.item_words(), g32, 1, g32);
    return r;
}
}  // namespace

DCt ev_rotate(Ctx &c, const DCt &a, int32_t step)
{
    MMFHE_REQUIRE(a.npolys == 2, MMFHE_E_LAYOUT, "rotate needs a 2-poly ciphertext");
    MMFHE_REQUIRE(step != MMFHE_STEP_CONJ_PROD, MMFHE_E_INVALID_ARG, "the conjugate-product key is not a rotation");
    int32_t k;
    const uint64_t g = galois_element(c, step, &k);
    if (k == 0) return copy_ct(c, a);
    const DKey &key = find_gk(c, k);
    if (k == MMFHE_STEP_CONJ)
        rec_n(c, "conj", a.level, a.batch);
    else
        rec_n(c, "hrot", a.level, a.batch, std::to_string(k));
    return automorphism_ks(c, a, g, key);
}

// Conj (DESIGN R28, oracle Evaluator.conjugate): every slot value conjugated
DCt ev_conjugate(Ctx &c, const DCt &a) { return ev_rotate(c, a, MMFHE_STEP_CONJ); }

DCt ev_rescale(Ctx &c, const DCt &a)
{
    MMFHE_REQUIRE(a.npolys == 2, MMFHE_E_LAYOUT, "rescale needs a 2-poly ciphertext");
    MMFHE_REQUIRE(a.level >= 1, MMFHE_E_DEPTH, "depth exhausted");
    const uint32_t l = a.level, B = a.batch;
    rec_n(c, "rescale", l, B);
    const size_t N = c.n;
    // t = [a_l + floor(q_l/2)]_{q_l} in coefficient form, both polys of every item: one
    // out-of-place INTT whose last stage adds the rounding offset
    DBuf t(2 * N * B, c.stream);
    const InvSrc src{a.data() + (size_t)l * N, a.item_words(), a.poly_words(), 2, 1, 1};
    ntt_inverse(c, t.get(), 2 * B, make_map({l}), &src);
    // v_i = NTT_{q_i}(([t]_{q_i} - [h]_{q_i}) mod q_i) for i < l: reduction and subtraction
    // are the forward NTT's fused first read (row (poly, i) reads t's poly row)
    DBuf v((size_t)2 * l * N * B, c.stream);
    DCt r = make_ct(c, l - 1, 2, a.n_slots, a.scale / (double)c.primes[l], B);
    {
        std::vector<uint32_t> pm(2 * l);
        ColSrc cs{};
        cs.x = t.get();
        cs.xs = 2 * N;
        cs.period = 2 * l;
        cs.sub = (const uint64_t *)c.bconv_ptr(c.off_rs_h) + (size_t)l * (c.L + 1);  // [h]_{q_i}, h = floor(q_l/2)
        for (uint32_t r = 0; r < 2 * l; ++r) {
            pm[r] = r % l;
            cs.src[r] = (uint8_t)(r / l);
        }
        MMFHE_REQUIRE(2 * l <= (uint32_t)kMapCap, MMFHE_E_PARAMS, "too many limbs for the fused rescale");
        // final step out_i = (a_i - v_i) q_l^{-1} as the epilogue of v's row pass
        RowEpi ep{};
        ep.out = r.data();
        ep.X = a.data();
        ep.mul = (const TwPair *)c.bconv_ptr(c.off_rs) + (size_t)l * (c.L + 1);
        ep.os = r.item_words();
        ep.ops = r.poly_words();
        ep.xs = a.item_words();
        ep.xps = a.poly_words();
        ep.per = l;
        ep.g0 = 1;
        ntt_forward(c, v.get(), 2 * l * B, make_map(pm), &cs, &ep);
    }
    return r;
}

// acc + HRot(acc, step) with the HAdd fused: ModDown adds sigma(c0) + c0 to poly 0 and c1
// to poly 1 (records "hrot" then "hadd", as the two ops it replaces).
DCt ev_rot_add(Ctx &c, const DCt &a, const DCt &b, int32_t step)
{
    MMFHE_REQUIRE(a.npolys == 2 && b.npolys == 2, MMFHE_E_LAYOUT, "rotate needs a 2-poly ciphertext");
    MMFHE_REQUIRE(a.level == b.level && a.batch == b.batch && a.item_words() == b.item_words(), MMFHE_E_LAYOUT,
                  "rotate-add operands must share level and batch");
    MMFHE_REQUIRE(a.scale == b.scale, MMFHE_E_SCALE, "hadd scale mismatch");
    int32_t k;
    const uint64_t g = galois_element(c, step, &k);
    if (k == 0) return ev_addsub(c, a, b, false);
    const DKey &key = find_gk(c, k);
    rec_n(c, "hrot", b.level, b.batch, std::to_string(k));
    rec_n(c, "hadd", a.level, a.batch);
    DCt r = make_ct(c, a.level, 2, a.n_slots, a.scale, a.batch);
    // as ev_rotate on b, with ModDown adding sigma_g(b0) + a0 to poly 0 and a1 to poly 1
    const uint32_t g32 = (uint32_t)g;
    ModUpOut m = ks_modup(c, b.poly(1), b.item_words(), b.level, b.batch, g32);
    ks_ip_moddown(c, b.poly(1), b.item_words(), m.y.get(), m, b.level, b.batch, key, r.data(), r.item_words(),
                  b.data(), a.poly(1), a.item_words(), g32, 1, g32, a.data());
    return r;
}

DCt ev_rot_add(Ctx &c, const DCt &a, int32_t step) { return ev_rot_add(c, a, a, step); }

DCt ev_rotsum(Ctx &c, const DCt &a, uint32_t count, uint32_t stride)
{
    if (count <= 1) return copy_ct(c, a);
    DCt acc = ev_rot_add(c, a, (int32_t)stride);
    uint32_t step = 2 * stride;
    for (uint32_t n = 2; n < count; n *= 2, step *= 2) acc = ev_rot_add(c, acc, (int32_t)step);
    return acc;
}

// ------------------------------------------------------------------ double hoisting
// (SURVEY §8(c)-5 "a third op"; oracle Evaluator.lift_pq / hoisted_step_pq / rotate_pq /
// add_pq / moddown_ct, pmult_sum_pq)
DCt ev_rotsum_hoisted_pq(Ctx &c, const DCt &a, const std::vector<int32_t> &steps)
{
    MMFHE_REQUIRE(a.npolys == 2 && !a.pk, MMFHE_E_LAYOUT, "rotate needs a 2-poly Q ciphertext");
    const uint32_t l = a.level, B = a.batch;
    std::vector<const uint64_t *> keys;
    std::vector<uint32_t> gs;
    std::vector<int32_t> ks;
    for (int32_t s : steps) {
        int32_t k;
        const uint64_t g = galois_element(c, s, &k);
        MMFHE_REQUIRE(k != 0 && k != MMFHE_STEP_CONJ, MMFHE_E_INVALID_ARG, "hoisted rotate-and-sum steps are rotations");
        keys.push_back(find_gk(c, k).buf.get());
        gs.push_back((uint32_t)g);
        ks.push_back(k);
    }
    MMFHE_REQUIRE(!keys.empty() && keys.size() <= 64 && c.modup[l].size() <= 8, MMFHE_E_LAYOUT,
                  "hoisted rotate-and-sum: 1..64 steps, <= 8 digits");
    // the oracle's op sequence (rotsum_dh_all): lift, the PQ steps, their PQ additions
    rec_n(c, "lift_pq", l, B);
    for (int32_t k : ks) rec_n(c, "hrot_hoisted_pq", l, B, std::to_string(k));
    for (size_t i = 0; i < ks.size(); ++i) rec_n(c, "hadd_pq", l, B);
    ModUpOut m = ks_modup(c, a.poly(1), a.item_words(), l, B);
    DCt r = make_pq(c, l, a.n_slots, a.scale, B);
    launch_hoisted_rotsum_pq(c, r.data(), r.item_words(), a.poly(1), a.item_words(), m.y.get(), m.T * c.n, m.off,
                             a.data(), a.item_words(), keys, gs, l, B);
    return r;
}

DCt ev_lift_pq(Ctx &c, const DCt &a)
{
    MMFHE_REQUIRE(a.npolys == 2 && !a.pk, MMFHE_E_LAYOUT, "lift needs a 2-poly Q ciphertext");
    rec_n(c, "lift_pq", a.level, a.batch);
    DCt r = make_pq(c, a.level, a.n_slots, a.scale, a.batch);
    launch_pq_lift(c, r.data(), r.item_words(), r.poly_words(), a.data(), a.item_words(), a.poly_words(), a.level, 2,
                   a.batch, 1, false);
    CUDA_CHECK(cudaMemset2DAsync(r.ppoly(0), r.item_words() * 8, 0, (size_t)2 * c.K * c.n * 8, a.batch, c.stream));
    return r;
}

std::vector<DCt> ev_rotate_hoisted_pq(Ctx &c, const DCt &a, const std::vector<int32_t> &steps)
{
    MMFHE_REQUIRE(a.npolys == 2 && !a.pk, MMFHE_E_LAYOUT, "rotate needs a 2-poly Q ciphertext");
    const uint32_t l = a.level, B = a.batch;
    bool need = false;
    for (int32_t s : steps) {
        int32_t k;
        galois_element(c, s, &k);
        if (k) {
            find_gk(c, k);
            need = true;
        }
    }
    ModUpOut m;
    if (need) m = ks_modup(c, a.poly(1), a.item_words(), l, B);
    std::vector<DCt> out;
    // the group's nonzero steps in one launch per 16 (y, x and c0 read once); the kernel keeps
    // every batch item's digit and c0 words of its coefficient in shared memory, so its occupancy
    // falls with the batch: batches run as balanced chunks of at most kHoistChunk items (each
    // chunk re-reads the keys).  Measured at C4 (B = 13, r02bz): one launch 3.58 ms, 7 + 6 3.33,
    // 5 + 5 + 3 3.46.  With more than 4 digits one inner product per step
#ifndef MMFHE_HOIST_CHUNK
#define MMFHE_HOIST_CHUNK 8
#endif
    const uint32_t n_chunks = (B + MMFHE_HOIST_CHUNK - 1) / MMFHE_HOIST_CHUNK;
    const uint32_t kHoistChunk = (B + n_chunks - 1) / n_chunks;
    const bool grouped = need && c.modup[l].size() <= 4;
    if (grouped) {
        std::vector<const uint64_t *> keys;
        std::vector<uint32_t> ginv;
        std::vector<uint64_t *> outs;
        auto flush = [&] {
            if (keys.empty()) return;
            const size_t ow = out.back().item_words(), aw = a.item_words(), yw = m.T * c.n;
            for (uint32_t b0 = 0; b0 < B; b0 += kHoistChunk) {
                std::vector<uint64_t *> o(outs);
                for (auto &p : o) p += b0 * ow;
                launch_hoisted_ip_pq(c, a.poly(1) + b0 * aw, aw, m.y.get() + b0 * yw, yw, m.off, a.data() + b0 * aw,
                                     aw, keys, ginv, o, ow, l, std::min(kHoistChunk, B - b0));
            }
            keys.clear();
            ginv.clear();
            outs.clear();
        };
        for (int32_t s : steps) {
            int32_t k;
            const uint64_t g = galois_element(c, s, &k);
            if (k == 0) {
                out.push_back(ev_lift_pq(c, a));
                continue;
            }
            rec_n(c, "hrot_hoisted_pq", l, B, std::to_string(k));
            out.push_back(make_pq(c, l, a.n_slots, a.scale, B));
            keys.push_back(find_gk(c, k).buf.get());
            // g is odd; the units mod 2N = 2^(log N + 1) have order N: g^-1 = g^(N-1) mod 2N
            ginv.push_back((uint32_t)host::pow(g, c.n - 1, 2ull * c.n));
            outs.push_back(out.back().data());
            if (keys.size() == (size_t)kDiagMax) flush();
        }
        flush();
        return out;
    }
    for (int32_t s : steps) {
        int32_t k;
        const uint32_t g = (uint32_t)galois_element(c, s, &k);
        if (k == 0) {
            out.push_back(ev_lift_pq(c, a));
            continue;
        }
        const DKey &key = find_gk(c, k);
        rec_n(c, "hrot_hoisted_pq", l, B, std::to_string(k));
        DCt r = make_pq(c, l, a.n_slots, a.scale, B);
        const IPOut os{r.item_words(), r.poly_words(), r.item_words(), (size_t)c.K * c.n};
        // (P sigma_g(c0) + IP0, IP1): the P lift of sigma_g(c0) is the inner product's fused
        // poly-0 addend on the Q rows (none on the P rows: P = 0 mod p_k)
        IPEpi ep;
        ep.add = a.data();
        ep.pmod = (const TwPair *)c.bconv_ptr(c.off_pd_pmod);
        ep.as = a.item_words();
        ep.ag = g;
        launch_key_ip(c, r.data(), r.ppoly(0), a.poly(1), a.item_words(), m.y.get(), m.T * c.n, m.off, key.buf.get(),
                      l, B, g, g, &os, &ep);
        out.push_back(std::move(r));
    }
    return out;
}

namespace {
// the PQ giant step into `r` (fresh, or += with accumulate): ModDown(a1), sigma_g, ModUp, key
// inner product whose fused epilogue adds sigma_g(a0) over Q_l u P (and r's old contents)
void rotate_pq_into(Ctx &c, const DCt &a, uint32_t g, const DKey &key, DCt &r, bool accumulate)
{
    const uint32_t l = a.level, B = a.batch;
    const size_t lw = (size_t)(l + 1) * c.n;
    DBuf a1(lw * B, c.stream);
    moddown(c, a.poly(1), a.item_words(), 0, a.ppoly(1), a.item_words(), l, B, 1, a1.get(), lw, 0);
    ModUpOut m = ks_modup(c, a1.get(), lw, l, B, g);
    const IPOut os{r.item_words(), r.poly_words(), r.item_words(), (size_t)c.K * c.n};
    IPEpi ep;
    ep.add = a.data();
    ep.as = a.item_words();
    ep.apbase = (size_t)2 * (l + 1) * c.n;  // a0's P rows: the PQ item layout's P part, poly 0
    ep.ag = g;
    ep.accumulate = accumulate ? 1 : 0;
    launch_key_ip(c, r.data(), r.ppoly(0), a1.get(), lw, m.y.get(), m.T * c.n, m.off, key.buf.get(), l, B, g, 1, &os,
                  &ep);
}
}  // namespace

DCt ev_rotate_pq(Ctx &c, const DCt &a, int32_t step)
{
    MMFHE_REQUIRE(a.pk == c.K && a.npolys == 2, MMFHE_E_LAYOUT, "PQ rotation needs a PQ ciphertext");
    int32_t k;
    const uint32_t g = (uint32_t)galois_element(c, step, &k);
    const uint32_t l = a.level, B = a.batch;
    DCt r = make_pq(c, l, a.n_slots, a.scale, B);
    if (k == 0) {
        CUDA_CHECK(cudaMemcpyAsync(r.data(), a.data(), a.item_words() * B * 8, cudaMemcpyDeviceToDevice, c.stream));
        return r;
    }
    const DKey &key = find_gk(c, k);
    rec_n(c, "hrot_pq", l, B, std::to_string(k));
    rotate_pq_into(c, a, g, key, r, false);
    return r;
}

void ev_rotate_pq_acc(Ctx &c, DCt &acc, const DCt &a, int32_t step)
{
    MMFHE_REQUIRE(a.pk == c.K && acc.pk == c.K && a.npolys == 2 && a.level == acc.level && a.batch == acc.batch,
                  MMFHE_E_LAYOUT, "PQ rotate-accumulate needs PQ ciphertexts of one shape");
    MMFHE_REQUIRE(a.scale == acc.scale, MMFHE_E_SCALE, "hadd scale mismatch");
    int32_t k;
    const uint32_t g = (uint32_t)galois_element(c, step, &k);
    if (k == 0) {
        DCt s = ev_addsub(c, acc, a, false);
        acc = std::move(s);
        return;
    }
    const DKey &key = find_gk(c, k);
    rec_n(c, "hrot_pq", a.level, a.batch, std::to_string(k));
    rec_n(c, "hadd_pq", a.level, a.batch);
    rotate_pq_into(c, a, g, key, acc, true);
}

DCt ev_moddown_ct(Ctx &c, const DCt &a)
{
    MMFHE_REQUIRE(a.pk == c.K && a.npolys == 2, MMFHE_E_LAYOUT, "ModDown needs a PQ ciphertext");
    rec_n(c, "moddown", a.level, a.batch);
    DCt r = make_ct(c, a.level, 2, a.n_slots, a.scale, a.batch);
    moddown(c, a.data(), a.item_words(), a.poly_words(), a.ppoly(0), a.item_words(), a.level, a.batch, 2, r.data(),
            r.item_words(), r.poly_words());
    return r;
}

// ------------------------------------------------------------------ merged ModDown + rescale (R31)
// (the same ops as the oracle's Evaluator.moddown_rescale_ct / relin_rescale_merged)
namespace {
// out (level l-1) = (a - BConv_{P u q_l -> Q_{l-1}}(a)) (P q_l)^{-1} for both polys of every item of the PQ
// batch a: INTT of its P rows and of its q_l rows, one conversion from K + 1 sources, then the forward
// NTT of the l converted rows whose row-pass epilogue writes (a_i - v_i) M^{-1}
void moddown_rescale_into(Ctx &c, const DCt &a, DCt &r)
{
    const uint32_t l = a.level, B = a.batch;
    const size_t N = c.n;
    std::vector<uint32_t> pm;
    for (uint32_t k = 0; k < c.K; ++k) pm.push_back(c.L + 1 + k);
    DBuf zP((size_t)B * 2 * c.K * N, c.stream), zq((size_t)B * 2 * N, c.stream);
    const InvSrc ps{a.ppoly(0), a.item_words(), N, 2 * c.K, 1};
    ntt_inverse(c, zP.get(), B * 2 * c.K, make_map(pm), &ps);
    const InvSrc qsrc{a.data() + (size_t)l * N, a.item_words(), a.poly_words(), 2, 1};
    ntt_inverse(c, zq.get(), B * 2, make_map({l}), &qsrc);
    DBuf w((size_t)B * 2 * l * N, c.stream);
    launch_moddown_bconv(c, w.get(), zP.get(), l, B, 2, zq.get());
    RowEpi ep{};
    ep.out = r.data();
    ep.X = a.data();
    ep.mul = (const TwPair *)c.bconv_ptr(c.off_mr_minv) + (size_t)l * (c.L + 1);
    ep.os = r.item_words();
    ep.ops = r.poly_words();
    ep.xs = a.item_words();
    ep.xps = a.poly_words();
    ep.per = l;
    ep.g0 = 1;
    ep.npoly = 2;
    ntt_forward(c, w.get(), B * 2 * l, qmap(c, l - 1), nullptr, &ep);
}
}  // namespace

DCt ev_conj_mul_relin_rescale(Ctx &c, const DCt &d)
{
    MMFHE_REQUIRE(d.npolys == 2 && !d.pk, MMFHE_E_LAYOUT, "needs a 2-poly Q ciphertext");
    MMFHE_REQUIRE(d.level >= 1, MMFHE_E_DEPTH, "depth exhausted");
    const DKey &kc = find_gk(c, MMFHE_STEP_CONJ), &kp = find_gk(c, MMFHE_STEP_CONJ_PROD);
    const uint32_t l = d.level, B = d.batch;
    rec_n(c, "conj_mul_relin_rescale", l, B);
    // t0 = d0 s(d0), t1 = d1 s(d0) as a 2-poly batch; t2 = d0 s(d1) for every item, then t3 = d1 s(d1)
    // for every item, as one 2B batch of single polynomials (s = sigma_{2N-1}, a gather in the NTT domain)
    DCt t01 = make_ct(c, l, 2, d.n_slots, d.scale * d.scale, B);
    DCt t23 = make_ct(c, l, 1, d.n_slots, d.scale * d.scale, 2 * B);
    launch_conj_tensor(c, t01.data(), t01.item_words(), t23.data(), t23.item(B), t23.item_words(), d.data(),
                       d.item_words(), l, B, (uint32_t)(2 * c.n - 1));
    ModUpOut m = ks_modup(c, t23.data(), t23.item_words(), l, 2 * B);
    DCt acc = make_pq(c, l, d.n_slots, d.scale * d.scale, B);
    const IPOut os{acc.item_words(), acc.poly_words(), acc.item_words(), (size_t)c.K * c.n};
    IPEpi ep;  // first inner product: + the P lift of (t0, t1)
    ep.add = t01.data();
    ep.add1 = t01.poly(1);
    ep.pmod = (const TwPair *)c.bconv_ptr(c.off_pd_pmod);
    ep.as = t01.item_words();
    launch_key_ip(c, acc.data(), acc.ppoly(0), t23.data(), t23.item_words(), m.y.get(), m.T * c.n, m.off,
                  kc.buf.get(), l, B, 1, 1, &os, &ep);
    IPEpi ea;  // second: accumulated
    ea.accumulate = 1;
    launch_key_ip(c, acc.data(), acc.ppoly(0), t23.item(B), t23.item_words(), m.y.get() + (size_t)B * m.T * c.n,
                  m.T * c.n, m.off, kp.buf.get(), l, B, 1, 1, &os, &ea);
    DCt r = make_ct(c, l - 1, 2, d.n_slots, d.scale * d.scale / (double)c.primes[l], B);
    moddown_rescale_into(c, acc, r);
    return r;
}

DCt ev_moddown_rescale_ct(Ctx &c, const DCt &a)
{
    MMFHE_REQUIRE(a.pk == c.K && a.npolys == 2, MMFHE_E_LAYOUT, "ModDown needs a PQ ciphertext");
    MMFHE_REQUIRE(a.level >= 1, MMFHE_E_DEPTH, "depth exhausted");
    rec_n(c, "moddown_rescale", a.level, a.batch);
    DCt r = make_ct(c, a.level - 1, 2, a.n_slots, a.scale / (double)c.primes[a.level], a.batch);
    moddown_rescale_into(c, a, r);
    return r;
}

DCt ev_relin_rescale_merged(Ctx &c, const DCt &a3)
{
    MMFHE_REQUIRE(a3.npolys == 3, MMFHE_E_LAYOUT, "relin needs a 3-poly ciphertext");
    MMFHE_REQUIRE(c.rlk != nullptr, MMFHE_E_MISSING_KEY, "missing relinearisation key");
    MMFHE_REQUIRE(a3.level >= 1, MMFHE_E_DEPTH, "depth exhausted");
    const uint32_t l = a3.level, B = a3.batch;
    rec_n(c, "relin_rescale", l, B);
    // the inner product of ModUp(c2) with rlk left over Q_l u P, its Q rows plus the P lift of
    // (c0, c1) (the key inner product's fused epilogue), then one division by P q_l
    ModUpOut m = ks_modup(c, a3.poly(2), a3.item_words(), l, B);
    DCt acc = make_pq(c, l, a3.n_slots, a3.scale, B);
    const IPOut os{acc.item_words(), acc.poly_words(), acc.item_words(), (size_t)c.K * c.n};
    IPEpi ep;
    ep.add = a3.data();
    ep.add1 = a3.poly(1);
    ep.pmod = (const TwPair *)c.bconv_ptr(c.off_pd_pmod);
    ep.as = a3.item_words();
    launch_key_ip(c, acc.data(), acc.ppoly(0), a3.poly(2), a3.item_words(), m.y.get(), m.T * c.n, m.off,
                  c.rlk->buf.get(), l, B, 1, 1, &os, &ep);
    DCt r = make_ct(c, l - 1, 2, a3.n_slots, a3.scale / (double)c.primes[l], B);
    moddown_rescale_into(c, acc, r);
    return r;
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
    ntt_forward(c, k.buf.get(), rows, pm);
    launch_to_mont(c, k.buf.get(), rows, pm);
}

void load_plain(Ctx &c, const std::string &name, uint32_t level, double scale, const uint64_t *coef, bool on_device,
                bool pq)
{
    MMFHE_REQUIRE(level <= c.L, MMFHE_E_DEPTH, "plaintext level above the chain");
    auto p = std::make_unique<DPlain>();
    p->level = level;
    p->pk = pq ? c.K : 0;
    p->scale = scale;
    const uint32_t rows = level + 1 + p->pk;
    const size_t words = (size_t)rows * c.n;
    p->buf = DBuf(words, c.stream);
    CUDA_CHECK(cudaMemcpyAsync(p->buf.get(), coef, words * 8,
                               on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, c.stream));
    PrimeMap pm = pq ? make_map(c.ext_basis(level)) : qmap(c, level);
    ntt_forward(c, p->buf.get(), rows, pm);
    launch_to_mont(c, p->buf.get(), rows, pm);
    c.plains[plain_key(pq ? name + ".pq" : name, level)] = std::move(p);
}

const DPlain &need_plain(const Ctx &c, const std::string &name, uint32_t level)
{
    DPlain *p = c.find_plain(name, level);
    MMFHE_REQUIRE(p != nullptr, MMFHE_E_MISSING_PLAIN, "missing plaintext operand " + plain_key(name, level));
    return *p;
}

}  // namespace mmfhe
