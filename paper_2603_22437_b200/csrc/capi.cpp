// capi.cpp -- extern "C" entry points of include/mmfhe.h.  Marshalling only:
// every step of the path runs in the CUDA kernels behind eval.h / chains.h.
#include <cstdio>

#include "chains.h"

struct mmfhe_ctx : mmfhe::Ctx {
    using mmfhe::Ctx::Ctx;
};

using namespace mmfhe;

namespace {
thread_local std::string g_last_error;

mmfhe_status fail(mmfhe_ctx *c, mmfhe_status s, const char *msg)
{
    g_last_error = msg;
    if (c) c->last_error = msg;
    return s;
}

// every entry point with a ctx allocates from that ctx's pool (PoolScope)
#define API_BEGIN                                                                                 \
    try {                                                                                         \
        DeviceScope dev_scope_(ctx ? ctx->device : -1);                                           \
        PoolScope pool_scope_(ctx ? ctx->mem.pool : nullptr);
#define API_BEGIN0 try {
#define API_END(C)                                                                                \
    }                                                                                             \
    catch (const Error &e) { return fail((C), e.status, e.what()); }                              \
    catch (const std::bad_alloc &) { return fail((C), MMFHE_E_OOM, "host allocation failed"); }   \
    catch (const std::exception &e) { return fail((C), MMFHE_E_CUDA, e.what()); }                 \
    return MMFHE_OK;

uint32_t npolys_of(const mmfhe_ct &ct) { return ct.n_polys ? ct.n_polys : 2; }

// Device NTT-form input used in place; anything else is imported (copied, NTT'd).
DCt input_ct(Ctx &c, const mmfhe_ct &ct)
{
    MMFHE_REQUIRE(ct.data != nullptr, MMFHE_E_INVALID_ARG, "null ciphertext");
    MMFHE_REQUIRE(ct.log_n == c.log_n, MMFHE_E_PARAMS, "ring dimension mismatch");
    MMFHE_REQUIRE(ct.level <= c.L, MMFHE_E_DEPTH, "level above the modulus chain");
    if (ct.on_device && ct.form == MMFHE_FORM_EVAL) return view_ct(c, ct, npolys_of(ct));
    return import_ct(c, ct, npolys_of(ct));
}

// Operand stores changed: cached chain graphs may bake in stale operands.
void state_changed(Ctx &c)
{
    c.drop_graphs();
    ++c.state_gen;
}

bool all_device(const mmfhe_ct *v, size_t n)
{
    for (size_t i = 0; i < n; ++i)
        if (!v[i].on_device) return false;
    return true;
}

template <class T>
void put(std::string &k, const T &x)
{
    k.append((const char *)&x, sizeof(T));
}

// Everything a captured chain graph depends on: chain, cfg, every buffer address and
// layout, and the operand-store generation.
std::string chain_key(const Ctx &c, const char *chain, const mmfhe_chain_cfg &cfg, const mmfhe_ct *in, size_t n_in,
                      const mmfhe_ct *out, size_t n_out)
{
    std::string k(chain);
    k.push_back('\0');
    put(k, cfg);
    put(k, c.state_gen);
    put(k, n_in);
    for (size_t i = 0; i < n_in; ++i) {
        put(k, in[i].data);
        put(k, in[i].level);
        put(k, in[i].scale);
        put(k, in[i].n_slots);
        put(k, in[i].form);
        put(k, in[i].n_polys);
        put(k, in[i].log_n);
    }
    put(k, n_out);
    for (size_t i = 0; i < n_out; ++i) {
        put(k, out[i].data);
        put(k, out[i].form);
    }
    return k;
}

void run_and_export(Ctx &c, const char *chain, const mmfhe_chain_cfg &cfg, const mmfhe_ct *in, size_t n_in,
                    mmfhe_ct *out, size_t n_out)
{
    std::vector<DCt> res = run_chain(c, chain, cfg, in, n_in);
    size_t o = 0;
    for (auto &d : res) {
        MMFHE_REQUIRE(o + d.batch <= n_out, MMFHE_E_LAYOUT, "chain produced an unexpected number of outputs");
        export_batch(c, d, out + o);
        o += d.batch;
    }
    MMFHE_REQUIRE(o == n_out, MMFHE_E_LAYOUT, "chain produced an unexpected number of outputs");
}

// Capture one chain call on a private stream; false if the call is not capturable (the
// caller then runs it eagerly).  Validation errors surface in that eager run.
bool capture_chain(Ctx &c, Ctx::ChainGraph &g, const char *chain, const mmfhe_chain_cfg &cfg, const mmfhe_ct *in,
                   size_t n_in, mmfhe_ct *out, size_t n_out)
{
    if (!c.cap_stream) CUDA_CHECK(cudaStreamCreateWithFlags(&c.cap_stream, cudaStreamNonBlocking));
    const cudaStream_t saved = c.stream;
    const uint64_t l0 = c.launches;
    c.stream = c.cap_stream;
    cudaGraph_t graph = nullptr;
    bool ok = cudaStreamBeginCapture(c.stream, cudaStreamCaptureModeRelaxed) == cudaSuccess;
    if (ok) {
        try {
            run_and_export(c, chain, cfg, in, n_in, out, n_out);
        } catch (...) {
            ok = false;
        }
        ok = cudaStreamEndCapture(c.stream, &graph) == cudaSuccess && ok;
    }
    c.stream = saved;
    g.launches = c.launches - l0;
    c.launches = l0;
    cudaGraphExec_t exec = nullptr;
    ok = ok && graph && cudaGraphInstantiate(&exec, graph, 0) == cudaSuccess;
    if (graph) cudaGraphDestroy(graph);
    if (!ok) {
        (void)cudaGetLastError();
        g.seen = -1;
        return false;
    }
    g.exec = exec;
    g.out_meta.assign(out, out + n_out);
    return true;
}

// mmfhe_eval_chain's body: repeated device-resident calls (trace / profile off) replay a
// captured CUDA graph, everything else runs eagerly.
void eval_chain_impl(Ctx &c, const char *chain, const mmfhe_chain_cfg &cfg, const mmfhe_ct *in, size_t n_in,
                     mmfhe_ct *out, size_t n)
{
    if (c.graphs_on && !c.trace_on && !c.prof_on && all_device(in, n_in) && all_device(out, n)) {
        // (one graph per distinct chain + buffer-address set: C5 keeps 2 per gesture session + its vital
        // groups, 1024 sessions included; a full cache is dropped and re-filled)
        if (c.graphs.size() >= 1100) c.drop_graphs();
        Ctx::ChainGraph &g = c.graphs[chain_key(c, chain, cfg, in, n_in, out, n)];
        if (!g.exec && g.seen >= 1) capture_chain(c, g, chain, cfg, in, n_in, out, n);
        if (g.exec) {
            CUDA_CHECK(cudaGraphLaunch(g.exec, c.stream));
            c.launches += g.launches;
            ++c.graph_replays;
            for (size_t i = 0; i < n; ++i) {
                out[i].log_n = g.out_meta[i].log_n;
                out[i].level = g.out_meta[i].level;
                out[i].scale = g.out_meta[i].scale;
                out[i].n_slots = g.out_meta[i].n_slots;
                out[i].n_polys = g.out_meta[i].n_polys;
            }
            return;
        }
        if (g.seen >= 0) ++g.seen;
    }
    run_and_export(c, chain, cfg, in, n_in, out, n);
}

mmfhe_chain_cfg cfg_or_default(const mmfhe_chain_cfg *cfg)
{
    mmfhe_chain_cfg d{};
    if (cfg) d = *cfg;
    if (!d.gamma) d.gamma = 1;
    if (!d.p_phi) d.p_phi = 1;
    if (!d.taylor_order) d.taylor_order = 1;
    return d;
}
}  // namespace

extern "C" {

mmfhe_status mmfhe_ctx_create(const mmfhe_params *params, int cuda_device, void *cuda_stream, mmfhe_ctx **out)
{
    if (!params || !out) return fail(nullptr, MMFHE_E_INVALID_ARG, "null argument");
    *out = nullptr;
    API_BEGIN0
    *out = new mmfhe_ctx(*params, cuda_device, (cudaStream_t)cuda_stream);
    API_END(nullptr)
}

mmfhe_status mmfhe_ctx_destroy(mmfhe_ctx *ctx)
{
    if (!ctx) return MMFHE_OK;
    API_BEGIN0
    cudaStreamSynchronize(ctx->stream);
    delete ctx;
    API_END(nullptr)
}

const char *mmfhe_last_error(const mmfhe_ctx *ctx) { return ctx ? ctx->last_error.c_str() : g_last_error.c_str(); }

mmfhe_status mmfhe_ctx_memory(mmfhe_ctx *ctx, size_t *bytes)
{
    API_BEGIN
    MMFHE_REQUIRE(bytes != nullptr, MMFHE_E_INVALID_ARG, "null argument");
    uint64_t used = 0;  // this ctx's own pool only
    CUDA_CHECK(cudaMemPoolGetAttribute(ctx->mem.pool, cudaMemPoolAttrUsedMemCurrent, &used));
    *bytes = (size_t)used;
    API_END(ctx)
}

mmfhe_status mmfhe_launch_count(mmfhe_ctx *ctx, uint64_t *count)
{
    if (!ctx || !count) return fail(ctx, MMFHE_E_INVALID_ARG, "null argument");
    *count = ctx->launches;
    return MMFHE_OK;
}

mmfhe_status mmfhe_chain_required_rotations(mmfhe_ctx *ctx, const char *chain, const mmfhe_chain_cfg *cfg,
                                            int32_t *steps, size_t cap, size_t *n)
{
    API_BEGIN
    MMFHE_REQUIRE(chain && n, MMFHE_E_INVALID_ARG, "null argument");
    std::vector<int32_t> v = chain_rotations(*ctx, chain, cfg_or_default(cfg));
    *n = v.size();
    MMFHE_REQUIRE(v.size() <= cap || !steps, MMFHE_E_LAYOUT, "rotation buffer too small");
    if (steps)
        for (size_t i = 0; i < v.size(); ++i) steps[i] = v[i];
    API_END(ctx)
}

mmfhe_status mmfhe_load_relin_key(mmfhe_ctx *ctx, const uint64_t *words, size_t n_words, int on_device)
{
    API_BEGIN
    state_changed(*ctx);
    MMFHE_REQUIRE(words, MMFHE_E_INVALID_ARG, "null key");
    auto k = std::make_unique<DKey>();
    load_key(*ctx, *k, words, n_words, on_device != 0);
    ctx->sync();
    ctx->rlk = std::move(k);
    API_END(ctx)
}

mmfhe_status mmfhe_load_galois_key(mmfhe_ctx *ctx, int32_t step, const uint64_t *words, size_t n_words,
                                   int on_device)
{
    API_BEGIN
    state_changed(*ctx);
    MMFHE_REQUIRE(words, MMFHE_E_INVALID_ARG, "null key");
    int32_t k;
    galois_element(*ctx, step, &k);
    MMFHE_REQUIRE(k != 0, MMFHE_E_INVALID_ARG, "rotation by 0 needs no key");
    auto key = std::make_unique<DKey>();
    load_key(*ctx, *key, words, n_words, on_device != 0);
    ctx->sync();
    ctx->gk[k] = std::move(key);
    API_END(ctx)
}

mmfhe_status mmfhe_load_plain(mmfhe_ctx *ctx, const char *name, const mmfhe_ct *pt)
{
    API_BEGIN
    state_changed(*ctx);
    MMFHE_REQUIRE(name && pt && pt->data, MMFHE_E_INVALID_ARG, "null argument");
    MMFHE_REQUIRE(pt->log_n == ctx->log_n, MMFHE_E_PARAMS, "ring dimension mismatch");
    MMFHE_REQUIRE(pt->form == MMFHE_FORM_COEFF, MMFHE_E_FORMAT, "plaintexts are imported in coefficient form");
    load_plain(*ctx, name, pt->level, pt->scale, pt->data, pt->on_device != 0);
    ctx->sync();
    API_END(ctx)
}

mmfhe_status mmfhe_load_plain_pq(mmfhe_ctx *ctx, const char *name, const mmfhe_ct *pt)
{
    API_BEGIN
    state_changed(*ctx);
    MMFHE_REQUIRE(name && pt && pt->data, MMFHE_E_INVALID_ARG, "null argument");
    MMFHE_REQUIRE(pt->log_n == ctx->log_n, MMFHE_E_PARAMS, "ring dimension mismatch");
    MMFHE_REQUIRE(pt->form == MMFHE_FORM_COEFF, MMFHE_E_FORMAT, "plaintexts are imported in coefficient form");
    load_plain(*ctx, name, pt->level, pt->scale, pt->data, pt->on_device != 0, true);
    ctx->sync();
    API_END(ctx)
}

mmfhe_status mmfhe_encode_plain(mmfhe_ctx *ctx, const char *name, const double *v, size_t n, uint32_t level,
                                double scale)
{
    API_BEGIN
    state_changed(*ctx);
    MMFHE_REQUIRE(name && v && n, MMFHE_E_INVALID_ARG, "null argument");
    encode_plain(*ctx, name, std::vector<double>(v, v + n), level, scale);
    API_END(ctx)
}

mmfhe_status mmfhe_load_scalars(mmfhe_ctx *ctx, const char *name, const double *v, size_t n)
{
    API_BEGIN
    state_changed(*ctx);
    MMFHE_REQUIRE(name && (v || !n), MMFHE_E_INVALID_ARG, "null argument");
    ctx->scalars[name] = std::vector<double>(v, v + n);
    API_END(ctx)
}

mmfhe_status mmfhe_prepare_chain(mmfhe_ctx *ctx, const char *chain, const mmfhe_chain_cfg *cfg, uint32_t in_level,
                                 const double *const *fc_w, const double *const *fc_b, const double *const *taps)
{
    API_BEGIN
    state_changed(*ctx);
    MMFHE_REQUIRE(chain && cfg, MMFHE_E_INVALID_ARG, "null argument");
    mmfhe_chain_cfg c = cfg_or_default(cfg);
    chain_rotations(*ctx, chain, c);  // validates the name
    (void)in_level;
    if (fc_w && fc_b) {
        ctx->fc_w.assign(3, {});
        ctx->fc_b.assign(3, {});
        for (int l = 0; l < 3; ++l) {
            const size_t rows = c.fc_dims[l + 1], cols = c.fc_dims[l];
            MMFHE_REQUIRE(rows && cols && fc_w[l] && fc_b[l], MMFHE_E_SHAPE, "FC dims/weights");
            ctx->fc_w[l].assign(fc_w[l], fc_w[l] + rows * cols);
            ctx->fc_b[l].assign(fc_b[l], fc_b[l] + rows);
        }
    }
    if (taps)
        for (uint32_t b = 0; b < c.n_bands; ++b) {
            MMFHE_REQUIRE(taps[b], MMFHE_E_SHAPE, "missing FIR taps");
            ctx->scalars["k5.b" + std::to_string(b)] = std::vector<double>(taps[b], taps[b] + c.n_taps[b]);
        }
    ctx->auto_encode = true;
    API_END(ctx)
}

mmfhe_status mmfhe_chain_plan(mmfhe_ctx *ctx, const char *chain, const mmfhe_chain_cfg *cfg, uint32_t in_level,
                              size_t n_in, uint32_t *out_levels, size_t cap, size_t *n_out)
{
    API_BEGIN
    MMFHE_REQUIRE(chain && n_out, MMFHE_E_INVALID_ARG, "null argument");
    std::vector<uint32_t> lv = chain_plan(*ctx, chain, cfg_or_default(cfg), in_level, n_in);
    *n_out = lv.size();
    MMFHE_REQUIRE(!out_levels || lv.size() <= cap, MMFHE_E_LAYOUT, "output buffer too small");
    if (out_levels)
        for (size_t i = 0; i < lv.size(); ++i) out_levels[i] = lv[i];
    API_END(ctx)
}

mmfhe_status mmfhe_eval_chain(mmfhe_ctx *ctx, const char *chain, const mmfhe_chain_cfg *cfg, const mmfhe_ct *in,
                              size_t n_in, mmfhe_ct *out, size_t cap, size_t *n_out)
{
    API_BEGIN
    MMFHE_REQUIRE(chain && in && n_in && out && n_out, MMFHE_E_INVALID_ARG, "null argument");
    mmfhe_chain_cfg c = cfg_or_default(cfg);
    std::vector<uint32_t> lv = chain_plan(*ctx, chain, c, in[0].level, n_in);
    *n_out = lv.size();
    MMFHE_REQUIRE(lv.size() <= cap, MMFHE_E_LAYOUT, "output capacity too small");
    eval_chain_impl(*ctx, chain, c, in, n_in, out, lv.size());
    API_END(ctx)
}

mmfhe_status mmfhe_eval_chain_async(mmfhe_ctx *ctx, const char *chain, const mmfhe_chain_cfg *cfg,
                                    const mmfhe_ct *in, size_t n_in, mmfhe_ct *out, size_t cap, size_t *n_out)
{
    API_BEGIN
    MMFHE_REQUIRE(chain && in && n_in && out && n_out, MMFHE_E_INVALID_ARG, "null argument");
    mmfhe_chain_cfg c = cfg_or_default(cfg);
    std::vector<uint32_t> lv = chain_plan(*ctx, chain, c, in[0].level, n_in);
    *n_out = lv.size();
    MMFHE_REQUIRE(lv.size() <= cap, MMFHE_E_LAYOUT, "output capacity too small");
    const size_t n = lv.size();
    if (all_device(in, n_in) && all_device(out, n)) {  // already asynchronous
        eval_chain_impl(*ctx, chain, c, in, n_in, out, n);
        return MMFHE_OK;
    }
    Ctx &x = *ctx;
    const mmfhe_ct &c0 = in[0];
    const size_t iw = (size_t)npolys_of(c0) * (c0.level + 1) * x.n;
    for (size_t i = 0; i < n_in; ++i)
        MMFHE_REQUIRE(in[i].data && in[i].level == c0.level && npolys_of(in[i]) == npolys_of(c0) &&
                          in[i].form == c0.form,
                      MMFHE_E_LAYOUT, "async chain inputs must share level, layout and form");
    std::vector<size_t> ooff(n + 1, 0);
    for (size_t i = 0; i < n; ++i) {
        MMFHE_REQUIRE(out[i].data, MMFHE_E_INVALID_ARG, "null output buffer");
        ooff[i + 1] = ooff[i] + (size_t)2 * (lv[i] + 1) * x.n;
    }
    std::string key(chain);
    key.push_back('\0');
    put(key, n_in);
    put(key, iw);
    put(key, ooff[n]);
    Ctx::Staging &st = x.staging[key];
    if (!x.copy_stream) CUDA_CHECK(cudaStreamCreateWithFlags(&x.copy_stream, cudaStreamNonBlocking));
    Ctx::StageSlot &sl = st.slot[st.next];
    st.next ^= 1;
    if (!sl.ready) {
        sl.in = DBuf(n_in * iw, x.stream);
        sl.out = DBuf(ooff[n], x.stream);
        CUDA_CHECK(cudaEventCreateWithFlags(&sl.ready, cudaEventDisableTiming));
        CUDA_CHECK(cudaEventCreateWithFlags(&sl.free, cudaEventDisableTiming));
        CUDA_CHECK(cudaEventRecord(sl.free, x.stream));
    }
    // upload on the copy stream once the compute that last read this slot is done
    CUDA_CHECK(cudaStreamWaitEvent(x.copy_stream, sl.free, 0));
    bool contig = true;
    for (size_t i = 1; i < n_in && contig; ++i) contig = in[i].data == c0.data + i * iw && !in[i].on_device;
    if (contig && !c0.on_device) {
        CUDA_CHECK(cudaMemcpyAsync(sl.in.get(), c0.data, n_in * iw * 8, cudaMemcpyHostToDevice, x.copy_stream));
    } else {
        for (size_t i = 0; i < n_in; ++i)
            CUDA_CHECK(cudaMemcpyAsync(sl.in.get() + i * iw, in[i].data, iw * 8,
                                       in[i].on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice,
                                       x.copy_stream));
    }
    CUDA_CHECK(cudaEventRecord(sl.ready, x.copy_stream));
    CUDA_CHECK(cudaStreamWaitEvent(x.stream, sl.ready, 0));
    std::vector<mmfhe_ct> din(in, in + n_in), dout(out, out + n);
    for (size_t i = 0; i < n_in; ++i) {
        din[i].data = sl.in.get() + i * iw;
        din[i].on_device = 1;
    }
    for (size_t i = 0; i < n; ++i) {
        dout[i].data = sl.out.get() + ooff[i];
        dout[i].on_device = 1;
    }
    eval_chain_impl(x, chain, c, din.data(), n_in, dout.data(), n);
    CUDA_CHECK(cudaEventRecord(sl.free, x.stream));
    for (size_t i = 0; i < n; ++i) {
        out[i].log_n = dout[i].log_n;
        out[i].level = dout[i].level;
        out[i].scale = dout[i].scale;
        out[i].n_slots = dout[i].n_slots;
        out[i].n_polys = dout[i].n_polys;
        CUDA_CHECK(cudaMemcpyAsync(out[i].data, dout[i].data, (ooff[i + 1] - ooff[i]) * 8,
                                   out[i].on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, x.stream));
    }
    API_END(ctx)
}

mmfhe_status mmfhe_ctx_sync(mmfhe_ctx *ctx)
{
    if (!ctx) return fail(ctx, MMFHE_E_INVALID_ARG, "null argument");
    API_BEGIN
    if (ctx->copy_stream) CUDA_CHECK(cudaStreamSynchronize(ctx->copy_stream));
    CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
    API_END(ctx)
}

mmfhe_status mmfhe_sum_partials(mmfhe_ctx *ctx, const mmfhe_ct *parts, size_t n, mmfhe_ct *out)
{
    API_BEGIN
    MMFHE_REQUIRE(parts && n && out, MMFHE_E_INVALID_ARG, "null argument");
    std::vector<DCt> ins;
    for (size_t i = 0; i < n; ++i) ins.push_back(input_ct(*ctx, parts[i]));
    std::vector<const DCt *> p;
    for (auto &x : ins) p.push_back(&x);
    DCt r = ev_sum(*ctx, p);
    export_ct(*ctx, r, *out);
    API_END(ctx)
}

// ---------------------------------------------------------------- primitives
static mmfhe_status ntt_rows(mmfhe_ctx *ctx, uint64_t *d_rows, uint32_t n_rows, const uint32_t *prime_idx, bool inv)
{
    API_BEGIN
    MMFHE_REQUIRE(d_rows && prime_idx && n_rows, MMFHE_E_INVALID_ARG, "null argument");
    std::vector<uint32_t> m(prime_idx, prime_idx + n_rows);
    for (uint32_t p : m) MMFHE_REQUIRE(p < ctx->primes.size(), MMFHE_E_INVALID_ARG, "prime index out of range");
    // a periodic prime list (a batch of items with the same limbs) goes in one launch
    for (uint32_t per = 1; per <= std::min<uint32_t>(kMapCap, n_rows); ++per) {
        if (n_rows % per) continue;
        bool ok = true;
        for (uint32_t i = per; i < n_rows && ok; ++i) ok = m[i] == m[i - per];
        if (!ok) continue;
        PrimeMap pm = make_map(std::vector<uint32_t>(m.begin(), m.begin() + per));
        if (inv)
            ntt_inverse(*ctx, d_rows, n_rows, pm);
        else
            ntt_forward(*ctx, d_rows, n_rows, pm);
        return MMFHE_OK;
    }
    for (uint32_t s = 0; s < n_rows; s += kMapCap) {
        uint32_t cnt = std::min<uint32_t>(kMapCap, n_rows - s);
        PrimeMap pm = make_map(std::vector<uint32_t>(m.begin() + s, m.begin() + s + cnt));
        uint64_t *d = d_rows + (size_t)s * ctx->n;
        if (inv)
            ntt_inverse(*ctx, d, cnt, pm);
        else
            ntt_forward(*ctx, d, cnt, pm);
    }
    API_END(ctx)
}

mmfhe_status mmfhe_ntt(mmfhe_ctx *ctx, uint64_t *d_rows, uint32_t n_rows, const uint32_t *prime_idx)
{
    return ntt_rows(ctx, d_rows, n_rows, prime_idx, false);
}
mmfhe_status mmfhe_intt(mmfhe_ctx *ctx, uint64_t *d_rows, uint32_t n_rows, const uint32_t *prime_idx)
{
    return ntt_rows(ctx, d_rows, n_rows, prime_idx, true);
}

static mmfhe_status addsub(mmfhe_ctx *ctx, const mmfhe_ct *a, const mmfhe_ct *b, mmfhe_ct *out, bool sub)
{
    API_BEGIN
    MMFHE_REQUIRE(a && b && out, MMFHE_E_INVALID_ARG, "null argument");
    DCt x = input_ct(*ctx, *a), y = input_ct(*ctx, *b);
    export_ct(*ctx, ev_addsub(*ctx, x, y, sub), *out);
    API_END(ctx)
}
mmfhe_status mmfhe_hadd(mmfhe_ctx *ctx, const mmfhe_ct *a, const mmfhe_ct *b, mmfhe_ct *out)
{
    return addsub(ctx, a, b, out, false);
}
mmfhe_status mmfhe_hsub(mmfhe_ctx *ctx, const mmfhe_ct *a, const mmfhe_ct *b, mmfhe_ct *out)
{
    return addsub(ctx, a, b, out, true);
}

mmfhe_status mmfhe_pmult(mmfhe_ctx *ctx, const mmfhe_ct *a, const char *pt_name, mmfhe_ct *out)
{
    API_BEGIN
    MMFHE_REQUIRE(a && pt_name && out, MMFHE_E_INVALID_ARG, "null argument");
    DCt x = input_ct(*ctx, *a);
    const DPlain &p = need_plain(*ctx, pt_name, x.level);
    export_ct(*ctx, ev_pmult_sum(*ctx, {{&p, &x}}), *out);
    API_END(ctx)
}

mmfhe_status mmfhe_hmult(mmfhe_ctx *ctx, const mmfhe_ct *a, const mmfhe_ct *b, mmfhe_ct *out)
{
    API_BEGIN
    MMFHE_REQUIRE(a && b && out, MMFHE_E_INVALID_ARG, "null argument");
    DCt x = input_ct(*ctx, *a), y = input_ct(*ctx, *b);
    export_ct(*ctx, ev_relin(*ctx, ev_tensor_sum(*ctx, {{&x, &y}})), *out);
    API_END(ctx)
}

mmfhe_status mmfhe_relin(mmfhe_ctx *ctx, const mmfhe_ct *a3, mmfhe_ct *out)
{
    API_BEGIN
    MMFHE_REQUIRE(a3 && out, MMFHE_E_INVALID_ARG, "null argument");
    MMFHE_REQUIRE(npolys_of(*a3) == 3, MMFHE_E_LAYOUT, "relin needs n_polys = 3");
    DCt x = input_ct(*ctx, *a3);
    export_ct(*ctx, ev_relin(*ctx, x), *out);
    API_END(ctx)
}

mmfhe_status mmfhe_hrot(mmfhe_ctx *ctx, const mmfhe_ct *a, int32_t step, mmfhe_ct *out)
{
    API_BEGIN
    MMFHE_REQUIRE(a && out, MMFHE_E_INVALID_ARG, "null argument");
    DCt x = input_ct(*ctx, *a);
    export_ct(*ctx, ev_rotate(*ctx, x, step), *out);
    API_END(ctx)
}

mmfhe_status mmfhe_hrot_hoisted(mmfhe_ctx *ctx, const mmfhe_ct *a, const int32_t *steps, size_t n_steps,
                                mmfhe_ct *out)
{
    API_BEGIN
    MMFHE_REQUIRE(a && steps && out && n_steps, MMFHE_E_INVALID_ARG, "null argument");
    DCt x = input_ct(*ctx, *a);
    std::vector<DCt> r = ev_rotate_hoisted(*ctx, x, std::vector<int32_t>(steps, steps + n_steps));
    for (size_t i = 0; i < n_steps; ++i) export_ct(*ctx, r[i], out[i]);
    API_END(ctx)
}

mmfhe_status mmfhe_hrot_hoisted_pq(mmfhe_ctx *ctx, const mmfhe_ct *a, const int32_t *steps, size_t n_steps,
                                   mmfhe_ct *out)
{
    API_BEGIN
    MMFHE_REQUIRE(a && steps && out && n_steps, MMFHE_E_INVALID_ARG, "null argument");
    DCt x = input_ct(*ctx, *a);
    std::vector<DCt> r = ev_rotate_hoisted_pq(*ctx, x, std::vector<int32_t>(steps, steps + n_steps));
    for (size_t i = 0; i < n_steps; ++i) export_pq(*ctx, r[i], out[i]);
    API_END(ctx)
}

mmfhe_status mmfhe_rescale(mmfhe_ctx *ctx, const mmfhe_ct *a, mmfhe_ct *out)
{
    API_BEGIN
    MMFHE_REQUIRE(a && out, MMFHE_E_INVALID_ARG, "null argument");
    DCt x = input_ct(*ctx, *a);
    export_ct(*ctx, ev_rescale(*ctx, x), *out);
    API_END(ctx)
}

mmfhe_status mmfhe_keyswitch(mmfhe_ctx *ctx, const mmfhe_ct *x, int32_t step, int use_relin, mmfhe_ct *out)
{
    API_BEGIN
    MMFHE_REQUIRE(x && out, MMFHE_E_INVALID_ARG, "null argument");
    MMFHE_REQUIRE(npolys_of(*x) == 1, MMFHE_E_LAYOUT, "keyswitch input is one polynomial (n_polys = 1)");
    DCt in = input_ct(*ctx, *x);
    const DKey *key;
    if (use_relin) {
        MMFHE_REQUIRE(ctx->rlk != nullptr, MMFHE_E_MISSING_KEY, "missing relinearisation key");
        key = ctx->rlk.get();
    } else {
        int32_t k;
        galois_element(*ctx, step, &k);
        key = &find_gk(*ctx, k);
    }
    ctx->rec("keyswitch", in.level);
    DCt r = make_ct(*ctx, in.level, 2, in.n_slots, in.scale);
    ev_keyswitch(*ctx, in.data(), in.item_words(), in.level, 1, *key, r.data(), r.item_words(), nullptr, nullptr, 0);
    export_ct(*ctx, r, *out);
    API_END(ctx)
}

mmfhe_status mmfhe_mod_switch(mmfhe_ctx *ctx, const mmfhe_ct *a, uint32_t level, mmfhe_ct *out)
{
    API_BEGIN
    MMFHE_REQUIRE(a && out, MMFHE_E_INVALID_ARG, "null argument");
    DCt x = input_ct(*ctx, *a);
    export_ct(*ctx, ev_drop_to(*ctx, x, level), *out);
    API_END(ctx)
}

mmfhe_status mmfhe_hrot_batch(mmfhe_ctx *ctx, const mmfhe_ct *a, size_t n, int32_t step, mmfhe_ct *out)
{
    API_BEGIN
    MMFHE_REQUIRE(a && out && n, MMFHE_E_INVALID_ARG, "null argument");
    DCt x = import_batch(*ctx, a, 0, 1, n);  // one batched KS: each evk word read once for all n
    DCt r = ev_rotate(*ctx, x, step);
    export_batch(*ctx, r, out);
    API_END(ctx)
}

mmfhe_status mmfhe_hmult_batch(mmfhe_ctx *ctx, const mmfhe_ct *a, const mmfhe_ct *b, size_t n, mmfhe_ct *out)
{
    API_BEGIN
    MMFHE_REQUIRE(a && b && out && n, MMFHE_E_INVALID_ARG, "null argument");
    DCt x = import_batch(*ctx, a, 0, 1, n), y = import_batch(*ctx, b, 0, 1, n);
    DCt r = ev_relin(*ctx, ev_tensor_sum(*ctx, {{&x, &y}}));
    export_batch(*ctx, r, out);
    API_END(ctx)
}

mmfhe_status mmfhe_trace_get(mmfhe_ctx *ctx, char *buf, size_t cap, size_t *len)
{
    API_BEGIN
    std::string s;
    for (auto &t : ctx->trace) {
        s += t;
        s += '\n';
    }
    if (len) *len = s.size();
    if (buf && cap) {
        size_t n = std::min(cap - 1, s.size());
        std::memcpy(buf, s.data(), n);
        buf[n] = 0;
    }
    API_END(ctx)
}

mmfhe_status mmfhe_trace_clear(mmfhe_ctx *ctx)
{
    API_BEGIN
    ctx->trace.clear();
    API_END(ctx)
}

mmfhe_status mmfhe_trace_enable(mmfhe_ctx *ctx, int on)
{
    API_BEGIN
    ctx->trace_on = on != 0;
    API_END(ctx)
}

mmfhe_status mmfhe_graph_enable(mmfhe_ctx *ctx, int on)
{
    if (!ctx) return fail(ctx, MMFHE_E_INVALID_ARG, "null argument");
    API_BEGIN
    ctx->graphs_on = on != 0;
    if (!ctx->graphs_on) ctx->drop_graphs();
    API_END(ctx)
}

mmfhe_status mmfhe_graph_stats(mmfhe_ctx *ctx, size_t *n_graphs, uint64_t *replays)
{
    if (!ctx || !n_graphs || !replays) return fail(ctx, MMFHE_E_INVALID_ARG, "null argument");
    size_t n = 0;
    for (const auto &kv : ctx->graphs) n += kv.second.exec != nullptr;
    *n_graphs = n;
    *replays = ctx->graph_replays;
    return MMFHE_OK;
}

mmfhe_status mmfhe_profile_enable(mmfhe_ctx *ctx, int on)
{
    API_BEGIN
    if (!on && ctx->prof_on) ctx->profile_report();
    ctx->prof_on = on != 0;
    API_END(ctx)
}

mmfhe_status mmfhe_microbench(mmfhe_ctx *ctx, int kind, double *ops_per_s)
{
    API_BEGIN
    MMFHE_REQUIRE(ops_per_s && kind >= 0 && kind <= 5, MMFHE_E_INVALID_ARG, "bad microbench kind");
    *ops_per_s = microbench_ops_per_s(*ctx, kind);
    API_END(ctx)
}

mmfhe_status mmfhe_profile_get(mmfhe_ctx *ctx, char *buf, size_t cap, size_t *len)
{
    API_BEGIN
    std::string s = ctx->profile_report();
    if (len) *len = s.size();
    if (buf && cap) {
        size_t n = std::min(cap - 1, s.size());
        std::memcpy(buf, s.data(), n);
        buf[n] = 0;
    }
    API_END(ctx)
}

}  // extern "C"
