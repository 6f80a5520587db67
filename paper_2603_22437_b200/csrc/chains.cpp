// chains.cpp -- the mmFHE kernel chains over the batched device evaluator.
//
// Each kernel follows the paper's circuit with the canonical op sequence of
// SURVEY §8(c)-7 (relinearisation / rescale placement, BSGS split, overflow
// folds), so the op trace and every residue equal the CPU oracle's:
//   K1  Eq. energy            P:767-771     K5  Eq. fir_iq
//   K2  Eqs. soft_power_*     P:777-788     K6  Eq. notch_mask
//   K2b Eq. gesture_soft_pow  P:128-133     K7  Eq. taylor_arctan
//   K3  Eqs. dft_kernel/re/im P:797-815,    FC  Eq. mlp_forward
//       BSGS P:164-176
//   K4  Eqs. phase_mask/iq
// Pipelines: vital signs P:901-902, dynamic classification P:904-907.
//
// Per-frame kernels run on batches of frames (cfg.frame_batch, op-major order
// inside a batch): one launch per op covers the whole batch, so plaintext
// diagonals and evaluation keys are streamed once per batch.  K5 (Toeplitz FIR
// over frames) and the narrowband DFT are banded / dense scalar matrix products
// over the frame batch (one kernel each).
//
// Public plaintext operands are looked up by (name, level); when absent and
// the ctx was prepared (mmfhe_prepare_chain), they are computed from the
// paper's formulas and encoded with the library's encoder on first use.
#include <cmath>
#include <cstdlib>
#include <complex>
#include <functional>

#include "chains.h"

namespace mmfhe {

namespace {

uint32_t ceil_sqrt(uint32_t x)
{
    uint32_t b = 0;
    while (b * b < x) ++b;
    return b;
}

uint32_t ilog2(uint32_t x)
{
    uint32_t r = 0;
    while ((1u << r) < x) ++r;
    return r;
}

std::vector<double> hann(uint32_t M)
{
    std::vector<double> w(M);
    if (M == 1) {
        w[0] = 1.0;
        return w;
    }
    for (uint32_t i = 0; i < M; ++i) w[i] = 0.5 - 0.5 * std::cos(2.0 * M_PI * i / (double)(M - 1));
    return w;
}

typedef std::complex<double> cd;

// Rot(v, k)[j] = v[(j + k) mod n]
template <typename T>
std::vector<T> rot(const std::vector<T> &v, int64_t k)
{
    const int64_t n = (int64_t)v.size();
    std::vector<T> o(n);
    for (int64_t j = 0; j < n; ++j) o[j] = v[(size_t)(((j + k) % n + n) % n)];
    return o;
}

// Lane-interleaved layout (DESIGN R20): a per-frame public vector with every
// entry repeated L times (slot L i + f holds entry i for every frame lane f).
template <typename T>
std::vector<T> lane_rep(const std::vector<T> &v, uint32_t L)
{
    if (L <= 1) return v;
    std::vector<T> o(v.size() * L);
    for (size_t i = 0; i < v.size(); ++i)
        for (uint32_t f = 0; f < L; ++f) o[i * L + f] = v[i];
    return o;
}

uint32_t lanes_of(const mmfhe_chain_cfg &cfg) { return cfg.lanes ? cfg.lanes : 1; }

// K3 / gesture chains on complex slots (DESIGN R28): one input ciphertext z = v_re + j v_im per
// frame (group) instead of the (v_re, v_im) pair
bool cplx_chain(const std::string &chain, const mmfhe_chain_cfg &cfg)
{
    return cfg.cplx && (chain == "k3_doppler_dft" || chain == "gesture" || chain == "gesture_frame" ||
                        chain == "gesture_features");
}

struct Sched {
    uint32_t b;
    struct G {
        uint32_t gp;
        int32_t G;
        std::vector<uint32_t> babies;
    };
    std::vector<G> giants;
};

Sched k3_schedule(const mmfhe_chain_cfg &cfg)
{
    const int32_t D = (int32_t)cfg.D, d = 2 * D - 1, o_min = -(D - 1);
    Sched s;
    s.b = cfg.bsgs_baby ? cfg.bsgs_baby : ceil_sqrt((uint32_t)d);
    const int32_t b = (int32_t)s.b;
    if (cfg.bsgs_aligned) {
        // DESIGN R29: giants G = b k, k = floor(-(D-1)/b) .. floor((D-1)/b); G = 0 needs no rotation
        uint32_t gp = 0;
        for (int32_t k = -((D - 1 + b - 1) / b); k <= (D - 1) / b; ++k, ++gp) {
            Sched::G gg{gp, b * k, {}};
            for (int32_t bs = 0; bs < b; ++bs)
                if (gg.G + bs >= -(D - 1) && gg.G + bs <= D - 1) gg.babies.push_back((uint32_t)bs);
            s.giants.push_back(gg);
        }
        return s;
    }
    const uint32_t g = ((uint32_t)d + s.b - 1) / s.b;
    for (uint32_t gp = 0; gp < g; ++gp) {
        Sched::G gg{gp, o_min + (int32_t)(gp * s.b), {}};
        for (uint32_t bs = 0; bs < s.b; ++bs)
            if (gg.G + (int32_t)bs <= D - 1) gg.babies.push_back(bs);
        s.giants.push_back(gg);
    }
    return s;
}

// size of the double-hoisted first rotate-and-sum level (R27): cfg.rotsum_inner, a power of two (0 -> 8)
uint32_t rotsum_inner(const mmfhe_chain_cfg &cfg) { return cfg.rotsum_inner ? cfg.rotsum_inner : 8; }

// plaintext-name prefix of K3's diagonals (the aligned schedule's differ, R29)
std::string k3_prefix(const mmfhe_chain_cfg &cfg) { return cfg.bsgs_aligned ? "k3a" : "k3"; }

Sched fc_schedule(uint32_t h, uint32_t fc_baby)
{
    Sched s;
    s.b = fc_baby ? std::min(fc_baby, h) : ceil_sqrt(h);
    const uint32_t g = (h + s.b - 1) / s.b;
    for (uint32_t gp = 0; gp < g; ++gp) {
        Sched::G gg{gp, (int32_t)(gp * s.b), {}};
        for (uint32_t bs = 0; bs < s.b; ++bs)
            if (gp * s.b + bs < h) gg.babies.push_back(bs);
        s.giants.push_back(gg);
    }
    return s;
}

std::vector<uint32_t> rotsum_steps(uint32_t count, uint32_t stride)
{
    std::vector<uint32_t> out;
    for (uint32_t c = 1, s = stride; c < count; c *= 2, s *= 2) out.push_back(s);
    return out;
}

// Copy a list of batches into one contiguous batch.
DCt concat(Ctx &c, const std::vector<DCt> &parts)
{
    uint32_t total = 0;
    for (auto &p : parts) total += p.batch;
    const DCt &p0 = parts[0];
    DCt r = make_ct(c, p0.level, p0.npolys, p0.n_slots, p0.scale, total);
    uint32_t at = 0;
    for (auto &p : parts) {
        CUDA_CHECK(cudaMemcpyAsync(r.item(at), p.data(), p.item_words() * p.batch * 8, cudaMemcpyDeviceToDevice,
                                   c.stream));
        at += p.batch;
    }
    return r;
}

class Runner {
  public:
    Runner(Ctx &c, const mmfhe_chain_cfg &cfg) : c_(c), cfg_(cfg) {}

    const DPlain &plain(const std::string &name, uint32_t level, double scale,
                        const std::function<std::vector<double>()> &values, bool pq = false)
    {
        const std::string key = pq ? name + ".pq" : name;
        DPlain *p = c_.find_plain(key, level);
        if (p) return *p;
        MMFHE_REQUIRE(c_.auto_encode, MMFHE_E_MISSING_PLAIN, "missing plaintext operand " + plain_key(key, level));
        encode_plain(c_, name, values(), level, scale, pq);
        return *c_.find_plain(key, level);
    }
    // a complex-valued public vector (DESIGN R28), encoded by the library's complex encoder
    const DPlain &plain_c(const std::string &name, uint32_t level, double scale,
                          const std::function<std::vector<cd>()> &values, bool pq = false)
    {
        const std::string key = pq ? name + ".pq" : name;
        DPlain *p = c_.find_plain(key, level);
        if (p) return *p;
        MMFHE_REQUIRE(c_.auto_encode, MMFHE_E_MISSING_PLAIN, "missing plaintext operand " + plain_key(key, level));
        encode_plain_c(c_, name, values(), level, scale, pq);
        return *c_.find_plain(key, level);
    }
    bool dh() const { return cfg_.hoist == 2; }

    // DESIGN R31 (cfg.ks_merge, gesture / K3 / FC chains): relinearisation + rescale and a PQ ciphertext's
    // ModDown + rescale as ONE division by P q_l (oracle CircuitEvaluator.merge_rescale)
    DCt relin_rescale(const DCt &t3) { return cfg_.ks_merge ? ev_relin_rescale_merged(c_, t3) : ev_relin_rescale(c_, t3); }
    DCt down_rescale(const DCt &x)
    {
        return cfg_.ks_merge ? ev_moddown_rescale_ct(c_, x) : ev_rescale(c_, ev_moddown_ct(c_, x));
    }
    double qscale(uint32_t level) const { return (double)c_.primes[level]; }

    const std::vector<double> &scalars(const std::string &name, const std::function<std::vector<double>()> &fn)
    {
        auto it = c_.scalars.find(name);
        if (it != c_.scalars.end()) return it->second;
        MMFHE_REQUIRE(c_.auto_encode && fn, MMFHE_E_MISSING_PLAIN, "missing scalar table " + name);
        return c_.scalars[name] = fn();
    }

    uint32_t frame_batch(uint32_t F) const { return cfg_.frame_batch ? std::min(cfg_.frame_batch, F) : F; }

    uint32_t L() const { return lanes_of(cfg_); }

    // rotate-and-sum; with double hoisting the first min(8, count) terms are one hoisted group
    // left over Q_l u P, summed there and brought down by one ModDown (oracle rotsum_dh_all,
    // reading R27), then the remaining rotate-and-add steps
    DCt rotsum(const DCt &x, uint32_t count, uint32_t stride)
    {
        const uint32_t a = std::min<uint32_t>(rotsum_inner(cfg_), count);
        if (!dh() || a <= 1) return ev_rotsum(c_, x, count, stride);
        std::vector<int32_t> st;
        for (uint32_t j = 1; j < a; ++j) st.push_back((int32_t)(stride * j));
        // lift + the a-1 PQ steps summed in one pass (k_hoisted_rotsum_pq), one ModDown
        DCt t = ev_moddown_ct(c_, ev_rotsum_hoisted_pq(c_, x, st));
        // R30: every level hoisted (oracle rotsum_dh_all(..., all_levels)); else rotate-and-adds
        if (cfg_.rotsum_hoist_all && count / a > 1) return rotsum(t, count / a, stride * a);
        return ev_rotsum(c_, t, count / a, stride * a);
    }

    // [x, Rot(x,L), ..., Rot(x,(nb-1)L)] (L = lanes): plain HRots, or (cfg.hoist) hoisted HRots
    // sharing one ModUp
    std::vector<DCt> baby_steps(const DCt &x, uint32_t nb)
    {
        std::vector<DCt> out;
        if (dh()) {
            // double hoisting: the baby steps stay over Q_l u P (identity: the P lift)
            out.push_back(ev_lift_pq(c_, x));
            std::vector<int32_t> st;
            for (uint32_t b = 1; b < nb; ++b) st.push_back((int32_t)(b * L()));
            if (!st.empty())
                for (auto &r : ev_rotate_hoisted_pq(c_, x, st)) out.push_back(std::move(r));
            return out;
        }
        out.push_back(copy_ct(c_, x));
        if (cfg_.hoist) {
            std::vector<int32_t> st;
            for (uint32_t b = 1; b < nb; ++b) st.push_back((int32_t)(b * L()));
            if (!st.empty())
                for (auto &r : ev_rotate_hoisted(c_, x, st)) out.push_back(std::move(r));
        } else {
            for (uint32_t b = 1; b < nb; ++b) out.push_back(ev_rotate(c_, x, (int32_t)(b * L())));
        }
        return out;
    }

    // ---------------------------------------------------------- K1 / K2
    DCt k1_energy(const DCt &re, const DCt &im)
    {
        std::vector<DCt> views;
        views.reserve(2 * re.batch);
        for (uint32_t t = 0; t < re.batch; ++t) {
            views.push_back(slice(re, t, 1));
            views.push_back(slice(im, t, 1));
        }
        std::vector<std::pair<const DCt *, const DCt *>> pairs;
        for (auto &v : views) pairs.push_back({&v, &v});
        return relin_rescale(ev_tensor_sum(c_, pairs));
    }

    // K1 for S sessions at once: re[t], im[t] are batches over the sessions
    std::pair<DCt, DCt> k2_soft_attention(const DCt &E)
    {
        DCt w = copy_ct(c_, E);
        for (uint32_t i = 0; i < ilog2(cfg_.gamma); ++i) w = relin_rescale(ev_tensor_sum(c_, {{&w, &w}}));
        const uint32_t n = E.n_slots, R = cfg_.R;
        const double FFR = (double)cfg_.F * cfg_.F * R;
        const DPlain &ramp = plain("k2.ramp", w.level, qscale(w.level), [&] {
            std::vector<double> v(n, 0.0);
            for (uint32_t r = 0; r < R; ++r) v[r] = (double)r / FFR;
            return v;
        });
        const DPlain &one = plain("k2.one", w.level, qscale(w.level), [&] {
            std::vector<double> v(n, 0.0);
            for (uint32_t r = 0; r < R; ++r) v[r] = 1.0 / FFR;
            return v;
        });
        DCt Nn = ev_rescale(c_, ev_pmult_sum(c_, {{&ramp, &w}}));
        DCt Dd = ev_rescale(c_, ev_pmult_sum(c_, {{&one, &w}}));
        DCt Ns = ev_rotsum(c_, Nn, R, 1);
        DCt Ds = ev_rotsum(c_, Dd, R, 1);
        return {std::move(Ns), std::move(Ds)};
    }

    // ---------------------------------------------------------- K3 (BSGS), batched over frames
    std::pair<DCt, DCt> k3_doppler_dft(const DCt &vre, const DCt &vim)
    {
        const uint32_t n = vre.n_slots / L(), D = cfg_.D, lvl = vre.level;
        Sched s = k3_schedule(cfg_);
        std::vector<DCt> xr = baby_steps(vre, s.b), xi = baby_steps(vim, s.b);
        // W = hann[m] e^{-j 2 pi sigma(d) m / D}, diagonal o of I (x) W, pre-rotated by -G
        auto diag = [&](bool imag, int32_t o, int32_t G, bool neg) {
            std::vector<double> w = hann(D), v(n, 0.0);
            for (uint32_t j = 0; j < n; ++j) {
                const uint32_t col = (uint32_t)((((int64_t)j + o) % (int64_t)n + n) % n);
                if (j / D != col / D) continue;
                const uint32_t d = j % D, m = col % D;
                const uint32_t sig = (d + D / 2) % D;
                const double ang = -2.0 * M_PI * (double)sig * (double)m / (double)D;
                v[j] = w[m] * (imag ? std::sin(ang) : std::cos(ang)) * (neg ? -1.0 : 1.0);
            }
            return lane_rep(rot(v, -G), L());
        };
        // inner sums of every giant step in one pass over the 2b baby steps (fused diagonal
        // MAC: babies read once, each diagonal once per frame batch), then the giant rotations
        std::vector<const DCt *> cts, pr, pi;
        for (uint32_t b = 0; b < s.b; ++b) cts.push_back(&xr[b]);
        for (uint32_t b = 0; b < s.b; ++b) cts.push_back(&xi[b]);
        for (uint32_t b = 0; b < s.b; ++b) {
            pr.push_back(&xr[b]);
            pi.push_back(&xi[b]);
        }
        std::vector<std::vector<const DPlain *>> rows, PC, PS, PN;
        for (auto &g : s.giants) {
            std::vector<const DPlain *> re(2 * s.b, nullptr), im(2 * s.b, nullptr), gc(s.b, nullptr), gs(s.b, nullptr),
                gn(s.b, nullptr);
            for (uint32_t b : g.babies) {
                const int32_t o = g.G + (int32_t)b;
                const std::string sfx = "." + std::to_string(g.gp) + "." + std::to_string(b);
                const std::string k3p = k3_prefix(cfg_);
                const DPlain &pc = plain(k3p + ".c" + sfx, lvl, qscale(lvl), [&] { return diag(false, o, g.G, false); }, dh());
                const DPlain &ps = plain(k3p + ".s" + sfx, lvl, qscale(lvl), [&] { return diag(true, o, g.G, false); }, dh());
                const DPlain &pn = plain(k3p + ".ns" + sfx, lvl, qscale(lvl), [&] { return diag(true, o, g.G, true); }, dh());
                re[b] = &pc;
                re[s.b + b] = &pn;
                im[b] = &ps;
                im[s.b + b] = &pc;
                gc[b] = &pc;
                gs[b] = &ps;
                gn[b] = &pn;
            }
            rows.push_back(re);
            rows.push_back(im);
            PC.push_back(gc);
            PS.push_back(gs);
            PN.push_back(gn);
        }
        // Gauss's three-product form (ev_k3_mac: the same residues and trace, 3/4 of the MACs);
        // MMFHE_K3_GAUSS=0 selects the generic four-product diagonal MAC (A/B runs)
        static const bool gauss = [] {
            const char *e = getenv("MMFHE_K3_GAUSS");
            return !(e && *e == '0');
        }();
        std::vector<DCt> inner;  // per giant one 2B batch: d_re items, then d_im items
        if (gauss && s.b <= (uint32_t)kDiagMax && s.giants.size() <= (size_t)kDiagMax) {
            inner = ev_k3_mac(c_, pr, pi, PC, PS, PN);
        } else {
            std::vector<DCt> sep = ev_diag_mac(c_, cts, rows);
            for (size_t gi = 0; gi < s.giants.size(); ++gi) {
                std::vector<DCt> two;
                two.push_back(std::move(sep[2 * gi]));
                two.push_back(std::move(sep[2 * gi + 1]));
                inner.push_back(concat(c_, two));
            }
        }
        // per giant: rotate d_re and d_im (one 2B launch set sharing the key), then accumulate
        // (oracle k3_giant_steps' order); double hoisting fuses the accumulation into the giant
        // step's inner product
        DCt out;
        for (size_t gi = 0; gi < s.giants.size(); ++gi) {
            const int32_t step = s.giants[gi].G * (int32_t)L();
            if (gi == 0)
                out = dh() ? ev_rotate_pq(c_, inner[0], step) : ev_rotate(c_, inner[0], step);
            else if (dh())
                ev_rotate_pq_acc(c_, out, inner[gi], step);
            else
                out = ev_addsub(c_, out, ev_rotate(c_, inner[gi], step), false);
        }
        // one ModDown per output ends the giant sum (with the rescale as one division under R31)
        DCt r = dh() ? down_rescale(out) : ev_rescale(c_, out);
        const uint32_t B = vre.batch;
        return {copy_ct(c_, slice(r, 0, B)), copy_ct(c_, slice(r, B, B))};
    }

    // K3 on complex slots (DESIGN R28, oracle k3_doppler_dft_frames_c): d = W~ z with the complex
    // diagonals of I (x) W pre-rotated by -G; one plaintext product per (giant, baby) -- the
    // complex multiplication is the slot-wise plaintext product -- then the giant rotations
    DCt k3_doppler_dft_c(const DCt &z)
    {
        const uint32_t n = z.n_slots / L(), D = cfg_.D, lvl = z.level;
        Sched s = k3_schedule(cfg_);
        std::vector<DCt> xs = baby_steps(z, s.b);
        std::vector<double> w = hann(D);
        auto diag = [&](int32_t o, int32_t G) {
            std::vector<cd> v(n, cd(0, 0));
            for (uint32_t j = 0; j < n; ++j) {
                const uint32_t col = (uint32_t)((((int64_t)j + o) % (int64_t)n + n) % n);
                if (j / D != col / D) continue;
                const uint32_t d = j % D, m = col % D;
                const uint32_t sig = (d + D / 2) % D;
                const double ang = -2.0 * M_PI * (double)sig * (double)m / (double)D;
                v[j] = w[m] * std::polar(1.0, ang);
            }
            return lane_rep(rot(v, -G), L());
        };
        std::vector<const DCt *> cts;
        for (auto &x : xs) cts.push_back(&x);
        std::vector<std::vector<const DPlain *>> rows;
        for (auto &g : s.giants) {
            std::vector<const DPlain *> row(s.b, nullptr);
            for (uint32_t b : g.babies) {
                const std::string name = k3_prefix(cfg_) + ".w." + std::to_string(g.gp) + "." + std::to_string(b);
                row[b] = &plain_c(name, lvl, qscale(lvl), [&] { return diag(g.G + (int32_t)b, g.G); }, dh());
            }
            rows.push_back(row);
        }
        std::vector<DCt> inner = ev_diag_mac(c_, cts, rows);
        DCt out;
        for (size_t gi = 0; gi < s.giants.size(); ++gi) {
            const int32_t step = s.giants[gi].G * (int32_t)L();
            if (gi == 0)
                out = dh() ? ev_rotate_pq(c_, inner[0], step) : ev_rotate(c_, inner[0], step);
            else if (dh())
                ev_rotate_pq_acc(c_, out, inner[gi], step);
            else
                out = ev_addsub(c_, out, ev_rotate(c_, inner[gi], step), false);
        }
        return dh() ? down_rescale(out) : ev_rescale(c_, out);
    }

    // ---------------------------------------------------------- gesture frame (batched)
    DCt k1_power(const DCt &dre, const DCt &dim)
    {
        return relin_rescale(ev_tensor_sum(c_, {{&dre, &dre}, {&dim, &dim}}));
    }

    // K1 on complex K3 outputs (oracle k1_power_c): |d|^2 = d Conj(d); with k1_conj_fuse (R32) one
    // conjugate-product key switch sharing a single division by P q_l
    DCt k1_power_c(const DCt &d)
    {
        if (cfg_.k1_conj_fuse) return ev_conj_mul_relin_rescale(c_, d);
        DCt cj = ev_conjugate(c_, d);
        return relin_rescale(ev_tensor_sum(c_, {{&d, &cj}}));
    }

    DCt k6_notch(const DCt &P)
    {
        const uint32_t D = cfg_.D, n = P.n_slots / L();
        const DPlain &m = plain("k6.mask", P.level, qscale(P.level), [&] {
            std::vector<double> w = hann(D);
            double sw = 0;
            for (double x : w) sw += x;
            const double s = (double)cfg_.R * cfg_.A * sw * sw;
            const uint32_t width = cfg_.notch_width ? cfg_.notch_width : 1;
            const uint32_t lo = D / 2 - (width - 1) / 2;
            std::vector<double> v(n);
            for (uint32_t j = 0; j < n; ++j) {
                const uint32_t d = j % D;
                v[j] = (d >= lo && d < lo + width) ? 0.0 : 1.0 / s;
            }
            return lane_rep(v, L());
        });
        return ev_rescale(c_, ev_pmult_sum(c_, {{&m, &P}}));
    }

    DCt k2_doppler_soft_power(const DCt &Pm)
    {
        DCt S = rotsum(Pm, Pm.n_slots / L() / cfg_.D, cfg_.D * L());
        for (uint32_t i = 0; i < ilog2(cfg_.gamma); ++i) S = relin_rescale(ev_tensor_sum(c_, {{&S, &S}}));
        DCt Pd = ev_drop_to(c_, Pm, S.level);
        return relin_rescale(ev_tensor_sum(c_, {{&Pd, &S}}));
    }

    DCt gesture_frame(const DCt &vre, const DCt &vim)
    {
        auto d = k3_doppler_dft(vre, vim);
        DCt P = k1_power(d.first, d.second);
        DCt Pm = k6_notch(P);
        return k2_doppler_soft_power(Pm);
    }

    DCt gesture_frame_c(const DCt &z) { return k2_doppler_soft_power(k6_notch(k1_power_c(k3_doppler_dft_c(z)))); }

    // ---------------------------------------------------------- FC
    DCt fc_layer(const DCt &x, uint32_t layer, bool square)
    {
        const uint32_t n_in = cfg_.fc_dims[layer - 1], h = cfg_.fc_dims[layer];
        const uint32_t lvl = x.level;
        Sched s = fc_schedule(h, cfg_.fc_baby);
        const std::vector<double> *W = nullptr, *bias = nullptr;
        if (c_.fc_w.size() >= layer) {
            W = &c_.fc_w[layer - 1];
            bias = &c_.fc_b[layer - 1];
        }
        std::vector<DCt> babies = baby_steps(x, std::min(s.b, h));
        std::vector<const DCt *> cts;
        for (auto &bb : babies) cts.push_back(&bb);
        std::vector<std::vector<const DPlain *>> rows;
        for (auto &g : s.giants) {
            std::vector<const DPlain *> row(babies.size(), nullptr);
            for (uint32_t b : g.babies) {
                const uint32_t i = (uint32_t)g.G + b;
                const std::string name = "fc" + std::to_string(layer) + ".d." + std::to_string(g.gp) + "." +
                                         std::to_string(b);
                row[b] = &plain(name, lvl, qscale(lvl), [&] {
                    MMFHE_REQUIRE(W != nullptr, MMFHE_E_MISSING_PLAIN, "FC weights not prepared");
                    std::vector<double> v(n_in);
                    for (uint32_t j = 0; j < n_in; ++j) v[j] = (*W)[(size_t)(j % h) * n_in + (j + i) % n_in];
                    return lane_rep(rot(v, -g.G), L());
                }, dh());
            }
            rows.push_back(row);
        }
        std::vector<DCt> inners = ev_diag_mac(c_, cts, rows);
        DCt acc;
        for (size_t gi = 0; gi < s.giants.size(); ++gi) {
            const auto &g = s.giants[gi];
            const int32_t step = g.G * (int32_t)L();
            if (gi > 0 && dh() && g.G) {  // rotate + accumulate, fused
                ev_rotate_pq_acc(c_, acc, inners[gi], step);
                continue;
            }
            DCt inner = std::move(inners[gi]);
            if (g.G) inner = dh() ? ev_rotate_pq(c_, inner, step) : ev_rotate(c_, inner, step);
            acc = gi == 0 ? std::move(inner) : ev_addsub(c_, acc, inner, false);
        }
        DCt z = dh() ? down_rescale(acc) : ev_rescale(c_, acc);
        DCt y = rotsum(z, n_in / h, h * L());
        const DPlain &bp = plain("fc" + std::to_string(layer) + ".bias", y.level, y.scale, [&] {
            MMFHE_REQUIRE(bias != nullptr, MMFHE_E_MISSING_PLAIN, "FC bias not prepared");
            return lane_rep(*bias, L());
        });
        y = ev_add_plain(c_, y, bp);
        if (square) y = relin_rescale(ev_tensor_sum(c_, {{&y, &y}}));
        return y;
    }

    // With L lanes the frames' features are first summed across lanes (lane 0 then holds the
    // session's features; oracle gesture_fc): before the first nonlinearity, after the frame
    // sum, so frame-sharded partial sums stay exact modular sums
    DCt gesture_fc(const DCt &feat)
    {
        DCt x = L() > 1 ? fc_layer(rotsum(feat, L(), 1), 1, true) : fc_layer(feat, 1, true);
        x = fc_layer(x, 2, true);
        return fc_layer(x, 3, false);
    }

    // ---------------------------------------------------------- vital V2 (batched over frames)
    std::pair<DCt, DCt> k4_soft_iq(const DCt &re, const DCt &im)
    {
        DCt p = relin_rescale(ev_tensor_sum(c_, {{&re, &re}, {&im, &im}}));
        for (uint32_t i = 0; i < ilog2(cfg_.p_phi); ++i) p = relin_rescale(ev_tensor_sum(c_, {{&p, &p}}));
        DCt red = ev_drop_to(c_, re, p.level);
        DCt i_ = relin_rescale(ev_tensor_sum(c_, {{&p, &red}}));
        DCt imd = ev_drop_to(c_, im, p.level);
        DCt q_ = relin_rescale(ev_tensor_sum(c_, {{&p, &imd}}));
        if (cfg_.iq_pack) {
            // reading R19: pack i, q (and 2^(k-1) frames) into the slot blocks of one
            // ciphertext, one rotate-and-sum, unpack (see oracle k4_packed_rotsum)
            const int32_t R = (int32_t)cfg_.R;
            const uint32_t k = cfg_.iq_pack;
            MMFHE_REQUIRE(i_.batch % (1u << (k - 1)) == 0, MMFHE_E_SHAPE,
                          "iq_pack = k needs a multiple of 2^(k-1) frames per frame batch");
            DCt x = ev_rot_add(c_, i_, q_, -R);
            for (uint32_t j = 1; j < k; ++j) {
                const uint32_t h = x.batch / 2;
                x = ev_rot_add(c_, slice(x, 0, h), slice(x, h, h), -(R << j));
            }
            x = ev_rotsum(c_, x, cfg_.R, 1);
            if (cfg_.hoist) {
                // every unpacking rotation acts on the packed x: one hoisted group
                // Rot(x, mR), m = 1..2^k - 1, sharing one ModUp (oracle k4_packed_rotsum)
                std::vector<int32_t> st;
                for (uint32_t mm = 1; mm < (1u << k); ++mm) st.push_back((int32_t)mm * R);
                std::vector<DCt> blocks;
                blocks.push_back(std::move(x));
                for (auto &r : ev_rotate_hoisted(c_, blocks[0], st)) blocks.push_back(std::move(r));
                std::vector<uint32_t> seq{0};
                for (uint32_t j = k - 1; j >= 1; --j) {
                    const size_t n0 = seq.size();
                    for (size_t i = 0; i < n0; ++i) seq.push_back(seq[i] + (1u << j));
                }
                std::vector<DCt> ip, qp;
                for (uint32_t sft : seq) {
                    ip.push_back(slice(blocks[sft], 0, blocks[sft].batch));
                    qp.push_back(slice(blocks[sft + 1], 0, blocks[sft + 1].batch));
                }
                DCt I = concat(c_, ip), Q = concat(c_, qp);
                return {std::move(I), std::move(Q)};
            }
            for (uint32_t j = k - 1; j >= 1; --j) {
                DCt hi = ev_rotate(c_, x, R << j);
                std::vector<DCt> parts;
                parts.push_back(std::move(x));
                parts.push_back(std::move(hi));
                x = concat(c_, parts);
            }
            DCt Q = ev_rotate(c_, x, R);
            return {std::move(x), std::move(Q)};
        }
        DCt I = ev_rotsum(c_, i_, cfg_.R, 1);
        DCt Q = ev_rotsum(c_, q_, cfg_.R, 1);
        return {std::move(I), std::move(Q)};
    }

    // I_f[t] = sum_{k <= t} h[k] I[t-k]: banded Toeplitz product over the frame batch, then rescale
    DCt k5_fir(const DCt &x, const std::vector<double> &taps)
    {
        const uint32_t F = x.batch, W = (uint32_t)taps.size();
        std::vector<double> coef((size_t)F * W);
        for (uint32_t j = 0; j < F; ++j)
            for (uint32_t w = 0; w < W; ++w) coef[(size_t)j * W + w] = taps[W - 1 - w];
        return ev_rescale(c_, ev_lincomb_mat(c_, x, F, W, -(int)(W - 1), 1, coef));
    }

    // K5 "Alternate Implementation": y = sum_k h[k] Rot(x, -k) for a sequence packed
    // in the slots of one ciphertext (oracle k5_fir_rot): hoisted baby steps Rot(x, -s), per giant
    // the exact scalar combination of the babies, giant rotation by -g'b, sum, one rescale
    DCt k5_fir_rot(const DCt &x, const std::vector<double> &taps)
    {
        const uint32_t W = (uint32_t)taps.size(), b = ceil_sqrt(W), g = (W + b - 1) / b, nb = std::min(b, W);
        std::vector<DCt> babies;
        babies.push_back(copy_ct(c_, x));
        std::vector<int32_t> st;
        for (uint32_t s = 1; s < nb; ++s) st.push_back(-(int32_t)s);
        if (!st.empty()) {
            if (cfg_.hoist) {
                for (auto &r : ev_rotate_hoisted(c_, x, st)) babies.push_back(std::move(r));
            } else {
                for (int32_t s : st) babies.push_back(ev_rotate(c_, x, s));
            }
        }
        DCt all = babies.size() == 1 ? std::move(babies[0]) : concat(c_, babies);
        const uint32_t full = W / b, last = W - full * b;  // giants with b taps, then a partial one
        std::vector<DCt> inners;
        if (full) {
            std::vector<double> coef((size_t)full * nb);
            for (uint32_t j = 0; j < full; ++j)
                for (uint32_t s = 0; s < nb; ++s) coef[(size_t)j * nb + s] = taps[j * b + s];
            DCt r = ev_lincomb_mat(c_, all, full, nb, 0, 0, coef);
            for (uint32_t j = 0; j < full; ++j) inners.push_back(copy_ct(c_, slice(r, j, 1)));
        }
        if (last) {
            std::vector<double> coef(taps.begin() + full * b, taps.end());
            inners.push_back(ev_lincomb_mat(c_, all, 1, last, 0, 0, coef));
        }
        MMFHE_REQUIRE(inners.size() == g, MMFHE_E_SHAPE, "FIR giant count");
        DCt acc = std::move(inners[0]);
        for (uint32_t j = 1; j < g; ++j) acc = ev_addsub(c_, acc, ev_rotate(c_, inners[j], -(int32_t)(j * b)), false);
        return ev_rescale(c_, acc);
    }

    DCt k7_taylor_phase(const DCt &If, const DCt &Qf)
    {
        const uint32_t F = If.batch;
        DCt I1 = slice(If, 1, F - 1), I0 = slice(If, 0, F - 1);
        DCt Q1 = slice(Qf, 1, F - 1), Q0 = slice(Qf, 0, F - 1);
        DCt ty = ev_tensor_sum(c_, {{&Q1, &I0}});
        DCt ty2 = ev_tensor_sum(c_, {{&I1, &Q0}});
        DCt y = relin_rescale(ev_addsub(c_, ty, ty2, true));
        if (cfg_.taylor_order == 1) return y;
        DCt x = relin_rescale(ev_tensor_sum(c_, {{&I1, &I0}, {&Q1, &Q0}}));
        DCt x2 = relin_rescale(ev_tensor_sum(c_, {{&x, &x}}));
        DCt y2 = relin_rescale(ev_tensor_sum(c_, {{&y, &y}}));
        std::vector<double> third(y.batch, -1.0 / 3.0);
        DCt yt = ev_rescale(c_, ev_lincomb_mat(c_, y, y.batch, 1, 0, 1, third));
        DCt yd = ev_drop_to(c_, y, x2.level);
        DCt yx2 = relin_rescale(ev_tensor_sum(c_, {{&yd, &x2}}));
        DCt y3 = relin_rescale(ev_tensor_sum(c_, {{&y2, &yt}}));
        return ev_addsub(c_, yx2, y3, false);
    }

    DCt vp_band_power(const DCt &ys, uint32_t band)
    {
        const uint32_t Fp = ys.batch, K = cfg_.n_bins[band];
        std::vector<double> coef((size_t)2 * K * Fp);
        for (uint32_t bi = 0; bi < K; ++bi) {
            const uint32_t k = cfg_.bins[band][bi];
            const std::string sfx = "." + std::to_string(band) + "." + std::to_string(k);
            auto gen = [=](bool imag) {
                return [=]() {
                    std::vector<double> w = hann(Fp), v(Fp);
                    for (uint32_t t = 0; t < Fp; ++t) {
                        const double ang = 2.0 * M_PI * (double)k * t / (double)Fp;
                        v[t] = imag ? -w[t] * std::sin(ang) / Fp : w[t] * std::cos(ang) / Fp;
                    }
                    return v;
                };
            };
            const std::vector<double> &cc = scalars("vp.c" + sfx, gen(false));
            const std::vector<double> &ss = scalars("vp.s" + sfx, gen(true));
            MMFHE_REQUIRE(cc.size() == Fp && ss.size() == Fp, MMFHE_E_SHAPE, "DFT coefficient count");
            std::copy(cc.begin(), cc.end(), coef.begin() + (size_t)bi * Fp);
            std::copy(ss.begin(), ss.end(), coef.begin() + (size_t)(K + bi) * Fp);
        }
        DCt X = ev_rescale(c_, ev_lincomb_mat(c_, ys, 2 * K, Fp, 0, 0, coef));
        DCt Xr = slice(X, 0, K), Xi = slice(X, K, K);
        return relin_rescale(ev_tensor_sum(c_, {{&Xr, &Xr}, {&Xi, &Xi}}));
    }

    // VP+ (SURVEY §8(c)-7): sharpen S_k = P_k^2, then N_f = sum_k f_k S_k and
    // D_f = sum_k S_k (f_k = k fs / Fp Hz) as one 2-output scalar matrix product + rescale
    DCt vp_weighted_average(const DCt &Pk, uint32_t band, uint32_t Fp)
    {
        const uint32_t K = Pk.batch;
        DCt S = relin_rescale(ev_tensor_sum(c_, {{&Pk, &Pk}}));
        std::vector<double> coef((size_t)2 * K);
        for (uint32_t bi = 0; bi < K; ++bi) {
            coef[bi] = (double)cfg_.bins[band][bi] * cfg_.fs / (double)Fp;
            coef[K + bi] = 1.0;
        }
        return ev_rescale(c_, ev_lincomb_mat(c_, S, 2, K, 0, 0, coef));
    }

    // K4 over every frame batch of (re_t, im_t) inputs: (I, Q) each a batch of F items
    std::pair<DCt, DCt> k4_all_frames(const mmfhe_ct *in, size_t n_in)
    {
        const uint32_t F = (uint32_t)(n_in / 2), fb = frame_batch(F);
        std::vector<DCt> Is, Qs;
        for (uint32_t t0 = 0; t0 < F; t0 += fb) {
            const uint32_t cnt = std::min(fb, F - t0);
            DCt re = import_batch(c_, in, 2 * (size_t)t0, 2, cnt);
            DCt im = import_batch(c_, in, 2 * (size_t)t0 + 1, 2, cnt);
            auto iq = k4_soft_iq(re, im);
            Is.push_back(std::move(iq.first));
            Qs.push_back(std::move(iq.second));
        }
        DCt I = Is.size() == 1 ? std::move(Is[0]) : concat(c_, Is);
        DCt Q = Qs.size() == 1 ? std::move(Qs[0]) : concat(c_, Qs);
        return {std::move(I), std::move(Q)};
    }

    const std::vector<double> &band_taps(uint32_t b)
    {
        const std::vector<double> &taps = scalars("k5.b" + std::to_string(b), nullptr);
        MMFHE_REQUIRE(cfg_.n_taps[b] == 0 || taps.size() == cfg_.n_taps[b], MMFHE_E_SHAPE, "FIR tap count");
        return taps;
    }

    std::vector<DCt> vitals_v2(const mmfhe_ct *in, size_t n_in)
    {
        auto iq = k4_all_frames(in, n_in);
        const DCt &I = iq.first, &Q = iq.second;
        std::vector<DCt> out;
        for (uint32_t b = 0; b < cfg_.n_bands; ++b) {
            const std::vector<double> &taps = band_taps(b);
            DCt If = k5_fir(I, taps);
            DCt Qf = k5_fir(Q, taps);
            DCt ys = k7_taylor_phase(If, Qf);
            DCt Pk = vp_band_power(ys, b);
            out.push_back(cfg_.vp_plus ? vp_weighted_average(Pk, b, ys.batch) : std::move(Pk));
        }
        return out;
    }

    // per frame batch: frame kernels, batch sum; batches added in order
    DCt gesture_features(const mmfhe_ct *in, size_t n_in)
    {
        const uint32_t F = (uint32_t)(cfg_.cplx ? n_in : n_in / 2), fb = frame_batch(F);
        DCt acc;
        for (uint32_t t0 = 0; t0 < F; t0 += fb) {
            const uint32_t cnt = std::min(fb, F - t0);
            DCt f;
            if (cfg_.cplx) {
                f = gesture_frame_c(import_batch(c_, in, t0, 1, cnt));
            } else {
                DCt vre = import_batch(c_, in, 2 * (size_t)t0, 2, cnt);
                DCt vim = import_batch(c_, in, 2 * (size_t)t0 + 1, 2, cnt);
                f = gesture_frame(vre, vim);
            }
            DCt part = ev_batch_sum(c_, f);
            acc = t0 == 0 ? std::move(part) : ev_addsub(c_, acc, part, false);
        }
        return acc;
    }

    // S sessions' inputs (S equal contiguous runs) as ONE batch through the per-frame chain, then
    // each session's frames summed on their own: item s = session s's features (cfg.sessions)
    DCt gesture_features_sessions(const mmfhe_ct *in, size_t n_in, uint32_t S)
    {
        DCt f;
        if (cfg_.cplx) {
            f = gesture_frame_c(import_batch(c_, in, 0, 1, n_in));
        } else {
            DCt vre = import_batch(c_, in, 0, 2, n_in / 2);
            DCt vim = import_batch(c_, in, 1, 2, n_in / 2);
            f = gesture_frame(vre, vim);
        }
        return ev_batch_sum_runs(c_, f, S);
    }

    DCt gesture(const mmfhe_ct *in, size_t n_in) { return gesture_fc(gesture_features(in, n_in)); }

  private:
    Ctx &c_;
    const mmfhe_chain_cfg &cfg_;
};

bool pow2_or_zero(uint32_t x) { return (x & (x - 1)) == 0; }

// Public-parameter checks shared by chain_plan and chain_rotations (the oracle raises on
// the same inputs): exponents are powers of two (log2 squarings),
// K7 is first or third order, and the packed K4 rotate-and-sum needs R a power
// of two (its blocks sit at multiples of R and one rotsum adds 2^ceil(log2 R) slots).
void validate_cfg(const std::string &chain, const mmfhe_chain_cfg &cfg)
{
    MMFHE_REQUIRE(pow2_or_zero(cfg.gamma), MMFHE_E_INVALID_ARG, "gamma must be a power of two");
    MMFHE_REQUIRE(pow2_or_zero(cfg.p_phi), MMFHE_E_INVALID_ARG, "p_phi must be a power of two");
    if (chain == "vitals_v2" || chain == "k7_taylor_phase")
        MMFHE_REQUIRE(cfg.taylor_order == 1 || cfg.taylor_order == 3, MMFHE_E_INVALID_ARG,
                      "taylor_order must be 1 or 3");
    if ((chain == "vitals_v2" || chain == "k4_soft_iq") && cfg.iq_pack)
        MMFHE_REQUIRE(cfg.R >= 1 && pow2_or_zero(cfg.R), MMFHE_E_SHAPE, "iq_pack needs R a power of two");
    MMFHE_REQUIRE(pow2_or_zero(cfg.lanes), MMFHE_E_SHAPE, "lanes must be a power of two");
    MMFHE_REQUIRE(cfg.hoist <= 2, MMFHE_E_INVALID_ARG, "hoist must be 0, 1 or 2");
    MMFHE_REQUIRE(cfg.cplx <= 1, MMFHE_E_INVALID_ARG, "cplx must be 0 or 1");
    MMFHE_REQUIRE(cfg.bsgs_aligned <= 1, MMFHE_E_INVALID_ARG, "bsgs_aligned must be 0 or 1");
    MMFHE_REQUIRE(pow2_or_zero(cfg.rotsum_inner) && cfg.rotsum_inner <= 64, MMFHE_E_INVALID_ARG,
                  "rotsum_inner must be a power of two <= 64");
    MMFHE_REQUIRE(cfg.rotsum_hoist_all <= 1, MMFHE_E_INVALID_ARG, "rotsum_hoist_all must be 0 or 1");
    MMFHE_REQUIRE(cfg.ks_merge <= 1, MMFHE_E_INVALID_ARG, "ks_merge must be 0 or 1");
    MMFHE_REQUIRE(cfg.k1_conj_fuse <= 1, MMFHE_E_INVALID_ARG, "k1_conj_fuse must be 0 or 1");
    MMFHE_REQUIRE(!cfg.k1_conj_fuse || (cfg.cplx && cfg.ks_merge), MMFHE_E_INVALID_ARG,
                  "k1_conj_fuse needs cplx and ks_merge");
    if (cfg.ks_merge)
        MMFHE_REQUIRE(chain == "gesture" || chain == "gesture_frame" || chain == "gesture_features" ||
                          chain == "gesture_fc" || chain == "fc_forward" || chain == "k3_doppler_dft" ||
                          chain == "vitals_v1" || chain == "vitals_v2",
                      MMFHE_E_SHAPE, "ks_merge applies to the gesture / K3 / FC / vital V1, V2 chains only");
    if (cfg.sessions > 1)
        MMFHE_REQUIRE(chain == "gesture_features", MMFHE_E_SHAPE, "sessions > 1 applies to gesture_features only");
    if (cfg.cplx)
        MMFHE_REQUIRE(cplx_chain(chain, cfg) || chain == "gesture_fc" || chain == "fc_forward" ||
                          chain == "k2_doppler_soft_power" || chain == "k6_notch",
                      MMFHE_E_SHAPE, "complex slots apply to the K3 / gesture chains only");
}

uint32_t chain_depth(const std::string &chain, const mmfhe_chain_cfg &cfg)
{
    validate_cfg(chain, cfg);
    const uint32_t lg = ilog2(cfg.gamma ? cfg.gamma : 1), lp = ilog2(cfg.p_phi ? cfg.p_phi : 1);
    const uint32_t gf = 3 + lg + 1, fc = 5;
    const uint32_t v2 = (1 + lp + 1) + 1 + (cfg.taylor_order == 3 ? 3 : 1) + 1 + 1 + (cfg.vp_plus ? 2 : 0);
    if (chain == "k1_energy") return 1;
    if (chain == "vitals_v1") return 1 + lg + 1;
    if (chain == "vitals_v2") return v2;
    if (chain == "k3_doppler_dft") return 1;
    if (chain == "gesture_frame") return gf;
    if (chain == "gesture_fc") return fc;
    if (chain == "gesture") return gf + fc;
    if (chain == "gesture_features") return gf;
    // the paper's kernels on their own ("can be used individually or composed")
    if (chain == "k2_soft_attention") return lg + 1;
    if (chain == "k2_doppler_soft_power") return lg + 1;
    if (chain == "k4_soft_iq") return 1 + lp + 1;
    if (chain == "k5_fir" || chain == "k5_fir_rot") return 1;
    if (chain == "k6_notch") return 1;
    if (chain == "k7_taylor_phase") return cfg.taylor_order == 3 ? 3 : 1;
    if (chain == "fc_forward") return fc;
    throw Error(MMFHE_E_INVALID_ARG, "unknown chain " + chain);
}

}  // namespace

std::vector<int32_t> chain_rotations(const Ctx &c, const std::string &chain, const mmfhe_chain_cfg &cfg)
{
    std::set<int32_t> ks;
    const int32_t half = (int32_t)(c.n / 2);
    auto add = [&](int64_t k) {
        int32_t v = (int32_t)(((k % half) + half) % half);
        if (v) ks.insert(v);
    };
    chain_depth(chain, cfg);  // validates the name
    if (chain == "vitals_v1" || chain == "vitals_v2" || chain == "k2_soft_attention" || chain == "k4_soft_iq")
        for (uint32_t s : rotsum_steps(cfg.R, 1)) add(s);
    if ((chain == "vitals_v2" || chain == "k4_soft_iq") && cfg.iq_pack) {
        MMFHE_REQUIRE(cfg.iq_pack <= 8 && ((size_t)cfg.R << cfg.iq_pack) <= (size_t)(cfg.n_slots ? cfg.n_slots : c.n / 2),
                      MMFHE_E_SHAPE, "iq_pack = k needs 2^k R <= n slots");
        for (uint32_t j = 0; j < cfg.iq_pack; ++j) {
            add((int64_t)cfg.R << j);
            add(-((int64_t)cfg.R << j));
        }
        if (cfg.hoist)
            for (uint32_t mm = 1; mm < (1u << cfg.iq_pack); ++mm) add((int64_t)mm * cfg.R);
    }
    if (chain == "k5_fir_rot") {
        uint32_t W = 0;
        for (uint32_t b = 0; b < cfg.n_bands; ++b) W = std::max(W, cfg.n_taps[b]);
        if (W) {
            const uint32_t b = ceil_sqrt(W), g = (W + b - 1) / b;
            for (uint32_t s = 1; s < std::min(b, W); ++s) add(-(int64_t)s);
            for (uint32_t j = 1; j < g; ++j) add(-(int64_t)(j * b));
        }
    }
    const bool frames = chain == "gesture_frame" || chain == "gesture" || chain == "gesture_features";
    const int64_t L = lanes_of(cfg);
    if (chain == "k3_doppler_dft" || frames) {
        Sched s = k3_schedule(cfg);
        for (uint32_t b = 1; b < s.b; ++b) add(b * L);
        for (auto &g : s.giants) add(g.G * L);
    }
    // a rotate-and-sum's keys; with double hoisting (R27) also j stride, j < min(8, count)
    auto add_rotsum = [&](uint32_t count, uint32_t stride) {
        if (cfg.hoist == 2) {  // the double-hoisted levels (R27 / R30), then plain rotate-and-add steps
            do {
                const uint32_t a = std::min<uint32_t>(rotsum_inner(cfg), count);
                if (a <= 1) break;
                for (uint32_t j = 1; j < a; ++j) add((int64_t)j * stride);
                count /= a;
                stride *= a;
            } while (cfg.rotsum_hoist_all && count > 1);
        }
        for (uint32_t s : rotsum_steps(count, stride)) add(s);
    };
    if (frames || chain == "k2_doppler_soft_power") add_rotsum(cfg.n_slots / cfg.D, cfg.D * (uint32_t)L);
    if (frames && cfg.cplx) ks.insert(MMFHE_STEP_CONJ);  // K1 = d Conj(d) (DESIGN R28)
    if (frames && cfg.cplx && cfg.k1_conj_fuse) ks.insert(MMFHE_STEP_CONJ_PROD);  // R32
    if (chain == "gesture_fc" || chain == "gesture" || chain == "fc_forward") {
        add_rotsum((uint32_t)L, 1);
        for (int layer = 0; layer < 3; ++layer) {
            const uint32_t h = cfg.fc_dims[layer + 1], n_in = cfg.fc_dims[layer];
            Sched s = fc_schedule(h, cfg.fc_baby);
            for (uint32_t b = 1; b < std::min(s.b, h); ++b) add(b * L);
            for (auto &g : s.giants) add(g.G * L);
            add_rotsum(n_in / h, h * (uint32_t)L);
        }
    }
    return std::vector<int32_t>(ks.begin(), ks.end());
}

std::vector<uint32_t> chain_plan(const Ctx &c, const std::string &chain, const mmfhe_chain_cfg &cfg, uint32_t in_level,
                                 size_t n_in)
{
    const uint32_t dep = chain_depth(chain, cfg);
    MMFHE_REQUIRE(in_level >= dep, MMFHE_E_DEPTH,
                  "chain " + chain + " needs " + std::to_string(dep) + " levels, input has " +
                      std::to_string(in_level));
    const uint32_t out = in_level - dep;
    size_t n_out = 1;
    if (chain == "k1_energy") {
        // S independent sessions of F frames: inputs session-major, (re_t, im_t) per frame
        MMFHE_REQUIRE(cfg.F > 0 && n_in % (2 * (size_t)cfg.F) == 0, MMFHE_E_SHAPE,
                      "expected 2F input ciphertexts per session");
        n_out = n_in / (2 * (size_t)cfg.F);
    } else if (chain == "vitals_v1" || chain == "vitals_v2") {
        MMFHE_REQUIRE(n_in == 2 * (size_t)cfg.F && cfg.F > 0, MMFHE_E_SHAPE, "expected 2F input ciphertexts");
    } else if (chain == "gesture") {
        const size_t L = lanes_of(cfg);
        if (cfg.cplx)
            MMFHE_REQUIRE(cfg.F > 0 && n_in == (cfg.F + L - 1) / L, MMFHE_E_SHAPE,
                          "expected ceil(F / lanes) complex-slot input ciphertexts");
        else
            MMFHE_REQUIRE(cfg.F > 0 && n_in == 2 * ((cfg.F + L - 1) / L), MMFHE_E_SHAPE,
                          "expected 2 ceil(F / lanes) input ciphertexts");
    } else if (cplx_chain(chain, cfg)) {  // k3_doppler_dft / gesture_frame / gesture_features
        MMFHE_REQUIRE(n_in >= 1, MMFHE_E_SHAPE, "expected one complex-slot ciphertext z per frame (group)");
        n_out = chain == "gesture_features" ? 1 : n_in;
    } else if (chain == "k3_doppler_dft" || chain == "gesture_frame" || chain == "gesture_features") {
        MMFHE_REQUIRE(n_in >= 2 && n_in % 2 == 0, MMFHE_E_SHAPE, "expected (v_re, v_im) per frame");
        n_out = chain == "k3_doppler_dft" ? n_in : chain == "gesture_frame" ? n_in / 2 : 1;
    }
    if (chain == "gesture_features" && cfg.sessions > 1) {
        const size_t per = cfg.cplx ? 1 : 2, groups = n_in / per;
        MMFHE_REQUIRE(groups % cfg.sessions == 0, MMFHE_E_SHAPE,
                      "sessions > 1: the inputs must split into equal runs, one per session");
        MMFHE_REQUIRE(cfg.frame_batch == 0 || cfg.frame_batch >= groups, MMFHE_E_SHAPE,
                      "sessions > 1 runs every session's frames as one batch (frame_batch 0)");
        n_out = cfg.sessions;
    } else if (chain == "gesture_fc" || chain == "fc_forward") {
        // one feature ciphertext per session, the sessions as one batch (one launch per op)
        MMFHE_REQUIRE(n_in >= 1, MMFHE_E_SHAPE, "expected one feature ciphertext per session");
        n_out = n_in;
    } else if (chain == "k2_soft_attention") {
        MMFHE_REQUIRE(n_in == 1 && cfg.F > 0, MMFHE_E_SHAPE, "expected one energy ciphertext E (and cfg.F)");
        n_out = 2;
    } else if (chain == "k2_doppler_soft_power" || chain == "k6_notch") {
        MMFHE_REQUIRE(cfg.D > 0 && cfg.n_slots % cfg.D == 0, MMFHE_E_SHAPE, "D must divide the packing period");
        n_out = n_in;
    } else if (chain == "k4_soft_iq") {
        MMFHE_REQUIRE(n_in == 2 * (size_t)cfg.F && cfg.F > 0, MMFHE_E_SHAPE, "expected 2F input ciphertexts");
        n_out = n_in;
        if (cfg.iq_pack) {
            const uint32_t g = 1u << (cfg.iq_pack - 1), fb = cfg.frame_batch ? std::min(cfg.frame_batch, cfg.F) : cfg.F;
            MMFHE_REQUIRE(cfg.iq_pack <= 8 && fb % g == 0 && (cfg.F % fb) % g == 0, MMFHE_E_SHAPE,
                          "iq_pack = k needs a multiple of 2^(k-1) frames in every frame batch");
            MMFHE_REQUIRE(((size_t)cfg.R << cfg.iq_pack) <= (size_t)(cfg.n_slots ? cfg.n_slots : c.n / 2),
                          MMFHE_E_SHAPE, "iq_pack = k needs 2^k R <= n slots");
        }
    } else if (chain == "k5_fir" || chain == "k5_fir_rot") {
        MMFHE_REQUIRE(n_in >= 1 && cfg.n_bands >= 1 && cfg.n_bands <= 4, MMFHE_E_SHAPE,
                      "expected a frame sequence and 1..4 FIR bands");
        n_out = n_in * cfg.n_bands;
    } else if (chain == "k7_taylor_phase") {
        MMFHE_REQUIRE(n_in >= 4 && n_in % 2 == 0, MMFHE_E_SHAPE, "expected (I_f, Q_f) per frame, F >= 2");
        n_out = n_in / 2 - 1;
    }
    if (chain == "vitals_v2") {
        MMFHE_REQUIRE(cfg.F >= 2 && cfg.n_bands <= 4, MMFHE_E_SHAPE, "vitals_v2 needs F >= 2 and <= 4 bands");
        for (uint32_t b = 0; b < cfg.n_bands; ++b)
            MMFHE_REQUIRE(cfg.n_bins[b] >= 1 && cfg.n_bins[b] <= 64, MMFHE_E_SHAPE, "1..64 DFT bins per band");
        if (cfg.iq_pack) {
            // every K4 frame batch (the last one may be short) must hold whole packing groups
            const uint32_t g = 1u << (cfg.iq_pack - 1), fb = cfg.frame_batch ? std::min(cfg.frame_batch, cfg.F) : cfg.F;
            MMFHE_REQUIRE(cfg.iq_pack <= 8 && fb % g == 0 && (cfg.F % fb) % g == 0, MMFHE_E_SHAPE,
                          "iq_pack = k needs a multiple of 2^(k-1) frames in every frame batch");
            MMFHE_REQUIRE(((size_t)cfg.R << cfg.iq_pack) <= (size_t)(cfg.n_slots ? cfg.n_slots : c.n / 2),
                          MMFHE_E_SHAPE, "iq_pack = k needs 2^k R <= n slots");
        }
    }
    if (lanes_of(cfg) > 1) {
        const bool lane_chain = chain == "gesture" || chain == "gesture_frame" || chain == "gesture_features" ||
                                chain == "gesture_fc" || chain == "k3_doppler_dft" || chain == "fc_forward" ||
                                chain == "k2_doppler_soft_power" || chain == "k6_notch";
        MMFHE_REQUIRE(lane_chain, MMFHE_E_SHAPE, "lanes > 1 applies to the gesture / K3 chains only");
        MMFHE_REQUIRE((size_t)lanes_of(cfg) * (cfg.n_slots ? cfg.n_slots : 1) <= c.n / 2, MMFHE_E_SHAPE,
                      "lanes * n_slots must not exceed N/2");
    }
    const bool k3_chain = chain == "k3_doppler_dft" || chain == "gesture" || chain == "gesture_frame" ||
                          chain == "gesture_features";
    if (k3_chain)  // the 2D-1 block-diagonal offsets alias when a period holds a single block
        MMFHE_REQUIRE(cfg.D >= 1 && cfg.n_slots % cfg.D == 0 && cfg.n_slots >= 2 * cfg.D, MMFHE_E_SHAPE,
                      "K3 needs n_slots a multiple of D and at least 2D");
    if (chain == "vitals_v1") n_out = 2;
    if (chain == "vitals_v2") {
        n_out = 0;
        for (uint32_t b = 0; b < cfg.n_bands; ++b) n_out += cfg.vp_plus ? 2 : cfg.n_bins[b];
    }
    return std::vector<uint32_t>(n_out, out);
}

std::vector<DCt> run_chain(Ctx &c, const std::string &chain, const mmfhe_chain_cfg &cfg, const mmfhe_ct *in,
                           size_t n_in)
{
    MMFHE_REQUIRE(in && n_in, MMFHE_E_SHAPE, "no inputs");
    chain_plan(c, chain, cfg, in[0].level, n_in);
    Runner r(c, cfg);
    std::vector<DCt> out;
    if (chain == "k1_energy") {
        // sessions batched: frame t of every session forms one batch (one launch per op)
        // one import of every session's frames (session-major), then the per-session sum of
        // squares reads frame t of every session at item stride 2F: the same op sequence as
        // k1_energy_sessions on per-frame batches, without 2F separate imports
        const uint32_t F = cfg.F, S = (uint32_t)(n_in / (2 * (size_t)F));
        DCt all = import_batch(c, in, 0, 1, n_in);
        out.push_back(ev_relin_rescale(c, ev_square_sum_items(c, all, 2 * F, S)));
    } else if (chain == "vitals_v1") {
        DCt re = import_batch(c, in, 0, 2, n_in / 2);
        DCt im = import_batch(c, in, 1, 2, n_in / 2);
        auto nd = r.k2_soft_attention(r.k1_energy(re, im));
        out.push_back(std::move(nd.first));
        out.push_back(std::move(nd.second));
    } else if (chain == "vitals_v2") {
        out = r.vitals_v2(in, n_in);
    } else if (cplx_chain(chain, cfg) && (chain == "k3_doppler_dft" || chain == "gesture_frame")) {
        // complex slots: one z per frame (group); per batch one output batch (d, or the features)
        const uint32_t F = (uint32_t)n_in, fb = r.frame_batch(F);
        for (uint32_t t0 = 0; t0 < F; t0 += fb) {
            DCt z = import_batch(c, in, t0, 1, std::min(fb, F - t0));
            out.push_back(chain == "k3_doppler_dft" ? r.k3_doppler_dft_c(z) : r.gesture_frame_c(z));
        }
    } else if (chain == "k3_doppler_dft" || chain == "gesture_frame") {
        // frames in batches of cfg.frame_batch; k3 outputs per batch: its d_re items, then its d_im items
        const uint32_t F = (uint32_t)(n_in / 2), fb = r.frame_batch(F);
        for (uint32_t t0 = 0; t0 < F; t0 += fb) {
            const uint32_t cnt = std::min(fb, F - t0);
            DCt vre = import_batch(c, in, 2 * (size_t)t0, 2, cnt);
            DCt vim = import_batch(c, in, 2 * (size_t)t0 + 1, 2, cnt);
            if (chain == "k3_doppler_dft") {
                auto d = r.k3_doppler_dft(vre, vim);
                out.push_back(std::move(d.first));
                out.push_back(std::move(d.second));
            } else {
                out.push_back(r.gesture_frame(vre, vim));
            }
        }
    } else if (chain == "gesture_fc" || chain == "fc_forward") {
        // sessions batched: every op of the head runs once over all sessions' features (the same
        // plaintext diagonals and keys for every item), item s = session s's logits
        DCt x = import_batch(c, in, 0, 1, n_in);
        out.push_back(r.gesture_fc(x));
    } else if (chain == "gesture") {
        out.push_back(r.gesture(in, n_in));
    } else if (chain == "gesture_features") {
        out.push_back(cfg.sessions > 1 ? r.gesture_features_sessions(in, n_in, cfg.sessions)
                                       : r.gesture_features(in, n_in));
    } else if (chain == "k2_soft_attention") {
        auto nd = r.k2_soft_attention(import_batch(c, in, 0, 1, 1));
        out.push_back(std::move(nd.first));
        out.push_back(std::move(nd.second));
    } else if (chain == "k2_doppler_soft_power" || chain == "k6_notch") {
        DCt x = import_batch(c, in, 0, 1, n_in);
        out.push_back(chain == "k6_notch" ? r.k6_notch(x) : r.k2_doppler_soft_power(x));
    } else if (chain == "k4_soft_iq") {
        auto iq = r.k4_all_frames(in, n_in);
        out.push_back(std::move(iq.first));
        out.push_back(std::move(iq.second));
    } else if (chain == "k5_fir") {
        DCt x = import_batch(c, in, 0, 1, n_in);
        for (uint32_t b = 0; b < cfg.n_bands; ++b) out.push_back(r.k5_fir(x, r.band_taps(b)));
    } else if (chain == "k5_fir_rot") {
        // every input is one slot-packed sequence; outputs band-major, sequence by sequence
        for (uint32_t b = 0; b < cfg.n_bands; ++b)
            for (size_t s = 0; s < n_in; ++s) out.push_back(r.k5_fir_rot(import_batch(c, in, s, 1, 1), r.band_taps(b)));
    } else if (chain == "k7_taylor_phase") {
        DCt If = import_batch(c, in, 0, 2, n_in / 2);
        DCt Qf = import_batch(c, in, 1, 2, n_in / 2);
        out.push_back(r.k7_taylor_phase(If, Qf));
    }
    return out;
}

}  // namespace mmfhe
