// context.cu -- ctx creation: parameter validation, NTT twiddle tables,
// base-conversion / rescale constants, device memory pool.
#include <algorithm>
#include <cstdio>
#include <set>

#include "context.h"

namespace mmfhe {

namespace host {
bool is_prime(uint64_t n)
{
    if (n < 2) return false;
    static const uint64_t small[] = {2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37};
    for (uint64_t p : small)
        if (n % p == 0) return n == p;
    uint64_t d = n - 1;
    int r = 0;
    while (!(d & 1)) {
        d >>= 1;
        ++r;
    }
    for (uint64_t a : small) {
        uint64_t x = pow(a, d, n);
        if (x == 1 || x == n - 1) continue;
        bool comp = true;
        for (int i = 1; i < r; ++i) {
            x = mul(x, x, n);
            if (x == n - 1) {
                comp = false;
                break;
            }
        }
        if (comp) return false;
    }
    return true;
}

// The minimal primitive 2N-th root of unity mod q.
static uint64_t min_psi(uint64_t q, uint32_t n)
{
    uint64_t two_n = 2ull * n, psi0 = 0;
    for (uint64_t x = 3; x < (1u << 20); x += 2) {
        uint64_t c = pow(x, (q - 1) / two_n, q);
        if (pow(c, n, q) == q - 1) {
            psi0 = c;
            break;
        }
    }
    MMFHE_REQUIRE(psi0 != 0, MMFHE_E_PARAMS, "no primitive 2N-th root");
    uint64_t best = psi0, sq = mul(psi0, psi0, q), cur = psi0;
    for (uint64_t k = 1; k < n; ++k) {  // odd powers psi0^(2k+1)
        cur = mul(cur, sq, q);
        if (cur < best) best = cur;
    }
    return best;
}
}  // namespace host

namespace {
thread_local cudaMemPool_t g_pool = nullptr;
}
PoolScope::PoolScope(cudaMemPool_t p) : saved_(g_pool) { g_pool = p; }
PoolScope::~PoolScope() { g_pool = saved_; }
cudaMemPool_t PoolScope::current() { return g_pool; }

PoolHolder::~PoolHolder()
{
    if (pool) cudaMemPoolDestroy(pool);
}

DBuf::DBuf(size_t words, cudaStream_t s) : n_(words), s_(s)
{
    if (!words) return;
    if (g_pool)
        CUDA_CHECK(cudaMallocFromPoolAsync((void **)&p_, words * sizeof(uint64_t), g_pool, s));
    else
        CUDA_CHECK(cudaMallocAsync((void **)&p_, words * sizeof(uint64_t), s));
}
DBuf::~DBuf() { release(); }
void DBuf::release()
{
    if (p_) cudaFreeAsync(p_, s_);
    p_ = nullptr;
    n_ = 0;
}

std::string plain_key(const std::string &name, uint32_t level) { return name + "@" + std::to_string(level); }

void Ctx::rec(const char *op, uint32_t level, const std::string &arg)
{
    if (!trace_on) return;
    std::string s = std::string(op) + " " + std::to_string(level);
    if (!arg.empty()) s += " " + arg;
    trace.push_back(std::move(s));
}

std::vector<uint32_t> Ctx::ext_basis(uint32_t level) const
{
    std::vector<uint32_t> v;
    for (uint32_t i = 0; i <= level; ++i) v.push_back(i);
    for (uint32_t k = 0; k < K; ++k) v.push_back(L + 1 + k);
    return v;
}

std::vector<uint32_t> Ctx::q_basis(uint32_t level) const
{
    std::vector<uint32_t> v;
    for (uint32_t i = 0; i <= level; ++i) v.push_back(i);
    return v;
}

DPlain *Ctx::find_plain(const std::string &name, uint32_t level) const
{
    auto it = plains.find(plain_key(name, level));
    return it == plains.end() ? nullptr : it->second.get();
}

void Ctx::sync() { CUDA_CHECK(cudaStreamSynchronize(stream)); }

cudaEvent_t Ctx::next_event()
{
    if (ev_used == ev_pool.size()) {
        cudaEvent_t e;
        CUDA_CHECK(cudaEventCreate(&e));
        ev_pool.push_back(e);
    }
    return ev_pool[ev_used++];
}

std::string Ctx::profile_report()
{
    sync();
    struct Agg {
        uint64_t count = 0;
        double ms = 0, bytes = 0, ops = 0;
    };
    std::map<std::string, Agg> agg;
    for (auto &r : prof) {
        float ms = 0;
        CUDA_CHECK(cudaEventElapsedTime(&ms, r.a, r.b));
        Agg &g = agg[r.name];
        g.count++;
        g.ms += ms;
        g.bytes += r.bytes;
        g.ops += r.ops;
    }
    prof.clear();
    ev_used = 0;
    std::string out;
    char line[256];
    for (auto &kv : agg) {
        snprintf(line, sizeof(line), "%s %llu %.6f %.0f %.0f\n", kv.first.c_str(), (unsigned long long)kv.second.count,
                 kv.second.ms, kv.second.bytes, kv.second.ops);
        out += line;
    }
    return out;
}

Ctx::Ctx(const mmfhe_params &p, int dev, cudaStream_t s) : device(dev), stream(s)
{
    MMFHE_REQUIRE(p.log_n >= 4 && p.log_n <= 16, MMFHE_E_PARAMS, "log_n must be in [4, 16]");
    MMFHE_REQUIRE(p.n_q >= 1 && p.q != nullptr, MMFHE_E_PARAMS, "need at least one q prime");
    MMFHE_REQUIRE(p.n_p >= 1 && p.p != nullptr, MMFHE_E_PARAMS, "need at least one special prime");
    MMFHE_REQUIRE(p.alpha >= 1 && p.alpha <= 15, MMFHE_E_PARAMS, "alpha must be in [1, 15]");
    MMFHE_REQUIRE(p.n_q + p.n_p <= 64, MMFHE_E_PARAMS, "at most 64 primes");
    log_n = p.log_n;
    n = 1u << log_n;
    L = p.n_q - 1;
    K = p.n_p;
    alpha = p.alpha;
    scale_bits = p.scale_bits;
    for (uint32_t i = 0; i < p.n_q; ++i) primes.push_back(p.q[i]);
    for (uint32_t i = 0; i < p.n_p; ++i) primes.push_back(p.p[i]);
    std::set<uint64_t> seen;
    for (uint64_t q : primes) {
        MMFHE_REQUIRE(q < (1ull << 60) && q > 2, MMFHE_E_PARAMS, "primes must be < 2^60");
        MMFHE_REQUIRE((q - 1) % (2ull * n) == 0, MMFHE_E_PARAMS, "prime != 1 mod 2N");
        MMFHE_REQUIRE(host::is_prime(q), MMFHE_E_PARAMS, "modulus is not prime");
        MMFHE_REQUIRE(seen.insert(q).second, MMFHE_E_PARAMS, "duplicate prime");
    }
    CUDA_CHECK(cudaSetDevice(device));
    // the ctx's own stream-ordered pool (steady-state steps never touch the OS allocator:
    // release threshold = max); destroyed with the ctx, the device's default pool untouched
    cudaMemPoolProps props{};
    props.allocType = cudaMemAllocationTypePinned;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = device;
    CUDA_CHECK(cudaMemPoolCreate(&mem.pool, &props));
    uint64_t thr = UINT64_MAX;
    CUDA_CHECK(cudaMemPoolSetAttribute(mem.pool, cudaMemPoolAttrReleaseThreshold, &thr));
    PoolScope scope(mem.pool);
    build_tables();
}

Ctx::~Ctx()
{
    cudaStreamSynchronize(stream);
    drop_graphs();
    if (copy_stream) cudaStreamSynchronize(copy_stream);
    for (auto &kv : staging)
        for (auto &sl : kv.second.slot) {
            if (sl.ready) cudaEventDestroy(sl.ready);
            if (sl.free) cudaEventDestroy(sl.free);
        }
    staging.clear();
    if (copy_stream) cudaStreamDestroy(copy_stream);
    if (cap_stream) cudaStreamDestroy(cap_stream);
    for (cudaEvent_t e : ev_pool) cudaEventDestroy(e);
}

void Ctx::drop_graphs()
{
    if (graphs.empty()) return;
    cudaStreamSynchronize(stream);
    for (auto &kv : graphs)
        if (kv.second.exec) cudaGraphExecDestroy(kv.second.exec);
    graphs.clear();
}

namespace {
struct Blob {
    std::vector<uint8_t> bytes;
    template <class T>
    size_t push(const std::vector<T> &v)
    {
        size_t off = (bytes.size() + 15) & ~size_t(15);
        bytes.resize(off + v.size() * sizeof(T));
        if (!v.empty()) std::memcpy(bytes.data() + off, v.data(), v.size() * sizeof(T));
        return off;
    }
};
}  // namespace

void Ctx::build_tables()
{
    const uint32_t np = (uint32_t)primes.size();
    std::vector<uint64_t> hq(np), hqinv(np), hr2(np);
    std::vector<TwPair> fwd((size_t)np * n), inv((size_t)np * n), ninv(np), ninvw(np);
    std::vector<uint32_t> br(n);
    for (uint32_t k = 0; k < n; ++k) {
        uint32_t r = 0;
        for (uint32_t b = 0; b < log_n; ++b) r |= ((k >> b) & 1u) << (log_n - 1 - b);
        br[k] = r;
    }
    std::vector<uint64_t> pw(n), ipw(n);
    for (uint32_t pi = 0; pi < np; ++pi) {
        uint64_t q = primes[pi];
        hq[pi] = q;
        hqinv[pi] = host::qinv_neg(q);
        uint64_t r1 = host::to_mont(1, q);  // 2^64 mod q
        hr2[pi] = host::mul(r1, r1, q);     // 2^128 mod q
        uint64_t psi = host::min_psi(q, n);
        uint64_t ipsi = host::inv(psi, q);
        pw[0] = ipw[0] = 1;
        for (uint32_t i = 1; i < n; ++i) {
            pw[i] = host::mul(pw[i - 1], psi, q);
            ipw[i] = host::mul(ipw[i - 1], ipsi, q);
        }
        for (uint32_t k = 0; k < n; ++k) {
            uint64_t w = pw[br[k]], wi = ipw[br[k]];
            fwd[(size_t)pi * n + k] = {w, host::shoup(w, q)};
            inv[(size_t)pi * n + k] = {wi, host::shoup(wi, q)};
        }
        uint64_t ni = host::inv(n, q);
        ninv[pi] = {ni, host::shoup(ni, q)};
        const uint64_t niw = host::mul(ni, inv[(size_t)pi * n + 1].w, q);
        ninvw[pi] = {niw, host::shoup(niw, q)};
    }
    auto up = [&](DBuf &b, const void *src, size_t bytes) {
        b = DBuf((bytes + 7) / 8, stream);
        CUDA_CHECK(cudaMemcpyAsync(b.get(), src, bytes, cudaMemcpyHostToDevice, stream));
    };
    up(tab_q, hq.data(), np * 8);
    up(tab_qinv, hqinv.data(), np * 8);
    up(tab_r2, hr2.data(), np * 8);
    up(tab_tw_fwd, fwd.data(), fwd.size() * sizeof(TwPair));
    up(tab_tw_inv, inv.data(), inv.size() * sizeof(TwPair));
    up(tab_ninv, ninv.data(), ninv.size() * sizeof(TwPair));
    up(tab_ninvw, ninvw.data(), ninvw.size() * sizeof(TwPair));
    kt.q = tab_q.get();
    kt.qinv_neg = tab_qinv.get();
    kt.r2 = tab_r2.get();
    kt.tw_fwd = (const TwPair *)tab_tw_fwd.get();
    kt.tw_inv = (const TwPair *)tab_tw_inv.get();
    kt.n_inv = (const TwPair *)tab_ninv.get();
    kt.n_inv_w = (const TwPair *)tab_ninvw.get();
    kt.log_n = log_n;
    kt.n = n;

    // ---- base conversion and rescale constants
    Blob blob;
    modup.assign(L + 1, {});
    for (uint32_t l = 0; l <= L; ++l) {
        std::vector<uint32_t> basis = ext_basis(l);
        for (uint32_t j = 0; j < dnum(l); ++j) {
            ModUpPlan pl;
            pl.lo = j * alpha;
            pl.hi = std::min(pl.lo + alpha, l + 1);
            std::vector<TwPair> hat_inv;
            std::vector<uint32_t> tgt;
            for (uint32_t r = 0; r < basis.size(); ++r)
                if (r < pl.lo || r >= pl.hi) tgt.push_back(r);
            pl.n_tgt = (uint32_t)tgt.size();
            std::vector<uint64_t> hat((size_t)(pl.hi - pl.lo) * pl.n_tgt);
            for (uint32_t i = pl.lo; i < pl.hi; ++i) {
                uint64_t qi = primes[i];
                uint64_t prod = 1;  // Qhat_i mod q_i
                for (uint32_t k = pl.lo; k < pl.hi; ++k)
                    if (k != i) prod = host::mul(prod, primes[k] % qi, qi);
                uint64_t hi_ = host::inv(prod, qi);
                hat_inv.push_back({hi_, host::shoup(hi_, qi)});
                for (uint32_t ti = 0; ti < pl.n_tgt; ++ti) {
                    uint64_t t = primes[basis[tgt[ti]]];
                    uint64_t pr = 1;
                    for (uint32_t k = pl.lo; k < pl.hi; ++k)
                        if (k != i) pr = host::mul(pr, primes[k] % t, t);
                    hat[(size_t)(i - pl.lo) * pl.n_tgt + ti] = host::to_mont(pr, t);
                }
            }
            pl.off_hat_inv = blob.push(hat_inv);
            pl.off_hat = blob.push(hat);
            pl.off_tgt = blob.push(tgt);
            modup[l].push_back(pl);
        }
    }
    {
        std::vector<TwPair> phinv(K);
        std::vector<uint64_t> phat((size_t)K * (L + 1));
        std::vector<TwPair> pinv(L + 1);
        for (uint32_t k = 0; k < K; ++k) {
            uint64_t pk = primes[L + 1 + k];
            uint64_t prod = 1;
            for (uint32_t m = 0; m < K; ++m)
                if (m != k) prod = host::mul(prod, primes[L + 1 + m] % pk, pk);
            uint64_t v = host::inv(prod, pk);
            phinv[k] = {v, host::shoup(v, pk)};
            for (uint32_t i = 0; i <= L; ++i) {
                uint64_t qi = primes[i];
                uint64_t pr = 1;
                for (uint32_t m = 0; m < K; ++m)
                    if (m != k) pr = host::mul(pr, primes[L + 1 + m] % qi, qi);
                phat[(size_t)k * (L + 1) + i] = host::to_mont(pr, qi);
            }
        }
        std::vector<TwPair> pmod(L + 1);
        for (uint32_t i = 0; i <= L; ++i) {
            uint64_t qi = primes[i];
            uint64_t P = 1;
            for (uint32_t m = 0; m < K; ++m) P = host::mul(P, primes[L + 1 + m] % qi, qi);
            uint64_t v = host::inv(P, qi);
            pinv[i] = {v, host::shoup(v, qi)};
            pmod[i] = {P, host::shoup(P, qi)};
        }
        // R31: ModDown and rescale as one division by M = P q_l (row l = the level being left)
        std::vector<TwPair> mhinv((size_t)(L + 1) * (K + 1), TwPair{0, 0}), mminv((size_t)(L + 1) * (L + 1), TwPair{0, 0});
        std::vector<uint64_t> mhat((size_t)(L + 1) * (K + 1) * (L + 1), 0);
        for (uint32_t l = 1; l <= L; ++l) {
            std::vector<uint64_t> src;
            for (uint32_t k = 0; k < K; ++k) src.push_back(primes[L + 1 + k]);
            src.push_back(primes[l]);
            for (uint32_t bi = 0; bi <= K; ++bi) {
                const uint64_t b = src[bi];
                uint64_t prod = 1;  // (M / b) mod b
                for (uint32_t m = 0; m <= K; ++m)
                    if (m != bi) prod = host::mul(prod, src[m] % b, b);
                const uint64_t v = host::inv(prod, b);
                mhinv[(size_t)l * (K + 1) + bi] = {v, host::shoup(v, b)};
                for (uint32_t i = 0; i < l; ++i) {
                    const uint64_t qi = primes[i];
                    uint64_t pr = 1;
                    for (uint32_t m = 0; m <= K; ++m)
                        if (m != bi) pr = host::mul(pr, src[m] % qi, qi);
                    mhat[((size_t)l * (K + 1) + bi) * (L + 1) + i] = host::to_mont(pr, qi);
                }
            }
            for (uint32_t i = 0; i < l; ++i) {
                const uint64_t qi = primes[i];
                uint64_t M = primes[l] % qi;
                for (uint32_t m = 0; m < K; ++m) M = host::mul(M, primes[L + 1 + m] % qi, qi);
                const uint64_t v = host::inv(M, qi);
                mminv[(size_t)l * (L + 1) + i] = {v, host::shoup(v, qi)};
            }
        }
        off_mr_hinv = blob.push(mhinv);
        off_mr_hat = blob.push(mhat);
        off_mr_minv = blob.push(mminv);
        off_pd_hat_inv = blob.push(phinv);
        off_pd_hat = blob.push(phat);
        off_pd_pinv = blob.push(pinv);
        off_pd_pmod = blob.push(pmod);
    }
    {
        std::vector<TwPair> rs((size_t)(L + 1) * (L + 1), TwPair{0, 0});
        std::vector<uint64_t> rh((size_t)(L + 1) * (L + 1), 0);
        for (uint32_t l = 1; l <= L; ++l) {
            uint64_t ql = primes[l];
            for (uint32_t i = 0; i < l; ++i) {
                uint64_t qi = primes[i];
                uint64_t v = host::inv(ql % qi, qi);
                rs[(size_t)l * (L + 1) + i] = {v, host::shoup(v, qi)};
                rh[(size_t)l * (L + 1) + i] = (ql >> 1) % qi;
            }
        }
        off_rs = blob.push(rs);
        off_rs_h = blob.push(rh);
        std::vector<uint64_t> recip(np);
        for (uint32_t i = 0; i < np; ++i) recip[i] = host::shoup(1, primes[i]);
        off_recip = blob.push(recip);
    }
    tab_bconv = DBuf((blob.bytes.size() + 7) / 8, stream);
    CUDA_CHECK(cudaMemcpyAsync(tab_bconv.get(), blob.bytes.data(), blob.bytes.size(), cudaMemcpyHostToDevice,
                               stream));
    CUDA_CHECK(cudaStreamSynchronize(stream));
    kt.recip = (const uint64_t *)bconv_ptr(off_recip);
}

}  // namespace mmfhe
