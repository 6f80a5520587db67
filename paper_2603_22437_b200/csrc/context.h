// context.h -- the mmfhe_ctx: parameters, device tables, key and plaintext
// stores, stream, device memory pool, op trace.
#pragma once
#include <map>
#include <unordered_map>
#include <memory>
#include <string>
#include <vector>

#include "common.h"

namespace mmfhe {

// The memory pool DBufs allocate from on this thread: set for the duration of every C-ABI
// call (and the ctx constructor) to the ctx's own pool, so each ctx's allocations are its
// own, reported per ctx and released with it (never the device's default pool).
struct PoolScope {
    explicit PoolScope(cudaMemPool_t p);
    ~PoolScope();
    PoolScope(const PoolScope &) = delete;
    PoolScope &operator=(const PoolScope &) = delete;
    static cudaMemPool_t current();

  private:
    cudaMemPool_t saved_;
};

// Stream-ordered device buffer from the current ctx's memory pool (cudaMallocFromPoolAsync).
class DBuf {
  public:
    DBuf() = default;
    DBuf(size_t words, cudaStream_t s);
    ~DBuf();
    DBuf(const DBuf &) = delete;
    DBuf &operator=(const DBuf &) = delete;
    DBuf(DBuf &&o) noexcept { swap(o); }
    DBuf &operator=(DBuf &&o) noexcept
    {
        if (this != &o) {
            release();
            swap(o);
        }
        return *this;
    }
    uint64_t *get() const { return p_; }
    size_t words() const { return n_; }
    void release();

  private:
    void swap(DBuf &o)
    {
        std::swap(p_, o.p_);
        std::swap(n_, o.n_);
        std::swap(s_, o.s_);
    }
    uint64_t *p_ = nullptr;
    size_t n_ = 0;
    cudaStream_t s_ = nullptr;
};

// A batch of `batch` ciphertexts (npolys = 2, or 3 after a tensor) in the
// library's NTT form, laid out [batch][npolys][level+1][N] contiguously.
struct DCt {
    DBuf buf;
    uint64_t *ext = nullptr;  // non-owning view (caller buffer / slice) when set
    uint32_t level = 0;
    uint32_t npolys = 2;
    uint32_t n_slots = 0;
    uint32_t batch = 1;
    uint32_t n = 0;  // ring dimension
    // PQ ciphertexts (double-hoisted BSGS): pk = K extra limbs p_0..p_{K-1} per polynomial.
    // Item layout: [npolys][level+1][N] (the Q part, as a plain ciphertext), then
    // [npolys][pk][N] (the P part).
    uint32_t pk = 0;
    double scale = 1.0;
    uint64_t *data() const { return ext ? ext : buf.get(); }
    size_t poly_words() const { return (size_t)(level + 1) * n; }
    size_t item_words() const { return (size_t)npolys * (level + 1 + pk) * n; }
    uint64_t *item(uint32_t b) const { return data() + (size_t)b * item_words(); }
    uint64_t *poly(uint32_t i, uint32_t b = 0) const { return item(b) + (size_t)i * poly_words(); }
    uint64_t *ppoly(uint32_t i, uint32_t b = 0) const
    {
        return item(b) + (size_t)npolys * poly_words() + (size_t)i * pk * n;
    }
    uint32_t rows() const { return batch * npolys * (level + 1 + pk); }
};

struct DKey {
    DBuf buf;  // [dnum_L][2][L+1+K][N], NTT form, Montgomery form
};

struct DPlain {
    DBuf buf;  // [level+1 (+pk)][N], NTT form, Montgomery form (x 2^64 mod q)
    uint32_t level = 0;
    uint32_t pk = 0;  // K: also reduced mod p_0..p_{K-1} (rows level+1..), double hoisting
    double scale = 1.0;
};

// Base-conversion constants for one (level, digit) ModUp.
struct ModUpPlan {
    uint32_t lo, hi;           // source limbs [lo, hi)
    uint32_t n_tgt;            // targets = (l+1+K) - (hi-lo)
    size_t off_hat_inv;        // TwPair [hi-lo]       [Qhat_i^{-1}]_{q_i}
    size_t off_hat;            // uint64 [hi-lo][n_tgt] [Qhat_i]_t * 2^64 mod t
    size_t off_tgt;            // uint32 [n_tgt] target row index in the l+1+K basis
};

// Owns the ctx's device memory pool; declared first in Ctx so that it is destroyed after
// every DBuf member has been released (cudaMemPoolDestroy then frees the pool's memory).
struct PoolHolder {
    cudaMemPool_t pool = nullptr;
    ~PoolHolder();
};

class Ctx {
  public:
    Ctx(const mmfhe_params &p, int device, cudaStream_t stream);
    ~Ctx();

    PoolHolder mem;  // first member: destroyed last

    // parameters
    uint32_t log_n, n, L, K, alpha, scale_bits;
    std::vector<uint64_t> primes;  // q_0..q_L, p_0..p_{K-1}
    int device;
    cudaStream_t stream;
    uint64_t launches = 0;
    std::string last_error;

    // device tables
    KTables kt{};
    DBuf tab_q, tab_qinv, tab_r2, tab_tw_fwd, tab_tw_inv, tab_ninv, tab_ninvw;
    // base conversion / rescale constant blob (device) and host plans
    DBuf tab_bconv;
    std::vector<std::vector<ModUpPlan>> modup;  // [level][digit]
    size_t off_pd_hat_inv = 0;   // TwPair[K]            [Phat_k^{-1}]_{p_k}
    size_t off_pd_hat = 0;       // uint64[K][L+1]       [Phat_k]_{q_i} * 2^64 mod q_i
    size_t off_pd_pinv = 0;      // TwPair[L+1]          [P^{-1}]_{q_i}
    size_t off_pd_pmod = 0;      // TwPair[L+1]          [P]_{q_i} (double hoisting's P lift)
    size_t off_mr_hinv = 0;      // TwPair[L+1][K+1]     R31 (ModDown + rescale, M = P q_l, row l): [(M/b)^{-1}]_b,
                                 //                      b = p_0..p_{K-1}, q_l
    size_t off_mr_hat = 0;       // uint64[L+1][K+1][L+1] [M/b]_{q_i} * 2^64 mod q_i
    size_t off_mr_minv = 0;      // TwPair[L+1][L+1]     [M^{-1}]_{q_i}
    size_t off_rs = 0;           // TwPair[L+1][L+1]     [q_l^{-1}]_{q_i} (row l)
    size_t off_rs_h = 0;         // uint64[L+1][L+1]     floor(q_l/2) mod q_i (row l)
    size_t off_recip = 0;        // uint64[np]           floor(2^64 / prime)

    // stores
    std::unique_ptr<DKey> rlk;
    std::map<int32_t, std::unique_ptr<DKey>> gk;
    std::map<std::string, std::unique_ptr<DPlain>> plains;  // key "name@level"
    std::map<std::string, std::vector<double>> scalars;
    std::map<std::string, DBuf> const_cache;  // encoded scalar tables by "name@level"
    // mmfhe_prepare_chain: encode absent public operands from the paper's formulas on first use
    bool auto_encode = false;
    std::vector<std::vector<double>> fc_w, fc_b;  // FC layer weights (row-major) and biases

    // per-kernel CUDA-event profile (bench roofline): events around each launch
    struct ProfRec {
        const char *name;
        cudaEvent_t a, b;
        double bytes, ops;  // algorithmic bytes and butterflies (NTT) of the launch
    };
    bool prof_on = false;
    std::vector<ProfRec> prof;
    std::vector<cudaEvent_t> ev_pool;
    size_t ev_used = 0;
    cudaEvent_t next_event();
    std::string profile_report();  // "name count total_ms bytes" lines; resets

    // CUDA-graph replay of repeated device-resident chain calls (mmfhe_eval_chain): the
    // second identical call is captured, later ones replay the graph, so the host-side
    // op dispatch (hundreds of launches, allocations, plan lookups) leaves the step.
    // Any operand-store change bumps state_gen, which is part of the key.
    struct ChainGraph {
        cudaGraphExec_t exec = nullptr;
        uint64_t launches = 0;           // kernel launches inside the graph
        std::vector<mmfhe_ct> out_meta;  // output level / scale / n_slots / n_polys
        int seen = 0;                    // < 0: capture failed, never retry
    };
    bool graphs_on = true;
    uint64_t state_gen = 0, graph_replays = 0;
    std::unordered_map<std::string, ChainGraph> graphs;
    cudaStream_t cap_stream = nullptr;
    void drop_graphs();

    // mmfhe_eval_chain_async: two device staging slots per (chain, shape) so that the
    // upload of call i+1 (copy_stream) overlaps the compute of call i (stream)
    struct StageSlot {
        DBuf in, out;
        cudaEvent_t ready = nullptr, free = nullptr;
    };
    struct Staging {
        StageSlot slot[2];
        int next = 0;
    };
    std::unordered_map<std::string, Staging> staging;
    cudaStream_t copy_stream = nullptr;

    // trace (Theorem P:999-1006)
    bool trace_on = true;
    std::vector<std::string> trace;
    void rec(const char *op, uint32_t level, const std::string &arg = "");

    // helpers
    uint32_t dnum(uint32_t level) const { return (level + alpha) / alpha; }
    size_t key_words() const { return (size_t)dnum(L) * 2 * (L + 1 + K) * n; }
    uint64_t prime(uint32_t idx) const { return primes[idx]; }
    // basis rows of the extended modulus Q_l u P
    std::vector<uint32_t> ext_basis(uint32_t level) const;
    std::vector<uint32_t> q_basis(uint32_t level) const;
    const void *bconv_ptr(size_t off) const { return (const char *)tab_bconv.get() + off; }
    DPlain *find_plain(const std::string &name, uint32_t level) const;
    void sync();

  private:
    void build_tables();
};

std::string plain_key(const std::string &name, uint32_t level);

// Records CUDA events around one kernel launch when the ctx profiler is on.
class ProfScope {
  public:
    ProfScope(Ctx &c, const char *name, double bytes, double ops = 0) : c_(c), name_(name), bytes_(bytes), ops_(ops)
    {
        if (c_.prof_on) {
            a_ = c_.next_event();
            cudaEventRecord(a_, c_.stream);
        }
    }
    ~ProfScope()
    {
        if (c_.prof_on) {
            cudaEvent_t b = c_.next_event();
            cudaEventRecord(b, c_.stream);
            c_.prof.push_back({name_, a_, b, bytes_, ops_});
        }
    }

  private:
    Ctx &c_;
    const char *name_;
    double bytes_, ops_;
    cudaEvent_t a_ = nullptr;
};

// ------------------------------------------------------------------ kernels (launchers)
// src: optional fused source of the col pass (ModUp of single-limb digits), see ColSrc
// epi: optional fused epilogue of the row pass (ModDown / rescale final step), see RowEpi;
// with epi the transform itself is not stored (d is scratch for the col pass)
void ntt_forward(Ctx &c, uint64_t *d, uint32_t rows, const PrimeMap &pm, const ColSrc *src = nullptr,
                 const RowEpi *epi = nullptr);
// src: optional out-of-place / automorphism-permuted source of the row pass, see InvSrc
void ntt_inverse(Ctx &c, uint64_t *d, uint32_t rows, const PrimeMap &pm, const InvSrc *src = nullptr);

}  // namespace mmfhe
