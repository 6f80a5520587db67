// ntt.cu -- batched negacyclic NTT / INTT across RNS limbs.
//
// Forward: Cooley-Tukey, natural order in, bit-reversed order out, psi-twist
// merged into the twiddles (tw_fwd[m + i] = psi^{bitrev(m+i)}): stage l (m = 2^l)
// pairs j, j + N/2^{l+1} with twiddle index m + (j >> (log N - l)).
// Inverse: Gentleman-Sande with psi^{-bitrev}, bit-reversed in, natural out,
// times N^{-1} (folded into the last stage).  Shoup products throughout (q < 2^60).
//
// B200 mapping.  A limb of N = 2^16 words (512 KiB) exceeds one SM's shared
// memory, so the transform is two passes over HBM (logN = L1 + L2):
//   col pass -- stages 0..L1-1 on 2^L2 strided columns of 2^L1 words; a warp
//               spans G consecutive columns (G*8-byte sector-aligned runs);
//   row pass -- stages L1..logN-1 on contiguous blocks of 2^L2 words.  Its first and
//               last rounds read / write HBM directly: in those rounds a thread's
//               registers cover runs of 2..8 consecutive words, moved with 16- or
//               32-byte vector accesses that are contiguous across lanes (measured
//               12-20% faster than staging the tile through shared memory).
// Inside a pass each thread holds E = 2^ELOG = 8 words in registers (radix-8)
// and runs up to ELOG butterfly stages there per round; rounds exchange through
// double-buffered, XOR-swizzled shared memory (one __syncthreads per exchange,
// bank-conflict-free).  Forward rounds put the narrow round FIRST (top bits) and
// inverse rounds LAST, so that in every round a stage's twiddle depends only on
// register bits above it: each distinct twiddle is loaded once per stage (one
// 16-byte read-only load per twiddle pair).
//
// Index arithmetic.  The whole pass geometry (LOGS, the other pass's bits, groups
// per CTA) is compile-time.  Every local index k = kmap(t, e) is the OR of a thread
// part and a register part on disjoint bits, and the XOR swizzle is GF(2)-linear,
// so each shared/global/twiddle address is one per-round thread base plus (or XOR)
// a compile-time constant: the loads and stores carry immediate offsets and the
// issue slots go to the butterflies.
//
// Butterfly product: Shoup with a truncated quotient (shoup_lazy4, V' = V w mod q in
// [0, 4q)).  Lazy forward reduction: with q < 2^60 every word may grow to 16q < 2^64;
// a CT butterfly (U, V) -> (U + V', U - V' + 4q) grows the bound by 4q, so instead of a
// per-butterfly correction the forward transform corrects U >= 8q only at odd global
// stages >= 3 (fwd_corr), and the row pass fully reduces its output to [0, q) with one
// estimated-quotient step (reduce_est).  Inputs of ntt_forward must be < 2q, inputs of
// ntt_inverse < 4q.
// Every limb of every polynomial of a batch goes in one launch.
#include <algorithm>

#include "context.h"
#include "modarith.cuh"

namespace mmfhe {

namespace {

constexpr int kCtaThreads = 256;

// Butterfly product: Shoup with a truncated quotient (shoup_lazy4, results in [0, 4q)):
// 3 wide + 2 high 32-bit products instead of 6 wide ones; measured 5% above the exact-
// quotient butterfly in the register-resident microbenchmark and 2-4% in the passes.
constexpr int kLazyMul = 4;  // V' < 4q
__device__ __forceinline__ uint64_t bfly_mul(uint64_t a, uint64_t w, uint64_t wp, uint64_t q)
{
    return shoup_lazy4(a, w, wp, q);
}
// Forward: is U >= 8q corrected before the butterflies of global stage s?  From the input
// bound 2q every stage grows the bound by 4q (U + V', U - V' + 4q); U < 16q must hold
// before a correction and every word stays < 16q < 2^64: bounds 2, 6, 10, 14 | 12, 16 |
// 12, 16 ... -> correct at odd s >= 3.
__host__ __device__ constexpr bool fwd_corr(int s) { return s >= 3 && (s & 1); }

// min CTAs/SM for __launch_bounds__: 4 (<= 64 registers) fits every pass without spills
// and keeps 32 warps resident; 5 (<= 51 registers) spills
#ifndef MMFHE_NTT_MINCTAS
#define MMFHE_NTT_MINCTAS 4
#endif
#ifndef MMFHE_NTT_TWSTAGE
#define MMFHE_NTT_TWSTAGE 0
#endif
constexpr int kMinCtas = MMFHE_NTT_MINCTAS;
constexpr bool kTwStage = MMFHE_NTT_TWSTAGE != 0;  // load each stage's twiddles just before it

template <int LOGS, int OTHER, bool COL>
struct Geo {
    static constexpr int ELOG = LOGS < 3 ? LOGS : 3;
    static constexpr int S = 1 << LOGS, E = 1 << ELOG, LOGT = LOGS - ELOG, T = 1 << LOGT;
    // groups per CTA: as many as fit kCtaThreads threads (and exist)
    static constexpr int LOGG = (8 - LOGT) < OTHER ? (8 - LOGT) : OTHER;
    static constexpr int G = 1 << LOGG, THREADS = T * G;
    static constexpr int R = (LOGS + ELOG - 1) / ELOG;  // register rounds
    static constexpr int LBASE = COL ? 0 : OTHER;       // global stage of local stage 0
    static constexpr size_t SMEM = 2 * sizeof(uint64_t) * (size_t)G * S;
};

// Local index of register e of thread t in a round that owns bits [lo, lo+w):
// y = top w bits of e -> bits lo..lo+w-1; z = (t, low ELOG-w bits of e) fills
// the free bit positions [0, lo) and [lo+w, LOGS) in ascending order.
// kmap(t, e) == kmap(t, 0) | kmap(0, e), on disjoint bits.
__host__ __device__ constexpr int kmap(int elog, int lo, int w, int t, int e)
{
    const int y = e >> (elog - w);
    const int z = (t << (elog - w)) | (e & ((1 << (elog - w)) - 1));
    return (z & ((1 << lo) - 1)) | (y << lo) | ((z >> lo) << (lo + w));
}

// XOR swizzle of a shared-memory word index: low bit b ^= parity((x >> 4) & M_b).
// Masks found by exhaustive bank simulation of every round's lane pattern (both
// directions); identity where the plain layout is already conflict-free.  Only the
// low 4 bits change, and swz(x ^ y) == swz(x) ^ swz(y).
struct Masks {
    int m0, m1, m2, m3;
};
template <int LOGS, bool COL>
__host__ __device__ constexpr Masks swz_masks()
{
    return (!COL && LOGS == 8)   ? Masks{7, 11, 13, 6}
           : (!COL && LOGS == 7) ? Masks{3, 1, 7, 4}
           : (!COL && LOGS == 6) ? Masks{1, 2, 1, 1}
           : (COL && LOGS == 8)  ? Masks{49, 27, 49, 6}
                                 : Masks{0, 0, 0, 0};
}
__host__ __device__ constexpr int cparity(int x)
{
    x ^= x >> 16;
    x ^= x >> 8;
    x ^= x >> 4;
    x ^= x >> 2;
    x ^= x >> 1;
    return x & 1;
}
template <int LOGS, bool COL>
__host__ __device__ constexpr int swz_ct(int x)
{
    constexpr Masks m = swz_masks<LOGS, COL>();
    const int h = x >> 4;
    return x ^ (cparity(h & m.m0) | (cparity(h & m.m1) << 1) | (cparity(h & m.m2) << 2) | (cparity(h & m.m3) << 3));
}
template <int LOGS, bool COL>
__device__ __forceinline__ int swz_rt(int x)
{
    constexpr Masks m = swz_masks<LOGS, COL>();
    if (m.m0 == 0 && m.m1 == 0 && m.m2 == 0 && m.m3 == 0) return x;
    const int h = x >> 4;
    return x ^ ((__popc(h & m.m0) & 1) | ((__popc(h & m.m1) & 1) << 1) | ((__popc(h & m.m2) & 1) << 2) |
                ((__popc(h & m.m3) & 1) << 3));
}

// Shared-memory word index of local element k = kt | ke of group g:
//   col: swz(k*G + g),   row: g*S + swz(k).
// sbase() is the per-round thread part, soff() adds the register part: the swizzle
// touches only the low 4 bits, whose constant is XORed, and the high constant bits are
// disjoint from the base's, so they become an immediate offset.
template <class Gm, int LOGS, bool COL>
__device__ __forceinline__ int sbase(int kt, int g)
{
    return COL ? swz_rt<LOGS, COL>((kt << Gm::LOGG) | g) : ((g << LOGS) | swz_rt<LOGS, COL>(kt));
}
template <class Gm, int LOGS, bool COL>
__device__ __forceinline__ int soff(int sb, int ke)
{
    const int C = swz_ct<LOGS, COL>(COL ? (ke << Gm::LOGG) : ke);
    return (sb ^ (C & 15)) + (C & ~15);
}

__device__ __forceinline__ uint64_t csub64(uint64_t x, uint64_t m) { return x >= m ? x - m : x; }

// One twiddle pair in a single 16-byte read-only load (the twiddle tables are separate,
// 16-byte aligned allocations of 16-byte entries).
__device__ __forceinline__ TwPair ld_tw(const TwPair *p)
{
    const ulonglong2 x = __ldg(reinterpret_cast<const ulonglong2 *>(p));
    return TwPair{x.x, x.y};
}

// log2 of the run of consecutive local indices a thread's registers cover in a round:
// the largest r with kmap(0, e) == e for every e < 2^r (then kmap(t, e0 + i) = kmap(t, e0) + i
// for i < 2^r and e0 a multiple of 2^r, and the thread part is 2^r-word aligned).
__host__ __device__ constexpr int run_log(int elog, int lo, int w)
{
    int r = 0;
    while (r < elog) {
        bool ok = true;
        for (int e = 0; e < (2 << r); ++e) ok = ok && kmap(elog, lo, w, 0, e) == e;
        if (!ok) break;
        ++r;
    }
    return r;
}

// Vectorised global I/O of 2^RL consecutive words (16 B / 32 B / 2 x 32 B per thread).
template <int RL>
__device__ __forceinline__ void ld_run(const uint64_t *p, uint64_t *v)
{
    if constexpr (RL == 0) {
        v[0] = p[0];
    } else if constexpr (RL == 1) {
        asm volatile("ld.global.v2.u64 {%0, %1}, [%2];" : "=l"(v[0]), "=l"(v[1]) : "l"(p));
    } else {
#pragma unroll
        for (int i = 0; i < (1 << RL); i += 4)
            asm volatile("ld.global.v4.u64 {%0, %1, %2, %3}, [%4];"
                         : "=l"(v[i]), "=l"(v[i + 1]), "=l"(v[i + 2]), "=l"(v[i + 3])
                         : "l"(p + i));
    }
}
template <int RL>
__device__ __forceinline__ void st_run(uint64_t *p, const uint64_t *v)
{
    if constexpr (RL == 0) {
        p[0] = v[0];
    } else if constexpr (RL == 1) {
        asm volatile("st.global.v2.u64 [%0], {%1, %2};" ::"l"(p), "l"(v[0]), "l"(v[1]) : "memory");
    } else {
#pragma unroll
        for (int i = 0; i < (1 << RL); i += 4)
            asm volatile("st.global.v4.u64 [%0], {%1, %2, %3, %4};" ::"l"(p + i), "l"(v[i]), "l"(v[i + 1]),
                         "l"(v[i + 2]), "l"(v[i + 3])
                         : "memory");
    }
}
// A round's register pattern straight from / to global memory, one vector per run.
template <int ELOG, int LO, int W>
__device__ __forceinline__ void ld_pattern(const uint64_t *blk, int ktr, uint64_t (&v)[1 << ELOG])
{
    constexpr int RL = run_log(ELOG, LO, W);
#pragma unroll
    for (int e = 0; e < (1 << ELOG); e += (1 << RL)) ld_run<RL>(blk + ktr + kmap(ELOG, LO, W, 0, e), v + e);
}
template <int ELOG, int LO, int W>
__device__ __forceinline__ void st_pattern(uint64_t *blk, int ktr, const uint64_t (&v)[1 << ELOG])
{
    constexpr int RL = run_log(ELOG, LO, W);
#pragma unroll
    for (int e = 0; e < (1 << ELOG); e += (1 << RL)) st_run<RL>(blk + ktr + kmap(ELOG, LO, W, 0, e), v + e);
}

// Batch structure of the rows: row = item * rstride + ri, ri < rstride, n_items items.
// z / n_items by multiply-high (Granlund-Montgomery; z < 2^31): q = (umulhi(z, mul) + z) >> shift.
struct RowMap {
    uint32_t n_items, rstride, mul, shift;
};
RowMap make_rowmap(uint32_t n_items, uint32_t rstride)
{
    uint32_t s = 0;
    while ((1ull << s) < n_items) ++s;
    const uint32_t mul = (uint32_t)(((1ull << 32) * ((1ull << s) - n_items)) / n_items + 1);
    return RowMap{n_items, rstride, mul, s};
}

// Which row / block / group / lane this thread works on.
//   col pass: CTA (x, y) = G consecutive columns of row y (coalesced strided columns).
//   row pass: groups are enumerated item-fastest, z -> (item, block, ri), so the groups of
//   a CTA are mostly the same block of the same residue row of different batch items:
//   their twiddles coincide (warp-broadcast loads) and need no per-CTA tail padding.
template <class Gm, int LOGS, int OTHER, bool COL>
__device__ __forceinline__ void locate(RowMap rm, size_t &row, int &gi, int &g, int &t)
{
    const int tid = threadIdx.x;
    if (COL) {
        g = tid & (Gm::G - 1);
        t = tid >> Gm::LOGG;
        gi = blockIdx.x * Gm::G + g;
        row = blockIdx.y;
    } else {
        g = tid >> Gm::LOGT;
        t = tid & (Gm::T - 1);
        const uint32_t z = blockIdx.x * Gm::G + g;
        const uint32_t rest = (__umulhi(z, rm.mul) + z) >> rm.shift;
        const uint32_t item = z - rest * rm.n_items;
        gi = rest & ((1u << OTHER) - 1);
        row = (size_t)item * rm.rstride + (rest >> OTHER);
    }
}

// ---------------------------------------------------------------- round bodies
// Forward round r: bits [lo, lo+w) with the narrow round first.  Loads the round's
// distinct twiddles (the twiddle of stage s depends only on the top s register bits:
// 2^s per stage, issued before the first butterfly so their latency overlaps) and runs
// its CT butterflies with the lazy 16q schedule (U >= 8q corrected at global stages
// = 3 mod 4).
template <class Gm, int LOGS>
struct FwdGeo {
    static constexpr int W0 = LOGS - (Gm::R - 1) * Gm::ELOG;
    __device__ static constexpr int w(int r) { return r == 0 ? W0 : Gm::ELOG; }
    __device__ static constexpr int hi(int r) { return LOGS - 1 - (r == 0 ? 0 : W0 + (r - 1) * Gm::ELOG); }
    __device__ static constexpr int lo(int r) { return hi(r) - w(r) + 1; }
};

template <class Gm, int LOGS>
__device__ __forceinline__ void fwd_bfly(uint64_t (&v)[Gm::E], int r, int ktr, int prefix, const TwPair *tw, uint64_t q)
{
    using F = FwdGeo<Gm, LOGS>;
    constexpr int ELOG = Gm::ELOG, E = Gm::E;
    const int w = F::w(r), lo = F::lo(r), lp0 = LOGS - 1 - F::hi(r);
    const uint64_t qm = kLazyMul * q, q8 = 8 * q;
    TwPair tws[E];
    auto load_stage = [&](int s) {
        const int lp = lp0 + s;
        const TwPair *tb = tw + (1 << (Gm::LBASE + lp)) + (prefix << lp) + (ktr >> (LOGS - lp));
#pragma unroll
        for (int mm = 0; mm < (1 << s); ++mm)
            tws[(1 << s) - 1 + mm] = ld_tw(tb + (kmap(ELOG, lo, w, 0, mm << (ELOG - s)) >> (LOGS - lp)));
    };
    if (!kTwStage) {
#pragma unroll
        for (int s = 0; s < w; ++s) load_stage(s);
    }
#pragma unroll
    for (int s = 0; s < w; ++s) {
        if (kTwStage) load_stage(s);
        const int bit = ELOG - 1 - s;  // register bit paired in this stage
        const bool corr = fwd_corr(Gm::LBASE + lp0 + s);
#pragma unroll
        for (int mm = 0; mm < (1 << s); ++mm) {
            const int erep = mm << (ELOG - s);
            const TwPair wt = tws[(1 << s) - 1 + mm];
#pragma unroll
            for (int e = erep; e < erep + (1 << (ELOG - s)); ++e) {
                if (e & (1 << bit)) continue;
                uint64_t U = v[e];
                uint64_t V = v[e | (1 << bit)];
                if (corr) U = csub64(U, q8);
                V = bfly_mul(V, wt.w, wt.wp, q);
                v[e] = U + V;
                v[e | (1 << bit)] = U - V + qm;
            }
        }
    }
}

// Inverse round r: bits [lo, lo+w) from the bottom up (the narrow round last); stage s
// needs 2^(w-1-s) distinct twiddles (register bits above it).  GS butterflies in [0, 4q).
template <class Gm, int LOGS>
struct InvGeo {
    __device__ static constexpr int lo(int r) { return r * Gm::ELOG; }
    __device__ static constexpr int w(int r) { return (LOGS - lo(r)) < Gm::ELOG ? (LOGS - lo(r)) : Gm::ELOG; }
};

// FOLD (last round of the col pass): the transform's final stage (local stage 0, one
// twiddle w1 = tw[1] for the whole limb) absorbs the N^{-1} scaling, X' = (X + Y) N^{-1},
// Y' = (X - Y) (w1 N^{-1}), fully reduced: no separate pass over the outputs.
template <class Gm, int LOGS, bool FOLD>
__device__ __forceinline__ void inv_bfly(uint64_t (&v)[Gm::E], int r, int ktr, int prefix, const TwPair *tw, uint64_t q,
                                         TwPair ninv, TwPair ninv_w)
{
    using I = InvGeo<Gm, LOGS>;
    constexpr int ELOG = Gm::ELOG, E = Gm::E;
    const int lo = I::lo(r), w = I::w(r);
    const uint64_t qm = kLazyMul * q;  // words stay in [0, kLazyMul q)
    TwPair tws[E];
    auto load_stage = [&](int s) {
        const int lp = LOGS - 1 - (lo + s);
        const int ntop = w - 1 - s;
        const TwPair *tb = tw + (1 << (Gm::LBASE + lp)) + (prefix << lp) + (ktr >> (LOGS - lp));
#pragma unroll
        for (int mm = 0; mm < (1 << ntop); ++mm)
            tws[(1 << ntop) - 1 + mm] = ld_tw(tb + (kmap(ELOG, lo, w, 0, mm << (ELOG - ntop)) >> (LOGS - lp)));
    };
    if (!kTwStage) {
#pragma unroll
        for (int s = 0; s < w; ++s) load_stage(s);
    }
#pragma unroll
    for (int s = 0; s < w; ++s) {
        if (kTwStage) load_stage(s);
        const int bit = ELOG - w + s;  // register bit of k-bit lo+s
        const int ntop = w - 1 - s;    // register bits above: the twiddle depends on these only
#pragma unroll
        for (int mm = 0; mm < (1 << ntop); ++mm) {
            const int erep = mm << (ELOG - ntop);
            const TwPair wt = tws[(1 << ntop) - 1 + mm];
#pragma unroll
            for (int e = erep; e < erep + (1 << (ELOG - ntop)); ++e) {
                if (e & (1 << bit)) continue;
                const uint64_t X = v[e];
                const uint64_t Y = v[e | (1 << bit)];
                if (FOLD && lo + s == LOGS - 1) {
                    v[e] = shoup(X + Y, ninv.w, ninv.wp, q);
                    v[e | (1 << bit)] = shoup(X - Y + qm, ninv_w.w, ninv_w.wp, q);
                } else {
                    v[e] = csub64(X + Y, qm);
                    v[e | (1 << bit)] = bfly_mul(X - Y + qm, wt.w, wt.wp, q);
                }
            }
        }
    }
}

// ---------------------------------------------------------------- forward
// Round widths: the first (top) round takes LOGS - (R-1)*ELOG bits, the others ELOG.
// EPI (row pass only): the RowEpi epilogue replaces the plain store; a separate instantiation
// so that the plain pass carries none of its code or registers
template <int LOGS, int OTHER, bool COL, bool EPI = false>
__global__ void __launch_bounds__(kCtaThreads, kMinCtas) ntt_fwd_pass(uint64_t *__restrict__ data, KTables kt, PrimeMap pm, RowMap rm,
                                                                      ColSrc cs, RowEpi ep)
{
    using Gm = Geo<LOGS, OTHER, COL>;
    constexpr int ELOG = Gm::ELOG, S = Gm::S, E = Gm::E, G = Gm::G, R = Gm::R;
    constexpr int LOGN = LOGS + OTHER;
    extern __shared__ uint64_t sm[];
    size_t row;
    int gi, g, t;
    locate<Gm, LOGS, OTHER, COL>(rm, row, gi, g, t);
    const int p = pm.idx[row % pm.period];
    const uint64_t q = kt.q[p];
    const TwPair *tw = kt.tw_fwd + ((size_t)p << LOGN);
    uint64_t *a = data + ((size_t)row << LOGN);
    uint64_t *buf0 = sm, *buf1 = sm + S * G;
    uint64_t *blk = a + ((size_t)gi << LOGS);  // row pass: this group's block
    uint64_t v[E];
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const int w = FwdGeo<Gm, LOGS>::w(r), lo = FwdGeo<Gm, LOGS>::lo(r);
        const int ktr = kmap(ELOG, lo, w, t, 0);
        const int sb = sbase<Gm, LOGS, COL>(ktr, g);
        if (r == 0 && !COL) {
            // row pass: the round's register pattern straight from the block (runs of
            // consecutive words per thread, 16/32-byte vector loads, coalesced across lanes)
            ld_pattern<ELOG, FwdGeo<Gm, LOGS>::lo(0), FwdGeo<Gm, LOGS>::w(0)>(blk, ktr, v);
        } else if (r == 0 && cs.x != nullptr) {
            // fused ModUp (alpha = 1): this row is x_j mod q of a source limb x_j
            const uint64_t *src = cs.x + (row / cs.period) * cs.xs + ((size_t)cs.src[row % cs.period] << LOGN);
            // (a fused BConv row of a single-limb digit: y = x_j mod q_t, reduced into [0, 2q))
            const uint64_t *col = src + gi + ((size_t)ktr << OTHER);
            const uint32_t rr = row % cs.period;
            if ((cs.below2q[rr >> 5] >> (rr & 31)) & 1) {
#pragma unroll
                for (int e = 0; e < E; ++e) v[e] = col[(size_t)kmap(ELOG, lo, w, 0, e) << OTHER];
            } else {
                const uint64_t rc = kt.recip[p];
#pragma unroll
                for (int e = 0; e < E; ++e) v[e] = shoup_lazy(col[(size_t)kmap(ELOG, lo, w, 0, e) << OTHER], 1, rc, q);
            }
            if (cs.sub != nullptr) {
                const uint64_t h = cs.sub[p];
#pragma unroll
                for (int e = 0; e < E; ++e) v[e] = sub_mod(csub64(v[e], q), h, q);
            }
        } else if (r == 0) {
            const uint64_t *col = a + gi + ((size_t)ktr << OTHER);
#pragma unroll
            for (int e = 0; e < E; ++e) v[e] = col[(size_t)kmap(ELOG, lo, w, 0, e) << OTHER];
        } else {
            const uint64_t *b = ((r - 1) & 1) ? buf1 : buf0;
#pragma unroll
            for (int e = 0; e < E; ++e) v[e] = b[soff<Gm, LOGS, COL>(sb, kmap(ELOG, lo, w, 0, e))];
        }
        fwd_bfly<Gm, LOGS>(v, r, ktr, COL ? 0 : gi, tw, q);
        if (r == R - 1 && !COL && EPI) {
            // fused epilogue (RowEpi): (X - v) mul + addends, written to ep.out
            constexpr int LOL = FwdGeo<Gm, LOGS>::lo(R - 1), WL = FwdGeo<Gm, LOGS>::w(R - 1);
            const float qinv = qinv_est(q);
            const uint32_t np = ep.npoly ? ep.npoly : 2;
            const size_t b = row / (np * ep.per);
            const uint32_t rr = (uint32_t)(row % (np * ep.per)), poly = rr / ep.per, i = rr % ep.per;
            const uint32_t k0 = ((uint32_t)gi << LOGS) | (uint32_t)ktr;  // this thread's first word
            uint64_t x[E];
            ld_pattern<ELOG, LOL, WL>(ep.X + b * ep.xs + poly * ep.xps + ((size_t)i << LOGN), k0, x);
            const TwPair m = ep.mul[i];
#pragma unroll
            for (int e = 0; e < E; ++e) v[e] = shoup(x[e] + q - reduce_est(v[e], q, qinv), m.w, m.wp, q);
            const size_t ao = b * ep.as + ((size_t)i << LOGN);
            if (poly == 0) {
                if (ep.add0) {
#pragma unroll
                    for (int e = 0; e < E; ++e) {
                        const uint32_t j = k0 + (uint32_t)kmap(ELOG, LOL, WL, 0, e);
                        uint32_t src = j;
                        if (ep.g0 != 1) {
                            const uint32_t ex = ((2u * (__brev(j) >> (32 - LOGN)) + 1u) * ep.g0) & ((2u << LOGN) - 1u);
                            src = __brev((ex - 1u) >> 1) >> (32 - LOGN);
                        }
                        v[e] = add_mod(v[e], ep.add0[ao + src], q);
                    }
                }
                if (ep.add2) {
                    ld_pattern<ELOG, LOL, WL>(ep.add2 + ao, k0, x);
#pragma unroll
                    for (int e = 0; e < E; ++e) v[e] = add_mod(v[e], x[e], q);
                }
            } else if (ep.add1) {
                ld_pattern<ELOG, LOL, WL>(ep.add1 + ao, k0, x);
#pragma unroll
                for (int e = 0; e < E; ++e) v[e] = add_mod(v[e], x[e], q);
            }
            st_pattern<ELOG, LOL, WL>(ep.out + b * ep.os + poly * ep.ops + ((size_t)i << LOGN), k0, v);
        } else if (r == R - 1 && !COL) {
            // row pass: full reduction (< 16q -> [0, q)), stored as the last round's runs
            // (8 consecutive words per thread: two 32-byte stores)
            const float qinv = qinv_est(q);
#pragma unroll
            for (int e = 0; e < E; ++e) v[e] = reduce_est(v[e], q, qinv);
            st_pattern<ELOG, FwdGeo<Gm, LOGS>::lo(R - 1), FwdGeo<Gm, LOGS>::w(R - 1)>(blk, ktr, v);
        } else if (r == R - 1) {
            uint64_t *col = a + gi + ((size_t)ktr << OTHER);
#pragma unroll
            for (int e = 0; e < E; ++e) col[(size_t)kmap(ELOG, lo, w, 0, e) << OTHER] = v[e];
        } else {
            uint64_t *b = (r & 1) ? buf1 : buf0;
#pragma unroll
            for (int e = 0; e < E; ++e) b[soff<Gm, LOGS, COL>(sb, kmap(ELOG, lo, w, 0, e))] = v[e];
            __syncthreads();
        }
    }
}

// ---------------------------------------------------------------- inverse
// Stages in reverse: local stage lp = LOGS-1 .. 0 operates on bit LOGS-1-lp, so
// rounds own bits from the bottom up (the narrow round last, at the top).  GS
// butterflies keep words in [0, 4q) (inputs must be < 4q); the col pass (last) folds
// N^{-1} into its final stage and writes canonical residues.
template <int LOGS, int OTHER, bool COL>
__global__ void __launch_bounds__(kCtaThreads, kMinCtas) ntt_inv_pass(uint64_t *__restrict__ data, KTables kt, PrimeMap pm, RowMap rm,
                                                                      InvSrc is)
{
    using Gm = Geo<LOGS, OTHER, COL>;
    constexpr int ELOG = Gm::ELOG, S = Gm::S, E = Gm::E, G = Gm::G, R = Gm::R;
    constexpr int LOGN = LOGS + OTHER;
    extern __shared__ uint64_t sm[];
    size_t row;
    int gi, g, t;
    locate<Gm, LOGS, OTHER, COL>(rm, row, gi, g, t);
    const int p = pm.idx[row % pm.period];
    const uint64_t q = kt.q[p];
    const TwPair *tw = kt.tw_inv + ((size_t)p << LOGN);
    uint64_t *a = data + ((size_t)row << LOGN);
    uint64_t *buf0 = sm, *buf1 = sm + S * G;
    uint64_t *blk = a + ((size_t)gi << LOGS);  // row pass: this group's block
    uint64_t v[E];
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const int lo = r * ELOG;
        const int w = (LOGS - lo) < ELOG ? (LOGS - lo) : ELOG;
        const int ktr = kmap(ELOG, lo, w, t, 0);
        const int sb = sbase<Gm, LOGS, COL>(ktr, g);
        if (r == 0 && !COL && is.x != nullptr) {
            // out-of-place source row, optionally through sigma_g
            const uint64_t *srow = is.x + (row / is.per) * is.xs + (row % is.per) * is.ss;
            if (is.g == 1) {
                ld_pattern<ELOG, InvGeo<Gm, LOGS>::lo(0), InvGeo<Gm, LOGS>::w(0)>(srow + ((size_t)gi << LOGS), ktr, v);
            } else {
                // perm_g maps every aligned 32-word span onto an aligned 32-word span, so a
                // warp's gathers stay within a few sectors (L1 serves the rest)
                const uint32_t base = ((uint32_t)gi << LOGS) | (uint32_t)ktr;
#pragma unroll
                for (int e = 0; e < E; ++e) {
                    const uint32_t j = base | (uint32_t)kmap(ELOG, lo, w, 0, e);
                    const uint32_t ex = ((2u * (__brev(j) >> (32 - LOGN)) + 1u) * is.g) & ((2u << LOGN) - 1u);
                    v[e] = srow[__brev((ex - 1u) >> 1) >> (32 - LOGN)];
                }
            }
        } else if (r == 0 && !COL) {
            ld_pattern<ELOG, InvGeo<Gm, LOGS>::lo(0), InvGeo<Gm, LOGS>::w(0)>(blk, ktr, v);
        } else if (r == 0) {
            const uint64_t *col = a + gi + ((size_t)ktr << OTHER);
#pragma unroll
            for (int e = 0; e < E; ++e) v[e] = col[(size_t)kmap(ELOG, lo, w, 0, e) << OTHER];
        } else {
            const uint64_t *b = ((r - 1) & 1) ? buf1 : buf0;
#pragma unroll
            for (int e = 0; e < E; ++e) v[e] = b[soff<Gm, LOGS, COL>(sb, kmap(ELOG, lo, w, 0, e))];
        }
        if (COL && r == R - 1)
            inv_bfly<Gm, LOGS, true>(v, r, ktr, 0, tw, q, kt.n_inv[p], kt.n_inv_w[p]);
        else
            inv_bfly<Gm, LOGS, false>(v, r, ktr, COL ? 0 : gi, tw, q, TwPair{}, TwPair{});
        if (r == R - 1 && !COL) {
            st_pattern<ELOG, InvGeo<Gm, LOGS>::lo(R - 1), InvGeo<Gm, LOGS>::w(R - 1)>(blk, ktr, v);
        } else if (r == R - 1) {
            // canonical [0, q): N^{-1} is folded into the last stage (inv_bfly<FOLD>)
            uint64_t *col = a + gi + ((size_t)ktr << OTHER);
            if (is.add_half) {
#pragma unroll
                for (int e = 0; e < E; ++e) v[e] = add_mod(v[e], q >> 1, q);
            }
#pragma unroll
            for (int e = 0; e < E; ++e) col[(size_t)kmap(ELOG, lo, w, 0, e) << OTHER] = v[e];
        } else {
            uint64_t *b = (r & 1) ? buf1 : buf0;
#pragma unroll
            for (int e = 0; e < E; ++e) b[soff<Gm, LOGS, COL>(sb, kmap(ELOG, lo, w, 0, e))] = v[e];
            __syncthreads();
        }
    }
}

template <bool FWD, int LOGS, int OTHER, bool COL>
void launch_one(uint64_t *d, uint32_t rows, const KTables &kt, const PrimeMap &pm, const ColSrc *cs, const InvSrc *is,
                const RowEpi *ep, cudaStream_t s)
{
    using Gm = Geo<LOGS, OTHER, COL>;
    static_assert(Gm::SMEM <= 48 * 1024, "NTT pass exceeds the default dynamic shared memory");
    // prefer the shared-memory carveout: residency is bounded by registers, not by L1
    static std::atomic<uint64_t> attr{0};
    once_per_device(attr, [] {
        if (FWD)
        {
            CUDA_CHECK(cudaFuncSetAttribute(ntt_fwd_pass<LOGS, OTHER, COL, false>,
                                            cudaFuncAttributePreferredSharedMemoryCarveout,
                                            cudaSharedmemCarveoutMaxShared));
            if (!COL)
                CUDA_CHECK(cudaFuncSetAttribute(ntt_fwd_pass<LOGS, OTHER, COL, true>,
                                                cudaFuncAttributePreferredSharedMemoryCarveout,
                                                cudaSharedmemCarveoutMaxShared));
        } else
            CUDA_CHECK(cudaFuncSetAttribute(ntt_inv_pass<LOGS, OTHER, COL>,
                                            cudaFuncAttributePreferredSharedMemoryCarveout,
                                            cudaSharedmemCarveoutMaxShared));
    });
    auto go = [&](dim3 grid, uint64_t *dd, RowMap rm, const ColSrc &src) {
        if constexpr (FWD) {
            if (!COL && ep)
                ntt_fwd_pass<LOGS, OTHER, COL, true><<<grid, Gm::THREADS, Gm::SMEM, s>>>(dd, kt, pm, rm, src, *ep);
            else
                ntt_fwd_pass<LOGS, OTHER, COL, false><<<grid, Gm::THREADS, Gm::SMEM, s>>>(dd, kt, pm, rm, src,
                                                                                         RowEpi{});
        }
        else
            ntt_inv_pass<LOGS, OTHER, COL><<<grid, Gm::THREADS, Gm::SMEM, s>>>(
                dd, kt, pm, rm, !is ? InvSrc{} : !COL ? *is : InvSrc{nullptr, 0, 0, 1, 1, is->add_half});
    };
    if (COL) {
        // grid.y <= 65535: chunks of whole periods keep row % period aligned
        const uint32_t chunk = 65535u / pm.period * pm.period;
        for (uint32_t r0 = 0; r0 < rows; r0 += chunk) {
            ColSrc src{};
            if (cs) {
                src = *cs;
                src.x += (size_t)(r0 / pm.period) * cs->xs;
            }
            go(dim3((1u << OTHER) / Gm::G, std::min(chunk, rows - r0)), d + ((size_t)r0 << (LOGS + OTHER)),
               make_rowmap(rows, 1), src);
        }
    } else {
        // rows are items of pm.period residue rows each whenever that divides
        const uint32_t stride = rows % pm.period == 0 ? pm.period : 1;
        const size_t groups = (size_t)rows << OTHER;
        MMFHE_REQUIRE(groups < (1ull << 31), MMFHE_E_SHAPE, "NTT batch too large for one launch");
        go(dim3((uint32_t)(groups / Gm::G)), d, make_rowmap(rows / stride, stride), ColSrc{});
    }
}

#ifndef MMFHE_NTT_L1_14
#define MMFHE_NTT_L1_14 7
#endif
// Radix-8 everywhere: radix-16 (ELOG = 4) halves the exchanges but its 64 KiB CTAs and
// 16 live words per thread halved occupancy and ran 2x slower on B200 (measured).
// log N = L1 + L2, L1 = floor(log N / 2): col pass <L1, L2>, row pass <L2, L1>.
template <bool FWD, bool COL>
void launch_pass(uint32_t log_n, uint64_t *d, uint32_t rows, const KTables &kt, const PrimeMap &pm, const ColSrc *cs,
                 const InvSrc *is, const RowEpi *ep, cudaStream_t s)
{
#define MMFHE_NTT_CASE(LN, A, B)                                    \
    case LN:                                                        \
        if (COL)                                                    \
            launch_one<FWD, A, B, true>(d, rows, kt, pm, cs, is, nullptr, s);  \
        else                                                        \
            launch_one<FWD, B, A, false>(d, rows, kt, pm, nullptr, is, ep, s); \
        break;
    switch (log_n) {
        MMFHE_NTT_CASE(4, 2, 2)
        MMFHE_NTT_CASE(5, 2, 3)
        MMFHE_NTT_CASE(6, 3, 3)
        MMFHE_NTT_CASE(7, 3, 4)
        MMFHE_NTT_CASE(8, 4, 4)
        MMFHE_NTT_CASE(9, 4, 5)
        MMFHE_NTT_CASE(10, 5, 5)
        MMFHE_NTT_CASE(11, 5, 6)
        MMFHE_NTT_CASE(12, 6, 6)
        MMFHE_NTT_CASE(13, 6, 7)
        MMFHE_NTT_CASE(14, MMFHE_NTT_L1_14, 14 - MMFHE_NTT_L1_14)
        MMFHE_NTT_CASE(15, 7, 8)
        MMFHE_NTT_CASE(16, 8, 8)
    default:
        throw Error(MMFHE_E_PARAMS, "unsupported NTT size");
    }
#undef MMFHE_NTT_CASE
}

void split(uint32_t log_n, int &L1, int &L2)
{
    L1 = log_n == 14 ? MMFHE_NTT_L1_14 : (int)log_n / 2;
    L2 = (int)log_n - L1;
}

}  // namespace

void ntt_forward(Ctx &c, uint64_t *d, uint32_t rows, const PrimeMap &pm, const ColSrc *src, const RowEpi *epi)
{
    if (!rows) return;
    MMFHE_REQUIRE(!src || src->period == pm.period, MMFHE_E_LAYOUT, "NTT source map period");
    int L1, L2;
    split(c.log_n, L1, L2);
    const double bytes = 16.0 * rows * c.n;  // one read + one write of every word per pass
    {
        ProfScope ps(c, "ntt_fwd_col", bytes, 0.5 * rows * c.n * L1);
        launch_pass<true, true>(c.log_n, d, rows, c.kt, pm, src, nullptr, nullptr, c.stream);
    }
    {
        // with the epilogue: + X read, out written, addends read (instead of the v write)
        const double ebytes = !epi ? 0.0
                                   : 8.0 * rows * c.n *
                                         (1.0 + (epi->add0 ? 0.5 : 0.0) + (epi->add1 ? 0.5 : 0.0) +
                                          (epi->add2 ? 0.5 : 0.0));
        MMFHE_REQUIRE(!epi || (epi->per >= 1 && rows % ((epi->npoly ? epi->npoly : 2) * epi->per) == 0),
                      MMFHE_E_LAYOUT, "NTT epilogue rows");
        // ops: the pass's butterflies, plus (epilogue) the final step's Shoup product by P^{-1} or
        // q_l^{-1} per word -- SURVEY §8(d)'s "2L'N [x P^{-1}]" modmuls -- counted as one
        // butterfly-equivalent each (the microbenchmark's Shoup modmul and CT butterfly rates
        // agree within 2%)
        ProfScope ps(c, epi ? "ntt_fwd_row_epi" : "ntt_fwd_row", bytes + ebytes,
                     0.5 * rows * c.n * L2 + (epi ? 1.0 * rows * c.n : 0.0));
        launch_pass<true, false>(c.log_n, d, rows, c.kt, pm, nullptr, nullptr, epi, c.stream);
    }
    c.launches += 2;
    CUDA_CHECK(cudaGetLastError());
}

void ntt_inverse(Ctx &c, uint64_t *d, uint32_t rows, const PrimeMap &pm, const InvSrc *src)
{
    if (!rows) return;
    int L1, L2;
    split(c.log_n, L1, L2);
    const double bytes = 16.0 * rows * c.n;
    {
        ProfScope ps(c, "ntt_inv_row", bytes, 0.5 * rows * c.n * L2);
        MMFHE_REQUIRE(!src || ((src->x || src->g == 1) && src->per >= 1 && (src->g & 1) && src->g < 2 * c.n),
                      MMFHE_E_LAYOUT, "INTT source");
        launch_pass<false, false>(c.log_n, d, rows, c.kt, pm, nullptr, src, nullptr, c.stream);
    }
    {
        ProfScope ps(c, "ntt_inv_col", bytes, 0.5 * rows * c.n * L1);
        launch_pass<false, true>(c.log_n, d, rows, c.kt, pm, nullptr, src, nullptr, c.stream);
    }
    c.launches += 2;
    CUDA_CHECK(cudaGetLastError());
}

}  // namespace mmfhe
