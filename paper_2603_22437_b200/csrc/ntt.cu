// ntt.cu -- batched negacyclic NTT / INTT across RNS limbs.
//
// Forward: Cooley-Tukey, natural order in, bit-reversed order out, psi-twist
// merged into the twiddles (tw_fwd[m + i] = psi^{bitrev(m+i)}): stage l (m = 2^l)
// pairs j, j + N/2^{l+1} with twiddle index m + (j >> (log N - l)).
// Inverse: Gentleman-Sande with psi^{-bitrev}, bit-reversed in, natural out,
// times N^{-1}.  Harvey lazy butterflies: values stay in [0, 4q) (q < 2^60).
//
// B200 mapping.  A limb of N = 2^16 words (512 KiB) exceeds one SM's shared
// memory, so the transform is two passes over HBM (logN = L1 + L2):
//   col pass -- stages 0..L1-1 on 2^L2 strided columns of 2^L1 words; a warp
//               spans G consecutive columns (G*8-byte sector-aligned runs);
//   row pass -- stages L1..logN-1 on contiguous blocks of 2^L2 words; one warp
//               per block, consecutive lanes on consecutive words.
// Inside a pass each thread holds E = 2^ELOG = 8 words in registers and runs
// ELOG butterfly stages there (radix-8); rounds exchange data through
// double-buffered shared memory (one __syncthreads per exchange).  All index
// arithmetic is shifts/masks of compile-time widths.  Every limb of every
// polynomial of a batch goes in one launch (grid.y = rows, prime per row).
#include <algorithm>

#include "context.h"
#include "modarith.cuh"

namespace mmfhe {

namespace {

constexpr int kCtaThreads = 256;

__device__ __forceinline__ uint64_t reduce4q(uint64_t x, uint64_t q)
{
    x = x >= 2 * q ? x - 2 * q : x;
    return x >= q ? x - q : x;
}

// Local index of register e of thread t in a round that owns bits [lo, lo+w):
// y = top w bits of e -> bits lo..lo+w-1; z = (t, low ELOG-w bits of e) fills
// the free bit positions [0, lo) and [lo+w, LOGS) in ascending order.
template <int ELOG>
__device__ __forceinline__ int kmap(int lo, int w, int t, int e)
{
    const int y = e >> (ELOG - w);
    const int z = (t << (ELOG - w)) | (e & ((1 << (ELOG - w)) - 1));
    return (z & ((1 << lo) - 1)) | (y << lo) | ((z >> lo) << (lo + w));
}

// Shared-memory word of local element k in the row pass.  One warp spans
// 32/T groups; in rounds 1-2 its lanes step k by 2-16 words, which would hit only
// 2-4 of the 16 64-bit bank pairs.  XOR-ing the low 4 bits with a function of
// the high bits makes every round's lane pattern cover all 16 bank pairs
// (derived for LOGS = 7 and 8, both directions; identity otherwise).
template <int LOGS>
__device__ __forceinline__ int swz(int k)
{
    if (LOGS == 8) return k ^ (((k >> 4) & 7) ^ (((k >> 5) & 3) << 2));
    if (LOGS == 7) return k ^ ((((k >> 4) & 7) << 1) ^ ((k >> 6) & 1));
    return k;
}

// Column pass (word a = k*G + g): conflict-free for LOGS <= 7; for LOGS = 8 (G = 8)
// rounds 2 would leave bit 3 constant across a warp -- flip it with a parity of bits 4, 6.
template <int LOGS>
__device__ __forceinline__ int colswz(int a)
{
    if (LOGS == 8) return a ^ ((((a >> 4) ^ (a >> 6)) & 1) << 3);
    return a;
}

// Global word offset (within the row) of local element k of group gi.
template <bool COL>
__device__ __forceinline__ size_t gaddr(int k, int gi, int L2, int LOGS)
{
    return COL ? (((size_t)k << L2) + gi) : (((size_t)gi << LOGS) + k);
}

// ---------------------------------------------------------------- forward
template <int LOGS, int ELOG, bool COL>
__global__ void __launch_bounds__(kCtaThreads) ntt_fwd_pass(uint64_t *__restrict__ data, KTables kt, PrimeMap pm,
                                                            int log_g)
{
    constexpr int S = 1 << LOGS, E = 1 << ELOG, T = S >> ELOG, R = (LOGS + ELOG - 1) / ELOG;
    extern __shared__ uint64_t sm[];
    const int G = 1 << log_g;
    const int row = blockIdx.y;
    const int p = pm.idx[row % pm.period];
    const uint64_t q = kt.q[p], q2 = 2 * q;
    const TwPair *tw = kt.tw_fwd + (size_t)p * kt.n;
    uint64_t *a = data + (size_t)row * kt.n;
    const int logn = kt.log_n;
    const int L2 = logn - LOGS;  // col pass: 2^L2 columns
    const int tid = threadIdx.x;
    int g, t;
    if (COL) {
        g = tid & (G - 1);
        t = tid >> log_g;
    } else {
        t = tid & (T - 1);
        g = tid / T;
    }
    const int gi = blockIdx.x * G + g;        // global column / block index
    const int lbase = COL ? 0 : logn - LOGS;  // global stage of local stage 0
    const int prefix = COL ? 0 : gi;
    uint64_t *buf0 = sm, *buf1 = sm + S * G;
    uint64_t v[E];
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const int hi = LOGS - 1 - r * ELOG;
        const int w = (LOGS - r * ELOG) < ELOG ? (LOGS - r * ELOG) : ELOG;
        const int lo = hi - w + 1;
        if (r == 0) {
#pragma unroll
            for (int e = 0; e < E; ++e) v[e] = a[gaddr<COL>(kmap<ELOG>(lo, w, t, e), gi, L2, LOGS)];
        } else {
            const uint64_t *b = ((r - 1) & 1) ? buf1 : buf0;
#pragma unroll
            for (int e = 0; e < E; ++e) {
                const int k = kmap<ELOG>(lo, w, t, e);
                v[e] = COL ? b[colswz<LOGS>(k * G + g)] : b[g * S + swz<LOGS>(k)];
            }
        }
#pragma unroll
        for (int s = 0; s < w; ++s) {
            const int lp = r * ELOG + s;   // local stage
            const int bit = ELOG - 1 - s;  // register bit paired in this stage
            // In a full-width round the twiddle depends only on the top s register bits: load
            // each distinct one once.  In the (last, lo = 0) partial round the spare register
            // bits map ABOVE the round's bits, so every butterfly has its own twiddle.
            const int tb = (w == ELOG) ? s : ELOG;  // ELOG: one twiddle per register
#pragma unroll
            for (int m = 0; m < (1 << tb); ++m) {
                const int erep = m << (ELOG - tb);
                if (erep & (1 << bit)) continue;  // per-register case: pair leaders only
                const int krep = kmap<ELOG>(lo, w, t, erep);
                const TwPair wt = tw[(1 << (lbase + lp)) + (prefix << lp) + (krep >> (LOGS - lp))];
#pragma unroll
                for (int e = erep; e < erep + (1 << (ELOG - tb)); ++e) {
                    if (e & (1 << bit)) continue;
                    uint64_t U = v[e];
                    uint64_t V = v[e | (1 << bit)];
                    U = U >= q2 ? U - q2 : U;
                    V = shoup_lazy(V, wt.w, wt.wp, q);
                    v[e] = U + V;
                    v[e | (1 << bit)] = U - V + q2;
                }
            }
        }
        if (r == R - 1) {
#pragma unroll
            for (int e = 0; e < E; ++e) {
                const uint64_t x = COL ? v[e] : reduce4q(v[e], q);
                a[gaddr<COL>(kmap<ELOG>(lo, w, t, e), gi, L2, LOGS)] = x;
            }
        } else {
            uint64_t *b = (r & 1) ? buf1 : buf0;
#pragma unroll
            for (int e = 0; e < E; ++e) {
                const int k = kmap<ELOG>(lo, w, t, e);
                if (COL)
                    b[colswz<LOGS>(k * G + g)] = v[e];
                else
                    b[g * S + swz<LOGS>(k)] = v[e];
            }
            __syncthreads();
        }
    }
}

// ---------------------------------------------------------------- inverse
// Stages in reverse: local stage lp = LOGS-1 .. 0 operates on bit LOGS-1-lp, so
// rounds own bits from the bottom up.  The col pass (last) multiplies by N^{-1}.
template <int LOGS, int ELOG, bool COL>
__global__ void __launch_bounds__(kCtaThreads) ntt_inv_pass(uint64_t *__restrict__ data, KTables kt, PrimeMap pm,
                                                            int log_g)
{
    constexpr int S = 1 << LOGS, E = 1 << ELOG, T = S >> ELOG, R = (LOGS + ELOG - 1) / ELOG;
    extern __shared__ uint64_t sm[];
    const int G = 1 << log_g;
    const int row = blockIdx.y;
    const int p = pm.idx[row % pm.period];
    const uint64_t q = kt.q[p], q2 = 2 * q;
    const TwPair *tw = kt.tw_inv + (size_t)p * kt.n;
    uint64_t *a = data + (size_t)row * kt.n;
    const int logn = kt.log_n;
    const int L2 = logn - LOGS;
    const int tid = threadIdx.x;
    int g, t;
    if (COL) {
        g = tid & (G - 1);
        t = tid >> log_g;
    } else {
        t = tid & (T - 1);
        g = tid / T;
    }
    const int gi = blockIdx.x * G + g;
    const int lbase = COL ? 0 : logn - LOGS;
    const int prefix = COL ? 0 : gi;
    uint64_t *buf0 = sm, *buf1 = sm + S * G;
    uint64_t v[E];
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const int lo = r * ELOG;
        const int w = (LOGS - lo) < ELOG ? (LOGS - lo) : ELOG;
        if (r == 0) {
#pragma unroll
            for (int e = 0; e < E; ++e) v[e] = a[gaddr<COL>(kmap<ELOG>(lo, w, t, e), gi, L2, LOGS)];
        } else {
            const uint64_t *b = ((r - 1) & 1) ? buf1 : buf0;
#pragma unroll
            for (int e = 0; e < E; ++e) {
                const int k = kmap<ELOG>(lo, w, t, e);
                v[e] = COL ? b[colswz<LOGS>(k * G + g)] : b[g * S + swz<LOGS>(k)];
            }
        }
#pragma unroll
        for (int s = 0; s < w; ++s) {
            const int lp = LOGS - 1 - (lo + s);  // local stage of bit lo+s
            const int bit = ELOG - w + s;        // register bit of k-bit lo+s
            const int ntop = w - 1 - s;          // register bits above: the twiddle depends on these only
#pragma unroll
            for (int m = 0; m < (1 << ntop); ++m) {
                const int erep = m << (ELOG - ntop);
                const int krep = kmap<ELOG>(lo, w, t, erep);
                const TwPair wt = tw[(1 << (lbase + lp)) + (prefix << lp) + (krep >> (LOGS - lp))];
#pragma unroll
                for (int e = erep; e < erep + (1 << (ELOG - ntop)); ++e) {
                    if (e & (1 << bit)) continue;
                    const uint64_t X = v[e];
                    const uint64_t Y = v[e | (1 << bit)];
                    const uint64_t sum = X + Y;
                    v[e] = sum >= q2 ? sum - q2 : sum;
                    v[e | (1 << bit)] = shoup_lazy(X - Y + q2, wt.w, wt.wp, q);
                }
            }
        }
        if (r == R - 1) {
            TwPair ninv{0, 0};
            if (COL) ninv = kt.n_inv[p];
#pragma unroll
            for (int e = 0; e < E; ++e) {
                const uint64_t x = COL ? shoup(v[e], ninv.w, ninv.wp, q) : v[e];
                a[gaddr<COL>(kmap<ELOG>(lo, w, t, e), gi, L2, LOGS)] = x;
            }
        } else {
            uint64_t *b = (r & 1) ? buf1 : buf0;
#pragma unroll
            for (int e = 0; e < E; ++e) {
                const int k = kmap<ELOG>(lo, w, t, e);
                if (COL)
                    b[colswz<LOGS>(k * G + g)] = v[e];
                else
                    b[g * S + swz<LOGS>(k)] = v[e];
            }
            __syncthreads();
        }
    }
}

struct Launch {
    dim3 grid;
    int threads;
    size_t smem;
    int log_g;
};

// Groups per CTA: as many as fit kCtaThreads threads (and exist).
Launch plan(int LOGS, int ELOG, int n_groups, uint32_t rows)
{
    const int T = 1 << (LOGS - ELOG);
    int log_g = 0;
    while ((T << (log_g + 1)) <= kCtaThreads && (1 << (log_g + 1)) <= n_groups) ++log_g;
    const int G = 1 << log_g;
    Launch l;
    l.log_g = log_g;
    l.threads = T * G;
    l.grid = dim3(n_groups / G, rows);
    l.smem = (LOGS > ELOG) ? 2 * sizeof(uint64_t) * ((size_t)G << LOGS) : 0;
    return l;
}

template <bool FWD, bool COL>
void launch_pass(int LOGS, uint32_t log_n, uint64_t *d, uint32_t rows, const KTables &kt, const PrimeMap &pm,
                 cudaStream_t s)
{
    const int ELOG = LOGS < 3 ? LOGS : 3;
    const int n_groups = 1 << (log_n - LOGS);
    Launch l = plan(LOGS, ELOG, n_groups, rows);
#define MMFHE_NTT_CASE(LS, EL)                                                                    \
    case LS:                                                                                      \
        if (FWD)                                                                                  \
            ntt_fwd_pass<LS, EL, COL><<<l.grid, l.threads, l.smem, s>>>(d, kt, pm, l.log_g);      \
        else                                                                                      \
            ntt_inv_pass<LS, EL, COL><<<l.grid, l.threads, l.smem, s>>>(d, kt, pm, l.log_g);      \
        break;
    switch (LOGS) {
        MMFHE_NTT_CASE(2, 2)
        MMFHE_NTT_CASE(3, 3)
        MMFHE_NTT_CASE(4, 3)
        MMFHE_NTT_CASE(5, 3)
        MMFHE_NTT_CASE(6, 3)
        MMFHE_NTT_CASE(7, 3)
        MMFHE_NTT_CASE(8, 3)
    default:
        throw Error(MMFHE_E_PARAMS, "unsupported NTT split");
    }
#undef MMFHE_NTT_CASE
}

void split(uint32_t log_n, int &L1, int &L2)
{
    L1 = (int)log_n / 2;
    L2 = (int)log_n - L1;
}

}  // namespace

void ntt_forward(Ctx &c, uint64_t *d, uint32_t rows, const PrimeMap &pm)
{
    if (!rows) return;
    int L1, L2;
    split(c.log_n, L1, L2);
    const double bytes = 16.0 * rows * c.n;  // one read + one write of every word per pass
    {
        ProfScope ps(c, "ntt_fwd_col", bytes, 0.5 * rows * c.n * L1);
        launch_pass<true, true>(L1, c.log_n, d, rows, c.kt, pm, c.stream);
    }
    {
        ProfScope ps(c, "ntt_fwd_row", bytes, 0.5 * rows * c.n * L2);
        launch_pass<true, false>(L2, c.log_n, d, rows, c.kt, pm, c.stream);
    }
    c.launches += 2;
    CUDA_CHECK(cudaGetLastError());
}

void ntt_inverse(Ctx &c, uint64_t *d, uint32_t rows, const PrimeMap &pm)
{
    if (!rows) return;
    int L1, L2;
    split(c.log_n, L1, L2);
    const double bytes = 16.0 * rows * c.n;
    {
        ProfScope ps(c, "ntt_inv_row", bytes, 0.5 * rows * c.n * L2);
        launch_pass<false, false>(L2, c.log_n, d, rows, c.kt, pm, c.stream);
    }
    {
        ProfScope ps(c, "ntt_inv_col", bytes, 0.5 * rows * c.n * L1);
        launch_pass<false, true>(L1, c.log_n, d, rows, c.kt, pm, c.stream);
    }
    c.launches += 2;
    CUDA_CHECK(cudaGetLastError());
}

}  // namespace mmfhe
