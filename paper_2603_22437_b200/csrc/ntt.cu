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
//   row pass -- stages L1..logN-1 on contiguous blocks of 2^L2 words; lanes
//               of a group on consecutive words.
// Inside a pass each thread holds E = 2^ELOG = 8 words in registers (radix-8)
// and runs up to ELOG butterfly stages there per round; rounds exchange through double-buffered, XOR-swizzled shared memory
// (one __syncthreads per exchange, bank-conflict-free).  Forward rounds put the
// narrow round FIRST (top bits) and inverse rounds LAST, so that in every round a
// stage's twiddle depends only on register bits above it: each distinct twiddle
// is loaded once per stage.  All index math is compile-time shifts and masks.
// Every limb of every polynomial of a batch goes in one launch (grid.y = rows).
#include <algorithm>

#include "context.h"
#include "modarith.cuh"

namespace mmfhe {

namespace {

constexpr int kCtaThreads = 256;
// min CTAs/SM for __launch_bounds__: forcing 5 (<= 51 registers) spilled and ran slower
constexpr int kMinCtas = 1;

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

// XOR swizzle of a shared-memory word index: low bit b ^= parity((x >> 4) & M_b).
// Masks found by exhaustive bank simulation of every round's lane pattern (both
// directions); identity where the plain layout is already conflict-free.
template <int M0, int M1, int M2, int M3>
__device__ __forceinline__ int pswz(int x)
{
    const int h = x >> 4;
    return x ^ ((__popc(h & M0) & 1) | ((__popc(h & M1) & 1) << 1) | ((__popc(h & M2) & 1) << 2) |
                ((__popc(h & M3) & 1) << 3));
}

template <int LOGS, int ELOG, bool COL>
__device__ __forceinline__ int swz(int x)
{
    if (!COL && LOGS == 8 && ELOG == 4) return pswz<4, 2, 3, 14>(x);
    if (!COL && LOGS == 8 && ELOG == 3) return pswz<7, 11, 13, 6>(x);
    if (!COL && LOGS == 7 && ELOG == 3) return pswz<3, 1, 7, 4>(x);
    if (!COL && LOGS == 6 && ELOG == 3) return pswz<1, 2, 1, 1>(x);
    if (COL && LOGS == 8 && ELOG == 3) return pswz<49, 27, 49, 6>(x);
    return x;
}

// Global word offset (within the row) of local element k of group gi.
template <bool COL>
__device__ __forceinline__ size_t gaddr(int k, int gi, int L2, int LOGS)
{
    return COL ? (((size_t)k << L2) + gi) : (((size_t)gi << LOGS) + k);
}

template <int LOGS, int ELOG, bool COL>
__device__ __forceinline__ int smem_index(int k, int g, int G)
{
    return COL ? swz<LOGS, ELOG, true>(k * G + g) : g * (1 << LOGS) + swz<LOGS, ELOG, false>(k);
}

// ---------------------------------------------------------------- forward
// Round widths: the first (top) round takes LOGS - (R-1)*ELOG bits, the others ELOG.
template <int LOGS, int ELOG, bool COL>
__global__ void __launch_bounds__(kCtaThreads, kMinCtas) ntt_fwd_pass(uint64_t *__restrict__ data, KTables kt, PrimeMap pm,
                                                            int log_g)
{
    constexpr int S = 1 << LOGS, E = 1 << ELOG, T = S >> ELOG, R = (LOGS + ELOG - 1) / ELOG;
    constexpr int W0 = LOGS - (R - 1) * ELOG;
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
        const int w = r == 0 ? W0 : ELOG;
        const int hi = LOGS - 1 - (r == 0 ? 0 : W0 + (r - 1) * ELOG);
        const int lo = hi - w + 1;
        const int lp0 = LOGS - 1 - hi;  // local stage of this round's first stage
        if (r == 0 && !COL) {
            // row pass: the CTA's G blocks are one contiguous tile -- load it coalesced
            // into shared memory, then read the round's register pattern from there
            const uint64_t *tile = data + (size_t)row * kt.n + ((size_t)blockIdx.x * G << LOGS);
#pragma unroll
            for (int i = 0; i < E; ++i) {
                const int idx = tid + i * (T << log_g);
                buf1[smem_index<LOGS, ELOG, false>(idx & (S - 1), idx >> LOGS, G)] = tile[idx];
            }
            __syncthreads();
#pragma unroll
            for (int e = 0; e < E; ++e) v[e] = buf1[smem_index<LOGS, ELOG, false>(kmap<ELOG>(lo, w, t, e), g, G)];
        } else if (r == 0) {
#pragma unroll
            for (int e = 0; e < E; ++e) v[e] = a[gaddr<COL>(kmap<ELOG>(lo, w, t, e), gi, L2, LOGS)];
        } else {
            const uint64_t *b = ((r - 1) & 1) ? buf1 : buf0;
#pragma unroll
            for (int e = 0; e < E; ++e) v[e] = b[smem_index<LOGS, ELOG, COL>(kmap<ELOG>(lo, w, t, e), g, G)];
        }
        // The twiddle of stage s depends only on the top s register bits (spare register
        // bits map below lo): 2^s distinct ones per stage.  Issue all of the round's
        // twiddle loads before the first butterfly so their L2 latency overlaps.
        TwPair tws[E];
#pragma unroll
        for (int s = 0; s < w; ++s) {
            const int lp = lp0 + s;
#pragma unroll
            for (int mm = 0; mm < (1 << s); ++mm) {
                const int krep = kmap<ELOG>(lo, w, t, mm << (ELOG - s));
                tws[(1 << s) - 1 + mm] = tw[(1 << (lbase + lp)) + (prefix << lp) + (krep >> (LOGS - lp))];
            }
        }
#pragma unroll
        for (int s = 0; s < w; ++s) {
            const int bit = ELOG - 1 - s;  // register bit paired in this stage
#pragma unroll
            for (int mm = 0; mm < (1 << s); ++mm) {
                const int erep = mm << (ELOG - s);
                const TwPair wt = tws[(1 << s) - 1 + mm];
#pragma unroll
                for (int e = erep; e < erep + (1 << (ELOG - s)); ++e) {
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
        if (r == R - 1 && !COL) {
            // row pass: through shared memory back to a coalesced store of the tile
            uint64_t *b = (r & 1) ? buf1 : buf0;
#pragma unroll
            for (int e = 0; e < E; ++e) b[smem_index<LOGS, ELOG, false>(kmap<ELOG>(lo, w, t, e), g, G)] = reduce4q(v[e], q);
            __syncthreads();
            uint64_t *tile = data + (size_t)row * kt.n + ((size_t)blockIdx.x * G << LOGS);
#pragma unroll
            for (int i = 0; i < E; ++i) {
                const int idx = tid + i * (T << log_g);
                tile[idx] = b[smem_index<LOGS, ELOG, false>(idx & (S - 1), idx >> LOGS, G)];
            }
        } else if (r == R - 1) {
#pragma unroll
            for (int e = 0; e < E; ++e) a[gaddr<COL>(kmap<ELOG>(lo, w, t, e), gi, L2, LOGS)] = v[e];
        } else {
            uint64_t *b = (r & 1) ? buf1 : buf0;
#pragma unroll
            for (int e = 0; e < E; ++e) b[smem_index<LOGS, ELOG, COL>(kmap<ELOG>(lo, w, t, e), g, G)] = v[e];
            __syncthreads();
        }
    }
}

// ---------------------------------------------------------------- inverse
// Stages in reverse: local stage lp = LOGS-1 .. 0 operates on bit LOGS-1-lp, so
// rounds own bits from the bottom up (the narrow round last, at the top).  The
// col pass (last) multiplies by N^{-1}.
template <int LOGS, int ELOG, bool COL>
__global__ void __launch_bounds__(kCtaThreads, kMinCtas) ntt_inv_pass(uint64_t *__restrict__ data, KTables kt, PrimeMap pm,
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
        if (r == 0 && !COL) {
            // row pass: coalesced load of the CTA's contiguous tile through shared memory
            const uint64_t *tile = data + (size_t)row * kt.n + ((size_t)blockIdx.x * G << LOGS);
#pragma unroll
            for (int i = 0; i < E; ++i) {
                const int idx = tid + i * (T << log_g);
                buf1[smem_index<LOGS, ELOG, false>(idx & (S - 1), idx >> LOGS, G)] = tile[idx];
            }
            __syncthreads();
#pragma unroll
            for (int e = 0; e < E; ++e) v[e] = buf1[smem_index<LOGS, ELOG, false>(kmap<ELOG>(lo, w, t, e), g, G)];
        } else if (r == 0) {
#pragma unroll
            for (int e = 0; e < E; ++e) v[e] = a[gaddr<COL>(kmap<ELOG>(lo, w, t, e), gi, L2, LOGS)];
        } else {
            const uint64_t *b = ((r - 1) & 1) ? buf1 : buf0;
#pragma unroll
            for (int e = 0; e < E; ++e) v[e] = b[smem_index<LOGS, ELOG, COL>(kmap<ELOG>(lo, w, t, e), g, G)];
        }
        // stage s needs 2^(w-1-s) distinct twiddles (register bits above it); load the
        // whole round's set up front
        TwPair tws[E];
#pragma unroll
        for (int s = 0; s < w; ++s) {
            const int lp = LOGS - 1 - (lo + s);
            const int ntop = w - 1 - s;
#pragma unroll
            for (int mm = 0; mm < (1 << ntop); ++mm) {
                const int krep = kmap<ELOG>(lo, w, t, mm << (ELOG - ntop));
                tws[(1 << ntop) - 1 + mm] = tw[(1 << (lbase + lp)) + (prefix << lp) + (krep >> (LOGS - lp))];
            }
        }
#pragma unroll
        for (int s = 0; s < w; ++s) {
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
                    const uint64_t sum = X + Y;
                    v[e] = sum >= q2 ? sum - q2 : sum;
                    v[e | (1 << bit)] = shoup_lazy(X - Y + q2, wt.w, wt.wp, q);
                }
            }
        }
        if (r == R - 1 && !COL) {
            // row pass: through shared memory back to a coalesced store of the tile
            uint64_t *b = (r & 1) ? buf1 : buf0;
#pragma unroll
            for (int e = 0; e < E; ++e) b[smem_index<LOGS, ELOG, false>(kmap<ELOG>(lo, w, t, e), g, G)] = v[e];
            __syncthreads();
            uint64_t *tile = data + (size_t)row * kt.n + ((size_t)blockIdx.x * G << LOGS);
#pragma unroll
            for (int i = 0; i < E; ++i) {
                const int idx = tid + i * (T << log_g);
                tile[idx] = b[smem_index<LOGS, ELOG, false>(idx & (S - 1), idx >> LOGS, G)];
            }
        } else if (r == R - 1) {
            const TwPair ninv = kt.n_inv[p];
#pragma unroll
            for (int e = 0; e < E; ++e) a[gaddr<COL>(kmap<ELOG>(lo, w, t, e), gi, L2, LOGS)] = shoup(v[e], ninv.w, ninv.wp, q);
        } else {
            uint64_t *b = (r & 1) ? buf1 : buf0;
#pragma unroll
            for (int e = 0; e < E; ++e) b[smem_index<LOGS, ELOG, COL>(kmap<ELOG>(lo, w, t, e), g, G)] = v[e];
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
    l.smem = 2 * sizeof(uint64_t) * ((size_t)G << LOGS);  // exchanges + the row pass's I/O staging
    return l;
}

// Radix-8 everywhere: radix-16 (ELOG = 4) halves the exchanges but its 64 KiB CTAs and
// 16 live words per thread halved occupancy and ran 2x slower on B200 (measured).
int elog_for(int LOGS) { return LOGS < 3 ? LOGS : 3; }

template <bool FWD, bool COL>
void launch_pass(int LOGS, uint32_t log_n, uint64_t *d, uint32_t rows, const KTables &kt, const PrimeMap &pm,
                 cudaStream_t s)
{
    const int ELOG = elog_for(LOGS);
    const int n_groups = 1 << (log_n - LOGS);
    Launch l = plan(LOGS, ELOG, n_groups, rows);
    // > 48 KiB of dynamic shared memory (radix-16 passes) needs an explicit opt-in, once
#define MMFHE_NTT_CASE(LS, EL)                                                                    \
    case LS: {                                                                                    \
        auto kern = FWD ? ntt_fwd_pass<LS, EL, COL> : ntt_inv_pass<LS, EL, COL>;                  \
        static bool attr_set = false;                                                             \
        if (!attr_set) {                                                                          \
            CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,    \
                                            96 * 1024));                                          \
            attr_set = true;                                                                      \
        }                                                                                         \
        kern<<<l.grid, l.threads, l.smem, s>>>(d, kt, pm, l.log_g);                               \
        break;                                                                                    \
    }
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
