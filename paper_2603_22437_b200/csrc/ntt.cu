// ntt.cu -- batched negacyclic NTT / INTT across RNS limbs.
//
// Forward: Cooley-Tukey, natural order in, bit-reversed order out, psi-twist
// merged into the twiddles (tw_fwd[m + i] = psi^{bitrev(m+i)}): stage l (m = 2^l)
// pairs j, j + N/2^{l+1} with twiddle index m + (j >> (log N - l)).
// Inverse: Gentleman-Sande with psi^{-bitrev}, bit-reversed in, natural out,
// times N^{-1}.  Harvey lazy butterflies: values stay in [0, 4q) (q < 2^60).
//
// B200 mapping: a limb of N = 2^16 words (512 KiB) does not fit one SM's
// shared memory, so the transform runs as two passes over HBM:
//   pass "col"  -- the first L1 stages on 2^L2 columns of 2^L1 strided words
//                  (G consecutive columns per CTA -> coalesced G*8-byte runs);
//   pass "row"  -- the last L2 stages on contiguous blocks of 2^L2 words.
// Each pass stages its tile in shared memory and runs the stages there; all
// limbs of all polynomials of a batch go in one launch (grid.y = rows).
#include <algorithm>

#include "common.h"
#include "modarith.cuh"

namespace mmfhe {

namespace {

constexpr int kTileWords = 4096;  // 32 KiB of shared memory per CTA
constexpr int kThreads = 256;

__device__ __forceinline__ uint64_t reduce4q(uint64_t x, uint64_t q)
{
    x = x >= 2 * q ? x - 2 * q : x;
    return x >= q ? x - q : x;
}

// ---------------------------------------------------------------- forward
// Columns: element (k, c) at a[(k << L2) + c], k < 2^LOGS; stages 0..LOGS-1.
template <int LOGS>
__global__ void __launch_bounds__(kThreads) ntt_fwd_col(uint64_t *__restrict__ data, KTables kt, PrimeMap pm,
                                                         int G)
{
    constexpr int S = 1 << LOGS;
    extern __shared__ uint64_t sm[];
    const int row = blockIdx.y;
    const int p = pm.idx[row % pm.period];
    const uint64_t q = kt.q[p];
    const uint64_t q2 = 2 * q;
    const TwPair *tw = kt.tw_fwd + (size_t)p * kt.n;
    uint64_t *a = data + (size_t)row * kt.n;
    const int L2 = kt.log_n - LOGS;
    const int c0 = blockIdx.x * G;
    const int tot = S * G;
    for (int e = threadIdx.x; e < tot; e += blockDim.x) {
        int k = e / G, cc = e - k * G;
        sm[e] = a[((size_t)k << L2) + c0 + cc];
    }
    __syncthreads();
#pragma unroll 1
    for (int l = 0; l < LOGS; ++l) {
        const int half = S >> (l + 1);
        for (int b = threadIdx.x; b < (S / 2) * G; b += blockDim.x) {
            int pi = b / G, cc = b - pi * G;
            int grp = pi / half, off = pi - grp * half;
            int k = grp * 2 * half + off;
            TwPair w = tw[(1 << l) + grp];
            uint64_t U = sm[k * G + cc];
            uint64_t V = sm[(k + half) * G + cc];
            U = U >= q2 ? U - q2 : U;
            V = shoup_lazy(V, w.w, w.wp, q);
            sm[k * G + cc] = U + V;
            sm[(k + half) * G + cc] = U - V + q2;
        }
        __syncthreads();
    }
    for (int e = threadIdx.x; e < tot; e += blockDim.x) {
        int k = e / G, cc = e - k * G;
        a[((size_t)k << L2) + c0 + cc] = sm[e];
    }
}

// Rows: blocks of 2^LOGS contiguous words, stages L1..logN-1; output reduced to [0, q).
template <int LOGS>
__global__ void __launch_bounds__(kThreads) ntt_fwd_row(uint64_t *__restrict__ data, KTables kt, PrimeMap pm,
                                                         int G)
{
    constexpr int S = 1 << LOGS;
    extern __shared__ uint64_t sm[];
    const int row = blockIdx.y;
    const int p = pm.idx[row % pm.period];
    const uint64_t q = kt.q[p];
    const uint64_t q2 = 2 * q;
    const TwPair *tw = kt.tw_fwd + (size_t)p * kt.n;
    const int L1 = kt.log_n - LOGS;
    const int blk0 = blockIdx.x * G;
    uint64_t *a = data + (size_t)row * kt.n + (size_t)blk0 * S;
    const int tot = S * G;
    for (int e = threadIdx.x; e < tot; e += blockDim.x) sm[e] = a[e];
    __syncthreads();
#pragma unroll 1
    for (int l = 0; l < LOGS; ++l) {
        const int half = S >> (l + 1);
        const int m = 1 << (L1 + l);
        for (int b = threadIdx.x; b < (S / 2) * G; b += blockDim.x) {
            int g = b / (S / 2), pi = b - g * (S / 2);
            int grp = pi / half, off = pi - grp * half;
            int k = g * S + grp * 2 * half + off;
            TwPair w = tw[m + ((blk0 + g) << l) + grp];
            uint64_t U = sm[k];
            uint64_t V = sm[k + half];
            U = U >= q2 ? U - q2 : U;
            V = shoup_lazy(V, w.w, w.wp, q);
            sm[k] = U + V;
            sm[k + half] = U - V + q2;
        }
        __syncthreads();
    }
    for (int e = threadIdx.x; e < tot; e += blockDim.x) a[e] = reduce4q(sm[e], q);
}

// ---------------------------------------------------------------- inverse
// Rows first: stages logN-1 .. L1 (reverse order) on contiguous blocks.
template <int LOGS>
__global__ void __launch_bounds__(kThreads) ntt_inv_row(uint64_t *__restrict__ data, KTables kt, PrimeMap pm,
                                                         int G)
{
    constexpr int S = 1 << LOGS;
    extern __shared__ uint64_t sm[];
    const int row = blockIdx.y;
    const int p = pm.idx[row % pm.period];
    const uint64_t q = kt.q[p];
    const uint64_t q2 = 2 * q;
    const TwPair *tw = kt.tw_inv + (size_t)p * kt.n;
    const int L1 = kt.log_n - LOGS;
    const int blk0 = blockIdx.x * G;
    uint64_t *a = data + (size_t)row * kt.n + (size_t)blk0 * S;
    const int tot = S * G;
    for (int e = threadIdx.x; e < tot; e += blockDim.x) sm[e] = a[e];
    __syncthreads();
#pragma unroll 1
    for (int l = LOGS - 1; l >= 0; --l) {
        const int half = S >> (l + 1);
        const int m = 1 << (L1 + l);
        for (int b = threadIdx.x; b < (S / 2) * G; b += blockDim.x) {
            int g = b / (S / 2), pi = b - g * (S / 2);
            int grp = pi / half, off = pi - grp * half;
            int k = g * S + grp * 2 * half + off;
            TwPair w = tw[m + ((blk0 + g) << l) + grp];
            uint64_t X = sm[k];
            uint64_t Y = sm[k + half];
            uint64_t s = X + Y;
            sm[k] = s >= q2 ? s - q2 : s;
            sm[k + half] = shoup_lazy(X - Y + q2, w.w, w.wp, q);
        }
        __syncthreads();
    }
    for (int e = threadIdx.x; e < tot; e += blockDim.x) a[e] = sm[e];
}

// Columns last: stages L1-1 .. 0, then times N^{-1}, output in [0, q).
template <int LOGS>
__global__ void __launch_bounds__(kThreads) ntt_inv_col(uint64_t *__restrict__ data, KTables kt, PrimeMap pm,
                                                         int G)
{
    constexpr int S = 1 << LOGS;
    extern __shared__ uint64_t sm[];
    const int row = blockIdx.y;
    const int p = pm.idx[row % pm.period];
    const uint64_t q = kt.q[p];
    const uint64_t q2 = 2 * q;
    const TwPair *tw = kt.tw_inv + (size_t)p * kt.n;
    const TwPair ninv = kt.n_inv[p];
    uint64_t *a = data + (size_t)row * kt.n;
    const int L2 = kt.log_n - LOGS;
    const int c0 = blockIdx.x * G;
    const int tot = S * G;
    for (int e = threadIdx.x; e < tot; e += blockDim.x) {
        int k = e / G, cc = e - k * G;
        sm[e] = a[((size_t)k << L2) + c0 + cc];
    }
    __syncthreads();
#pragma unroll 1
    for (int l = LOGS - 1; l >= 0; --l) {
        const int half = S >> (l + 1);
        for (int b = threadIdx.x; b < (S / 2) * G; b += blockDim.x) {
            int pi = b / G, cc = b - pi * G;
            int grp = pi / half, off = pi - grp * half;
            int k = grp * 2 * half + off;
            TwPair w = tw[(1 << l) + grp];
            uint64_t X = sm[k * G + cc];
            uint64_t Y = sm[(k + half) * G + cc];
            uint64_t s = X + Y;
            sm[k * G + cc] = s >= q2 ? s - q2 : s;
            sm[(k + half) * G + cc] = shoup_lazy(X - Y + q2, w.w, w.wp, q);
        }
        __syncthreads();
    }
    for (int e = threadIdx.x; e < tot; e += blockDim.x) {
        int k = e / G, cc = e - k * G;
        a[((size_t)k << L2) + c0 + cc] = shoup(sm[e], ninv.w, ninv.wp, q);
    }
}

#define MMFHE_NTT_DISPATCH(FN)                                                                    \
    template <int LOGS>                                                                           \
    struct FN##_k {                                                                               \
        static void run(dim3 g, size_t smem, cudaStream_t s, uint64_t *d, const KTables &kt,      \
                        const PrimeMap &pm, int G)                                                \
        {                                                                                         \
            FN<LOGS><<<g, kThreads, smem, s>>>(d, kt, pm, G);                                     \
        }                                                                                         \
    };

MMFHE_NTT_DISPATCH(ntt_fwd_col)
MMFHE_NTT_DISPATCH(ntt_fwd_row)
MMFHE_NTT_DISPATCH(ntt_inv_col)
MMFHE_NTT_DISPATCH(ntt_inv_row)

template <template <int> class K>
void launch_logs(int logs, dim3 g, size_t smem, cudaStream_t s, uint64_t *d, const KTables &kt,
                 const PrimeMap &pm, int G)
{
    switch (logs) {
    case 1: K<1>::run(g, smem, s, d, kt, pm, G); break;
    case 2: K<2>::run(g, smem, s, d, kt, pm, G); break;
    case 3: K<3>::run(g, smem, s, d, kt, pm, G); break;
    case 4: K<4>::run(g, smem, s, d, kt, pm, G); break;
    case 5: K<5>::run(g, smem, s, d, kt, pm, G); break;
    case 6: K<6>::run(g, smem, s, d, kt, pm, G); break;
    case 7: K<7>::run(g, smem, s, d, kt, pm, G); break;
    case 8: K<8>::run(g, smem, s, d, kt, pm, G); break;
    default: throw Error(MMFHE_E_PARAMS, "unsupported NTT split");
    }
}

void split(uint32_t log_n, int &L1, int &L2)
{
    L1 = (int)log_n / 2;
    L2 = (int)log_n - L1;
}

}  // namespace

void ntt_forward(const KTables &kt, uint64_t *d, uint32_t rows, const PrimeMap &pm, cudaStream_t s,
                 uint64_t &launches)
{
    if (!rows) return;
    int L1, L2;
    split(kt.log_n, L1, L2);
    int S1 = 1 << L1, S2 = 1 << L2;
    int G1 = std::max(1, std::min(kTileWords / S1, S2));
    int G2 = std::max(1, std::min(kTileWords / S2, S1));
    launch_logs<ntt_fwd_col_k>(L1, dim3(S2 / G1, rows), (size_t)S1 * G1 * 8, s, d, kt, pm, G1);
    launch_logs<ntt_fwd_row_k>(L2, dim3(S1 / G2, rows), (size_t)S2 * G2 * 8, s, d, kt, pm, G2);
    launches += 2;
    CUDA_CHECK(cudaGetLastError());
}

void ntt_inverse(const KTables &kt, uint64_t *d, uint32_t rows, const PrimeMap &pm, cudaStream_t s,
                 uint64_t &launches)
{
    if (!rows) return;
    int L1, L2;
    split(kt.log_n, L1, L2);
    int S1 = 1 << L1, S2 = 1 << L2;
    int G1 = std::max(1, std::min(kTileWords / S1, S2));
    int G2 = std::max(1, std::min(kTileWords / S2, S1));
    launch_logs<ntt_inv_row_k>(L2, dim3(S1 / G2, rows), (size_t)S2 * G2 * 8, s, d, kt, pm, G2);
    launch_logs<ntt_inv_col_k>(L1, dim3(S2 / G1, rows), (size_t)S1 * G1 * 8, s, d, kt, pm, G1);
    launches += 2;
    CUDA_CHECK(cudaGetLastError());
}

}  // namespace mmfhe
