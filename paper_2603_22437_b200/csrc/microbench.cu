// microbench.cu -- the integer roofline: register-resident
// loops of exactly the arithmetic the kernels use, over the whole GPU, so that the
// NTT and base-conversion kernels can be reported against a MEASURED integer peak:
//   kind 0: Harvey CT butterfly (lazy Shoup product + lazy add/sub), as in ntt.cu
//   kind 1: Gentleman-Sande butterfly, as in the inverse NTT
//   kind 2: 64x64->128 multiply-accumulate (the key inner product / BConv MAC)
//   kind 3: Shoup modular product (fixed operand), fully reduced
//   kind 4: CT butterfly with the truncated-quotient Shoup product (shoup_lazy4, [0, 4q))
//   kind 5: GS butterfly with shoup_lazy4
#include "context.h"
#include "modarith.cuh"

namespace mmfhe {

namespace {

constexpr int kChains = 8;

__global__ void __launch_bounds__(256) mb_kernel(uint64_t *out, uint64_t q, uint64_t w0, uint64_t wp0, int iters,
                                                 int kind)
{
    const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    const uint64_t q2 = 2 * q;
    uint64_t a[kChains], b[kChains];
#pragma unroll
    for (int j = 0; j < kChains; ++j) {
        a[j] = (tid * 0x9E3779B97F4A7C15ull + j) % q;
        b[j] = (tid * 0xBF58476D1CE4E5B9ull + 3 * j) % q;
    }
    if (kind == 0) {
        for (int it = 0; it < iters; ++it) {
#pragma unroll
            for (int j = 0; j < kChains; ++j) {
                uint64_t U = a[j] >= q2 ? a[j] - q2 : a[j];
                uint64_t V = shoup_lazy(b[j], w0, wp0, q);
                a[j] = U + V;
                b[j] = U - V + q2;
            }
        }
    } else if (kind == 1) {
        for (int it = 0; it < iters; ++it) {
#pragma unroll
            for (int j = 0; j < kChains; ++j) {
                const uint64_t X = a[j], Y = b[j];
                const uint64_t s = X + Y;
                a[j] = s >= q2 ? s - q2 : s;
                b[j] = shoup_lazy(X - Y + q2, w0, wp0, q);
            }
        }
    } else if (kind == 2) {
        U128 acc[kChains];
#pragma unroll
        for (int j = 0; j < kChains; ++j) acc[j] = U128{0, 0};
        for (int it = 0; it < iters; ++it) {
#pragma unroll
            for (int j = 0; j < kChains; ++j) {
                mac128(acc[j], a[j], b[j]);
                a[j] += acc[j].hi & 1;  // dependency so the loop is not collapsed
            }
        }
#pragma unroll
        for (int j = 0; j < kChains; ++j) a[j] ^= acc[j].lo ^ acc[j].hi;
    } else if (kind == 3) {
        for (int it = 0; it < iters; ++it) {
#pragma unroll
            for (int j = 0; j < kChains; ++j) a[j] = shoup(a[j] ^ b[j], w0, wp0, q);
        }
    } else if (kind == 4) {
        const uint64_t q4 = 4 * q, q8 = 8 * q;
        for (int it = 0; it < iters; ++it) {
#pragma unroll
            for (int j = 0; j < kChains; ++j) {
                uint64_t U = a[j] >= q8 ? a[j] - q8 : a[j];
                uint64_t V = shoup_lazy4(b[j], w0, wp0, q);
                a[j] = U + V;
                b[j] = U - V + q4;
            }
        }
    } else {
        const uint64_t q4 = 4 * q;
        for (int it = 0; it < iters; ++it) {
#pragma unroll
            for (int j = 0; j < kChains; ++j) {
                const uint64_t X = a[j], Y = b[j];
                const uint64_t s = X + Y;
                a[j] = s >= q4 ? s - q4 : s;
                b[j] = shoup_lazy4(X - Y + q4, w0, wp0, q);
            }
        }
    }
    uint64_t x = 0;
#pragma unroll
    for (int j = 0; j < kChains; ++j) x ^= a[j] ^ b[j];
    out[tid] = x;
}

}  // namespace

double microbench_ops_per_s(Ctx &c, int kind)
{
    int dev, sms = 148;
    CUDA_CHECK(cudaGetDevice(&dev));
    CUDA_CHECK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    const int blocks = sms * 8, threads = 256, iters = 2048;
    const uint64_t q = c.primes[0];
    const uint64_t w = c.primes[0] / 3, wp = host::shoup(w, q);
    DBuf out((size_t)blocks * threads, c.stream);
    cudaEvent_t e0, e1;
    CUDA_CHECK(cudaEventCreate(&e0));
    CUDA_CHECK(cudaEventCreate(&e1));
    mb_kernel<<<blocks, threads, 0, c.stream>>>(out.get(), q, w, wp, 64, kind);  // warm-up
    CUDA_CHECK(cudaEventRecord(e0, c.stream));
    mb_kernel<<<blocks, threads, 0, c.stream>>>(out.get(), q, w, wp, iters, kind);
    CUDA_CHECK(cudaEventRecord(e1, c.stream));
    CUDA_CHECK(cudaEventSynchronize(e1));
    c.launches += 2;
    float ms = 0;
    CUDA_CHECK(cudaEventElapsedTime(&ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    return (double)blocks * threads * iters * kChains / (ms * 1e-3);
}

}  // namespace mmfhe
