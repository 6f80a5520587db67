// common.h -- shared host/device declarations of the mmFHE CUDA library.
#pragma once
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/mmfhe.h"

namespace mmfhe {

// ---------------------------------------------------------------- errors
struct Error : std::runtime_error {
    mmfhe_status status;
    Error(mmfhe_status s, const std::string &m) : std::runtime_error(m), status(s) {}
};

#define MMFHE_REQUIRE(cond, status, msg)                                                          \
    do {                                                                                          \
        if (!(cond)) throw ::mmfhe::Error((status), (msg));                                       \
    } while (0)

#define CUDA_CHECK(expr)                                                                          \
    do {                                                                                          \
        cudaError_t e_ = (expr);                                                                  \
        if (e_ != cudaSuccess)                                                                    \
            throw ::mmfhe::Error(e_ == cudaErrorMemoryAllocation ? MMFHE_E_OOM : MMFHE_E_CUDA,    \
                                 std::string(#expr) + ": " + cudaGetErrorString(e_));             \
    } while (0)

// cudaFuncSetAttribute applies to the current device only: run fn once per device (the
// attribute set is idempotent, so a concurrent first call on two threads is harmless).
template <class F>
void once_per_device(std::atomic<uint64_t> &done, F &&fn)
{
    int dev = 0;
    CUDA_CHECK(cudaGetDevice(&dev));
    const uint64_t bit = 1ull << (dev & 63);
    if (done.load(std::memory_order_acquire) & bit) return;
    fn();
    done.fetch_or(bit, std::memory_order_acq_rel);
}

// Makes `device` current for the scope of one C-ABI call (kernels launch on the ctx's
// stream, which belongs to that device) and restores the caller's device afterwards.
struct DeviceScope {
    explicit DeviceScope(int device)
    {
        if (device < 0 || cudaGetDevice(&saved_) != cudaSuccess || saved_ == device) {
            saved_ = -1;
            return;
        }
        CUDA_CHECK(cudaSetDevice(device));
    }
    ~DeviceScope()
    {
        if (saved_ >= 0) cudaSetDevice(saved_);
    }
    DeviceScope(const DeviceScope &) = delete;
    DeviceScope &operator=(const DeviceScope &) = delete;

  private:
    int saved_ = -1;
};

// ---------------------------------------------------------------- host modular math
// (own implementation; the oracle's is separate and never linked)
namespace host {
typedef unsigned __int128 u128;
inline uint64_t mul(uint64_t a, uint64_t b, uint64_t q) { return (uint64_t)((u128)a * b % q); }
inline uint64_t add(uint64_t a, uint64_t b, uint64_t q) { uint64_t s = a + b; return s >= q ? s - q : s; }
inline uint64_t sub(uint64_t a, uint64_t b, uint64_t q) { return a >= b ? a - b : a + q - b; }
inline uint64_t pow(uint64_t b, uint64_t e, uint64_t q)
{
    uint64_t r = 1 % q;
    b %= q;
    while (e) {
        if (e & 1) r = mul(r, b, q);
        b = mul(b, b, q);
        e >>= 1;
    }
    return r;
}
inline uint64_t inv(uint64_t a, uint64_t q) { return pow(a % q, q - 2, q); }
inline uint64_t shoup(uint64_t w, uint64_t q) { return (uint64_t)(((u128)w << 64) / q); }
// -q^{-1} mod 2^64 by Newton iteration
inline uint64_t qinv_neg(uint64_t q)
{
    uint64_t x = q;  // correct to 3 bits for odd q
    for (int i = 0; i < 6; ++i) x *= 2 - q * x;
    return (uint64_t)0 - x;
}
inline uint64_t to_mont(uint64_t a, uint64_t q) { return (uint64_t)((((u128)(a % q)) << 64) % q); }
bool is_prime(uint64_t n);
}  // namespace host

// ---------------------------------------------------------------- device-side tables
struct TwPair {
    uint64_t w, wp;  // value and Shoup companion floor(w 2^64 / q)
};

struct KTables {
    const uint64_t *q;         // [np]
    const uint64_t *qinv_neg;  // [np]
    const uint64_t *r2;        // [np] 2^128 mod q
    const TwPair *tw_fwd;      // [np][N]  psi^{bitrev(k)}
    const TwPair *tw_inv;      // [np][N]  psi^{-bitrev(k)}
    const TwPair *n_inv;       // [np]
    const TwPair *n_inv_w;     // [np] N^{-1} tw_inv[1]: the inverse's last stage with N^{-1} folded in
    const uint64_t *recip;     // [np] floor(2^64 / q): shoup_lazy(x, 1, recip, q) = x mod q in [0, 2q)
    uint32_t log_n;
    uint32_t n;
};

// row r of a batch uses prime idx[r % period] (indices into q_0..q_L, p_0..p_{K-1})
constexpr int kMapCap = 256;
struct PrimeMap {
    uint8_t idx[kMapCap];
    uint32_t period;
};

// Optional source of the forward NTT's col pass: row r reads
// x + (r / period) * xs + src[r % period] * N and reduces it into [0, 2q) on load.
// ModUp of single-limb digits (alpha = 1) is exactly y = x_j mod q_t,
// so the base conversion fuses into the transform's first HBM read.  With sub != nullptr
// the loaded word is fully reduced and sub[p] (p = the row's prime index) is subtracted
// mod q: the rescale's ([t]_{q_i} - [h]_{q_i}) mod q_i.
struct ColSrc {
    const uint64_t *x;    // nullptr: the pass transforms its own rows
    size_t xs;            // item stride of x (words)
    uint32_t period;      // == the PrimeMap period
    const uint64_t *sub;  // optional per-prime subtrahend (canonical), indexed by prime
    uint8_t src[kMapCap];
    // bit r % period set: the source words are canonical residues of a prime q_s < 2q for the
    // row's prime q, hence already < 2q: the load skips the reduction (sub == nullptr only)
    uint32_t below2q[kMapCap / 32];
};

// Optional source of the inverse NTT's row pass (its first pass): output row r reads
// x + (r / per) * xs + (r % per) * ss instead of transforming in place, and with g != 1
// reads it through the NTT-domain automorphism sigma_g (word j <- word perm_g(j),
// perm_g(j) = bitrev(((2 bitrev(j) + 1) g mod 2N - 1) / 2)): the rotation's permutation
// and the key switch's INTT are one pass over HBM.
struct InvSrc {
    const uint64_t *x;  // nullptr: in place
    size_t xs, ss;      // item stride, sub-row stride (words)
    uint32_t per;       // rows per item
    uint32_t g;         // Galois element (odd, < 2N); 1 = identity
    uint32_t add_half;  // 1: the col pass adds floor(q/2) mod q to every output (rescale's rounding offset)
};

// Optional epilogue of the forward NTT's row pass (its last pass): instead of storing the
// transform v of row r = (item b, poly, limb i) (rows per item = 2 * per), it stores
//   out[b os + poly ops + i N] = (X[b xs + poly xps + i N] - v) mul[i] mod q_i
//                               (+ add0[b as + i N + perm_g0(k)] + add2[b as + i N + k] on poly 0,
//                                + add1[b as + i N + k] on poly 1),
// which is ModDown's final step (X = accQ, mul = P^{-1}) and the rescale's (X = a,
// mul = q_l^{-1}): the transform's output never goes to HBM.
struct RowEpi {
    uint64_t *out;                       // nullptr: no epilogue
    const uint64_t *X;
    const TwPair *mul;                   // [per] Shoup pairs, indexed by i
    const uint64_t *add0, *add1, *add2;  // each may be null
    size_t os, ops, xs, xps, as;
    uint32_t per, g0;
    uint32_t npoly;  // polynomials per item (0 is read as 2)
};

inline PrimeMap make_map(const std::vector<uint32_t> &v)
{
    PrimeMap m;
    MMFHE_REQUIRE(!v.empty() && v.size() <= (size_t)kMapCap, MMFHE_E_LAYOUT, "prime map size");
    m.period = (uint32_t)v.size();
    for (size_t i = 0; i < (size_t)kMapCap; ++i) m.idx[i] = i < v.size() ? (uint8_t)v[i] : 0;
    return m;
}

}  // namespace mmfhe
