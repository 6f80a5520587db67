// encoder.cpp -- the library's own CKKS encoder (setup-time, host): canonical
// embedding with slot j <-> zeta^(5^j mod 2N), zeta = e^(i pi / N) (P:397-402,
// "packs up to N/2 real values"; complex slot values for DESIGN R28); period-n vectors are replicated to N/2
// slots (sparse packing).  Used by mmfhe_encode_plain and
// mmfhe_prepare_chain; parity tests import the oracle's encodings instead
// (floating-point encodings are not bit-reproducible across implementations,
// SURVEY §8(c)-5).
#include <cmath>
#include <complex>

#include "eval.h"

namespace mmfhe {

namespace {
typedef std::complex<double> cd;

// in-place iterative radix-2 DFT, X_k = sum_i x_i e^{sign * 2 pi i ik / n}
void fft(std::vector<cd> &a, int sign)
{
    const size_t n = a.size();
    for (size_t i = 1, j = 0; i < n; ++i) {
        size_t bit = n >> 1;
        for (; j & bit; bit >>= 1) j ^= bit;
        j ^= bit;
        if (i < j) std::swap(a[i], a[j]);
    }
    for (size_t len = 2; len <= n; len <<= 1) {
        const double ang = sign * 2 * M_PI / (double)len;
        for (size_t i = 0; i < n; i += len)
            for (size_t j = 0; j < len / 2; ++j) {
                cd w = std::polar(1.0, ang * (double)j);
                cd u = a[i + j], v = a[i + j + len / 2] * w;
                a[i + j] = u + v;
                a[i + j + len / 2] = u - v;
            }
    }
}
}  // namespace

// m with m(zeta^(5^j)) = z_j and m(zeta^(-5^j)) = conj z_j: real coefficients for any complex
// slot vector (DESIGN R28); a real vector is the special case z = conj z.
std::vector<int64_t> encode_slots(const Ctx &c, const std::vector<cd> &v, double scale)
{
    const uint32_t n = c.n, half = n / 2;
    MMFHE_REQUIRE(!v.empty() && half % v.size() == 0, MMFHE_E_LAYOUT, "packing period must divide N/2");
    std::vector<cd> E(n, cd(0, 0));
    uint64_t e = 1;
    for (uint32_t j = 0; j < half; ++j) {
        const cd z = v[j % v.size()];
        E[(e - 1) / 2] = z;
        E[(2ull * n - e - 1) / 2] = std::conj(z);
        e = e * 5 % (2ull * n);
    }
    fft(E, -1);  // b_i = sum_k E_k e^{-2 pi i ik/N}
    std::vector<int64_t> m(n);
    for (uint32_t i = 0; i < n; ++i) {
        cd b = E[i] / (double)n * std::polar(1.0, -M_PI * (double)i / (double)n);
        const double x = b.real() * scale;
        MMFHE_REQUIRE(std::fabs(x) < 4.6e18, MMFHE_E_SCALE, "encoding overflow");
        m[i] = (int64_t)std::llround(x);
    }
    return m;
}

std::vector<int64_t> encode_real(const Ctx &c, const std::vector<double> &v, double scale)
{
    return encode_slots(c, std::vector<cd>(v.begin(), v.end()), scale);
}

namespace {
void store_encoded(Ctx &c, const std::string &name, const std::vector<int64_t> &m, uint32_t level, double scale,
                   bool pq)
{
    std::vector<uint32_t> basis = pq ? c.ext_basis(level) : c.q_basis(level);
    std::vector<uint64_t> res(basis.size() * c.n);
    for (size_t i = 0; i < basis.size(); ++i) {
        const int64_t q = (int64_t)c.primes[basis[i]];
        for (uint32_t k = 0; k < c.n; ++k) {
            int64_t r = m[k] % q;
            res[i * c.n + k] = (uint64_t)(r < 0 ? r + q : r);
        }
    }
    load_plain(c, name, level, scale, res.data(), false, pq);
    CUDA_CHECK(cudaStreamSynchronize(c.stream));
}
}  // namespace

void encode_plain(Ctx &c, const std::string &name, const std::vector<double> &v, uint32_t level, double scale,
                  bool pq)
{
    MMFHE_REQUIRE(level <= c.L, MMFHE_E_DEPTH, "plaintext level above the chain");
    store_encoded(c, name, encode_real(c, v, scale), level, scale, pq);
}

void encode_plain_c(Ctx &c, const std::string &name, const std::vector<cd> &v, uint32_t level, double scale,
                    bool pq)
{
    MMFHE_REQUIRE(level <= c.L, MMFHE_E_DEPTH, "plaintext level above the chain");
    store_encoded(c, name, encode_slots(c, v, scale), level, scale, pq);
}

}  // namespace mmfhe
