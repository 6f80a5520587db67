"""O-DSP: the paper's closed forms in numpy float64 -- TEST INFRASTRUCTURE ONLY.

Each function is the plaintext definition the decrypted output of a kernel
approximates, with the same public normalisation constants
folded in as the encrypted circuits (readings in DESIGN.md §3), so the two
can be compared at 1e-3 relative (north_star gate 2).
"""
from __future__ import annotations

import numpy as np


def energy(z: np.ndarray) -> np.ndarray:
    """Eq. energy: E_r = sum_t Re(z_r[t])^2 + Im(z_r[t])^2; z is [F][R]."""
    return np.sum(z.real ** 2 + z.imag ** 2, axis=0)


def soft_attention(E: np.ndarray, gamma: int, F: int):
    """Eqs. soft_power_weight / soft_argmax_stats with the overflow
    fold 1/(F^2 R) of SURVEY §8(c)-7 K2a (r_hat = N/D is unchanged)."""
    R = len(E)
    w = E ** gamma
    r = np.arange(R)
    N = np.sum(r * w) / (F * F * R)
    D = np.sum(w) / (F * F * R)
    return N, D, N / D


def hann(D: int) -> np.ndarray:
    """Symmetric Hanning window (np.hanning), SURVEY §8(c)-8 #11."""
    return np.hanning(D)


def dft_matrix(D: int) -> np.ndarray:
    """Eq. dft_kernel: W_{d,n} = w[n] exp(-j 2 pi sigma(d) n / D),
    sigma(d) = (d + D/2) mod D (fftshift)."""
    w = hann(D)
    d = np.arange(D)
    sig = (d + D // 2) % D
    n = np.arange(D)
    return w[None, :] * np.exp(-2j * np.pi * np.outer(sig, n) / D)


def doppler_dft(v: np.ndarray, D: int) -> np.ndarray:
    """Eq. dft_re/dft_im: d = (I_AR (x) W) v on the Doppler layout."""
    W = dft_matrix(D)
    blocks = v.reshape(-1, D)
    return (blocks @ W.T).reshape(-1)


def power(d: np.ndarray) -> np.ndarray:
    return d.real ** 2 + d.imag ** 2


def notch_mask(D: int, width: int = 1) -> np.ndarray:
    """Eq. notch_mask, reading #3: zero bin D/2 (zero Doppler after fftshift)."""
    m = np.ones(D)
    lo = D // 2 - (width - 1) // 2
    m[lo: lo + width] = 0.0
    return m


def spectral_scale(R: int, A: int, D: int) -> float:
    """s = R * A * (sum_n w[n])^2."""
    return R * A * float(np.sum(hann(D))) ** 2


def gesture_frame_features(v: np.ndarray, A: int, R: int, D: int, gamma: int = 4) -> np.ndarray:
    """K3 -> |.|^2 -> K6 (with the 1/s fold) -> Eq. gesture_soft_power
    -> weighting f = P_masked * S^gamma, on the Doppler layout (length A*R*D)."""
    d = doppler_dft(v, D)
    P = power(d)
    s = spectral_scale(R, A, D)
    Pm = P * np.tile(notch_mask(D), A * R) / s
    S = Pm.reshape(A * R, D).sum(axis=0)        # S[d] = sum_{a,r} Pm[a,r,d]
    Sg = S ** gamma
    return Pm * np.tile(Sg, A * R)


def mlp_forward(x: np.ndarray, Ws, bs) -> np.ndarray:
    """Eq. mlp_forward: square activation on every layer but the last."""
    h = x
    for i, (W, b) in enumerate(zip(Ws, bs)):
        h = W @ h + b
        if i < len(Ws) - 1:
            h = h * h
    return h


def soft_iq(z_t: np.ndarray, p_phi: int):
    """Eqs. phase_mask / phase_iq for one frame z_t[r]."""
    m = (z_t.real ** 2 + z_t.imag ** 2) ** p_phi
    return np.sum(m * z_t.real), np.sum(m * z_t.imag)


def fir(x: np.ndarray, h: np.ndarray) -> np.ndarray:
    """Eq. fir_iq: Toeplitz T x = causal convolution, zero initial state."""
    from scipy.signal import lfilter
    return lfilter(h, 1.0, x)


def taylor_phase(I: np.ndarray, Q: np.ndarray, order: int) -> np.ndarray:
    """Eq. taylor_arctan, the literal polynomial (reading #2)."""
    y = Q[1:] * I[:-1] - I[1:] * Q[:-1]
    if order == 1:
        return y
    x = I[1:] * I[:-1] + Q[1:] * Q[:-1]
    return y * x * x - y ** 3 / 3.0


def band_bins(F_phase: int, fs: float, band) -> np.ndarray:
    """Bins k with f_k = k fs / F_phase inside [band]; F_phase = F - 1 (reading #24)."""
    k = np.arange(F_phase // 2 + 1)
    f = k * fs / F_phase
    return k[(f >= band[0]) & (f <= band[1])]


def narrowband_dft_coefs(F_phase: int, k: int):
    """c_{k,t}, s_{k,t} of X[k] = sum_t w[t] y[t] e^{-j 2 pi k t / F_phase} / F_phase
    (reading #25 folds 1/(F-1)); returns (real, imag) coefficient vectors."""
    w = np.hanning(F_phase)
    t = np.arange(F_phase)
    ang = 2 * np.pi * k * t / F_phase
    return w * np.cos(ang) / F_phase, -w * np.sin(ang) / F_phase


def narrowband_power(y: np.ndarray, bins) -> np.ndarray:
    out = []
    for k in bins:
        c, s = narrowband_dft_coefs(len(y), int(k))
        out.append(np.dot(c, y) ** 2 + np.dot(s, y) ** 2)
    return np.array(out)


def weighted_average(P: np.ndarray, bins, fs: float, F_phase: int):
    """VP+ sums: N_f = sum_k f_k P_k^2, D_f = sum_k P_k^2, f_k = k fs / F_phase."""
    f = np.asarray(bins, dtype=np.float64) * fs / F_phase
    w = np.asarray(P, dtype=np.float64) ** 2
    return float(np.sum(f * w)), float(np.sum(w))


def bpm_from_power(P: np.ndarray, bins, fs: float, F_phase: int) -> float:
    """Client: sharpen (P_k^2) and weighted frequency average -> BPM."""
    f = np.asarray(bins) * fs / F_phase
    w = P ** 2
    return 60.0 * float(np.sum(f * w) / np.sum(w))
