"""Seeded synthetic radar scenes shaped like the paper's workloads, plus the
client-side preprocessing the paper puts BEFORE encryption.

Workloads (PAPER.md Table tab:dataset_config P:1096-1110):
  * vital: R range bins, F frames at fs (Children: R=64, F=200, 20 Hz);
  * gesture: A antennas x R bins x D chirps per frame, F frames at 33 Hz
    (Zenodo: A=3, R=16, D=32, F=100).
Scene recipe (SURVEY §8(d) "Concrete synthetic inputs"):
  * vital: one target at r* in [R/8, 3R/4] with +-2-bin sinc leakage; phase
    4*pi*(d_r sin 2 pi f_r t + d_h sin 2 pi f_h t)/lambda (A8),
    lambda = c/60.25 GHz; static clutter 3x the target amplitude; complex
    Gaussian noise sigma = 0.05;
  * gesture: one hand target following one of five trajectory classes (push,
    pull, swipe-left, swipe-right, circle) in (range, radial velocity,
    azimuth); chirp phase progression 4 pi v T_c / lambda; ULA lambda/2
    antenna phase; noise.
Client preprocessing (A3/A4; out of the cloud path):
clutter removal z~[t] = z[t] - mean_t z[t], then frame-local (vital) or
batch-global (gesture) normalisation to |z| <= 1.

Nothing here is cloud-side method arithmetic; the scenes only feed both sides.
"""
from __future__ import annotations

import numpy as np

C_LIGHT = 299_792_458.0


def _sinc_profile(R: int, center: float, width: int = 2) -> np.ndarray:
    r = np.arange(R)
    prof = np.sinc(r - center)
    prof[np.abs(r - center) > width + 0.5] = 0.0
    return prof


def vital_scene(R: int, F: int, fs: float, seed: int, fc_hz: float = 60.25e9):
    """Raw complex range profiles z[t, r] and the ground truth (dict)."""
    rng = np.random.default_rng(seed)
    lam = C_LIGHT / fc_hz
    r_star = int(rng.integers(R // 8, (3 * R) // 4))
    frac = rng.choice([0.0, 0.2, -0.2])  # keep frac(r_hat) away from .5
    f_r = rng.uniform(0.15, 0.5)
    d_r = rng.uniform(2e-3, 6e-3)
    f_h = rng.uniform(0.9, 2.2)
    d_h = rng.uniform(1e-4, 5e-4)
    t = np.arange(F) / fs
    phase = 4 * np.pi * (d_r * np.sin(2 * np.pi * f_r * t) + d_h * np.sin(2 * np.pi * f_h * t)) / lam
    prof = _sinc_profile(R, r_star + frac)
    target = prof[None, :] * np.exp(1j * phase)[:, None]
    clutter_bins = rng.choice(R, size=3, replace=False)
    clutter = np.zeros(R, dtype=np.complex128)
    clutter[clutter_bins] = 3.0 * np.exp(1j * rng.uniform(0, 2 * np.pi, 3))
    noise = 0.05 * (rng.normal(size=(F, R)) + 1j * rng.normal(size=(F, R))) / np.sqrt(2)
    z = target + clutter[None, :] + noise
    truth = dict(r_star=r_star + frac, f_r=f_r, f_h=f_h, d_r=d_r, d_h=d_h, fs=fs)
    return z, truth


def preprocess_vital(z: np.ndarray) -> np.ndarray:
    """Clutter removal (mean over frames) then frame-local normalisation |z| <= 1."""
    zt = z - z.mean(axis=0, keepdims=True)
    m = np.abs(zt).max(axis=1, keepdims=True)
    m[m == 0] = 1.0
    return zt / m


GESTURES = ("push", "pull", "swipe_left", "swipe_right", "circle")


def gesture_scene(A: int, R: int, D: int, F: int, seed: int, cls: int | None = None,
                  fc_hz: float = 60.5e9, frame_rate: float = 33.0, t_chirp: float = 400e-6):
    """Raw cube Z[t, a, r, c] (complex) for one gesture of class `cls`."""
    rng = np.random.default_rng(seed)
    if cls is None:
        cls = int(rng.integers(0, len(GESTURES)))
    lam = C_LIGHT / fc_hz
    bin_m = C_LIGHT / (2 * 4e9)  # 3.75 cm range bins (4 GHz bandwidth)
    tt = np.arange(F) / frame_rate
    T = F / frame_rate
    r0 = rng.uniform(0.25, 0.45) * R * bin_m
    jitter = rng.uniform(0.8, 1.2)
    name = GESTURES[cls]
    if name == "push":
        rng_m = r0 - 0.3 * R * bin_m * jitter * tt / T
        az = np.zeros(F)
    elif name == "pull":
        rng_m = r0 - 0.3 * R * bin_m * jitter * (1 - tt / T)
        az = np.zeros(F)
    elif name == "swipe_left":
        rng_m = np.full(F, r0)
        az = np.deg2rad(-40 + 80 * tt / T) * jitter
    elif name == "swipe_right":
        rng_m = np.full(F, r0)
        az = np.deg2rad(40 - 80 * tt / T) * jitter
    else:
        w = 2 * np.pi / T
        rng_m = r0 + 0.1 * R * bin_m * jitter * np.sin(w * tt)
        az = np.deg2rad(25) * np.cos(w * tt)
    vel = np.gradient(rng_m, tt)
    vmax = lam / (4 * t_chirp)
    Z = np.zeros((F, A, R, D), dtype=np.complex128)
    c = np.arange(D)
    for f in range(F):
        prof = _sinc_profile(R, rng_m[f] / bin_m)
        dop = np.exp(1j * 4 * np.pi * np.clip(vel[f], -vmax, vmax) * t_chirp * c / lam)
        for a in range(A):
            ant = np.exp(1j * np.pi * a * np.sin(az[f]))
            Z[f, a] = prof[:, None] * dop[None, :] * ant
    Z += 0.05 * (rng.normal(size=Z.shape) + 1j * rng.normal(size=Z.shape)) / np.sqrt(2)
    return Z, dict(cls=cls, name=name)


def preprocess_gesture(Z: np.ndarray) -> np.ndarray:
    """Clutter removal over frames, then batch-global normalisation |z| <= 1."""
    Zt = Z - Z.mean(axis=0, keepdims=True)
    m = np.abs(Zt).max()
    return Zt / (m if m > 0 else 1.0)


def pack_doppler(frame: np.ndarray) -> np.ndarray:
    """Doppler layout slot[a*R*D + r*D + c], length A*R*D (complex)."""
    return np.asarray(frame).reshape(-1)


def pack_vital(profile: np.ndarray, n_slots: int) -> np.ndarray:
    """Vital layout: R bins in the first R slots, zeros up to the period."""
    v = np.zeros(n_slots, dtype=np.asarray(profile).dtype)
    v[: len(profile)] = profile
    return v


def fir_taps(n_taps: int, band, fs: float) -> np.ndarray:
    """Public FIR taps: scipy firwin band-pass (SURVEY §8(c)-8 #10 reading)."""
    from scipy.signal import firwin
    return firwin(n_taps, list(band), pass_zero=False, fs=fs)


def fc_weights(dims, seed: int, scale: float = 1.0):
    """Seeded Xavier-normal weights/biases for layers dims[0]->dims[1]->...
    (synthetic stand-ins for trained weights, SURVEY §8(c)-7 FC)."""
    rng = np.random.default_rng(seed)
    Ws, bs = [], []
    for i in range(len(dims) - 1):
        fan_in, fan_out = dims[i], dims[i + 1]
        std = np.sqrt(2.0 / (fan_in + fan_out))
        Ws.append(rng.normal(0, std, size=(fan_out, fan_in)) * scale)
        bs.append(rng.normal(0, 0.01, size=fan_out))
    return Ws, bs


def vital_adc_scene(M: int, F: int, fs: float, seed: int, fc_hz: float = 60.25e9):
    """Raw complex ADC samples x[t, n] (n < M samples of one chirp per frame) of a vital scene:
    the beat tone of a target at range bin r* (exp(j 2 pi r* n / M)) carrying the same
    breathing / heartbeat phase as vital_scene, static clutter tones and noise -- the input of
    the paper's raw-ADC variant, whose range FFT (Eq. range_fft) is
    computed under encryption by the K3 kernel.  Returns (x, truth)."""
    rng = np.random.default_rng(seed)
    lam = C_LIGHT / fc_hz
    r_star = int(rng.integers(M // 8, (3 * M) // 8))
    f_r = rng.uniform(0.15, 0.5)
    d_r = rng.uniform(2e-3, 6e-3)
    f_h = rng.uniform(0.9, 2.2)
    d_h = rng.uniform(1e-4, 5e-4)
    t = np.arange(F) / fs
    n = np.arange(M)
    phase = 4 * np.pi * (d_r * np.sin(2 * np.pi * f_r * t) + d_h * np.sin(2 * np.pi * f_h * t)) / lam
    x = np.exp(1j * (2 * np.pi * r_star * n[None, :] / M + phase[:, None]))
    for rb in rng.choice(M // 2, size=3, replace=False):
        x = x + 3.0 * np.exp(1j * (2 * np.pi * rb * n[None, :] / M + rng.uniform(0, 2 * np.pi)))
    x = x + 0.05 * (rng.normal(size=(F, M)) + 1j * rng.normal(size=(F, M))) / np.sqrt(2)
    return x, dict(r_star=r_star, f_r=f_r, f_h=f_h, fs=fs)


def preprocess_adc(x: np.ndarray, peak_ratio: float = 1.0) -> np.ndarray:
    """Client preprocessing for raw ADC: clutter removal over frames (linear, so it
    commutes with the range FFT), then an O(M) Parseval-based normalisation without spectral
    computation: the spectrum's peak is estimated as peak_ratio * ||x_t|| * sum(window) /
    sqrt(M) and the frame is scaled so that the estimated peak is 1.  The paper calibrates
    |X_peak| / sqrt(sum |x_k|^2) ~ 0.74 on its gesture data; 1.0 keeps the synthetic vital
    scenes' windowed spectra at |X| <= 1 (the bound the circuit plans assume)."""
    xt = x - x.mean(axis=0, keepdims=True)
    M = x.shape[1]
    w = np.hanning(M)
    est = peak_ratio * np.sqrt(np.sum(np.abs(xt) ** 2, axis=1, keepdims=True)) * np.sum(w) / np.sqrt(M)
    est[est == 0] = 1.0
    return xt / est
