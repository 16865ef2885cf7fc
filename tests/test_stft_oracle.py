"""Pins of the STFT front end / resynthesis oracle (oracle/stft_oracle.c) against
things other than itself: numpy.fft of the same windowed frames, the analytic DFT of a bin-centred
sinusoid and of a constant, Parseval, the inverse relation (istft(stft(x)) = x where the window covers
x), and the masking identities of S:429-431."""
import numpy as np
import pytest


def hann(L):
    return 0.5 - 0.5 * np.cos(2 * np.pi * np.arange(L) / L)


@pytest.mark.parametrize("L,H,n", [(64, 16, 300), (32, 8, 32), (128, 32, 1000)])
def test_stft_equals_numpy_fft_of_windowed_frames(oracle, L, H, n):
    rng = np.random.default_rng(L + n)
    x = rng.standard_normal(n).astype(np.float32)
    X, V = oracle.stft(x, L, H, gain=2.5)
    T = 1 + (n - L) // H
    frames = np.stack([x[t * H:t * H + L].astype(np.float64) * hann(L) for t in range(T)])
    ref = np.fft.rfft(frames, axis=1)
    np.testing.assert_allclose(X, ref, rtol=0, atol=1e-12 * np.abs(ref).max())
    np.testing.assert_allclose(V, 2.5 * np.abs(ref), rtol=1e-12, atol=1e-12)


def test_bin_centred_sinusoid_and_dc(oracle):
    L, H = 64, 16
    n = np.arange(512)
    k0 = 5
    # Hann window: a bin-centred cosine has energy only in bins k0 - 1 .. k0 + 1 (the window's 3-tap DFT)
    X, _ = oracle.stft(np.cos(2 * np.pi * k0 * n / L).astype(np.float32), L, H)
    mag = np.abs(X)
    assert np.all(mag[:, [k for k in range(L // 2 + 1) if abs(k - k0) > 1]] <= 1e-6 * mag.max())
    np.testing.assert_allclose(mag[:, k0], L / 4, rtol=1e-6)          # sum_n w[n] / 2 = L / 4
    np.testing.assert_allclose(mag[:, k0 + 1], L / 8, rtol=1e-6)      # the window's neighbouring taps
    Xd, _ = oracle.stft(np.ones(256, np.float32), L, H)                 # DC: sum w = L / 2 in bin 0, bin 1 = -L/4
    np.testing.assert_allclose(Xd[:, 0], L / 2, rtol=1e-12)
    np.testing.assert_allclose(np.abs(Xd[:, 1]), L / 4, rtol=1e-12)
    assert np.abs(Xd[:, 2:]).max() <= 1e-9


def test_parseval_per_frame(oracle):
    L, H = 128, 32
    rng = np.random.default_rng(3)
    x = rng.standard_normal(600).astype(np.float32)
    X, _ = oracle.stft(x, L, H)
    T = X.shape[0]
    for t in range(T):
        f = x[t * H:t * H + L].astype(np.float64) * hann(L)
        full = np.concatenate([X[t], np.conj(X[t][1:-1][::-1])])
        np.testing.assert_allclose(np.sum(np.abs(full) ** 2) / L, np.sum(f * f), rtol=1e-10)


@pytest.mark.parametrize("L,H", [(64, 16), (128, 32), (64, 32)])
def test_round_trip_identity_mask(oracle, L, H):
    rng = np.random.default_rng(L * H)
    n = 20 * H + L
    x = rng.standard_normal(n).astype(np.float32)
    X, _ = oracle.stft(x, L, H)
    y = oracle.istft(X, np.abs(X), L, H, n)
    T = X.shape[0]
    covered = np.zeros(n)
    for t in range(T):
        covered[t * H:t * H + L] += hann(L) ** 2
    ok = covered > 1e-6
    np.testing.assert_allclose(y[ok], x[ok].astype(np.float64), rtol=0, atol=1e-9)
    assert np.all(y[covered == 0] == 0)
    z = oracle.istft(X, np.zeros_like(np.abs(X)), L, H, n)            # zero mask -> silence
    assert np.all(z == 0)


def test_disjoint_band_masks_separate(oracle):
    """two band-limited sources mixed; the ideal masks (mixture magnitude on each source's bins)
    resynthesise each source with out-of-band energy <= 1% of in-band."""
    L, H = 128, 32
    n = np.arange(4096)
    a = (np.sin(2 * np.pi * 6.2 * n / L) + 0.5 * np.sin(2 * np.pi * 9.7 * n / L)).astype(np.float32)
    b = (np.sin(2 * np.pi * 40.3 * n / L) + 0.7 * np.sin(2 * np.pi * 47.1 * n / L)).astype(np.float32)
    X, _ = oracle.stft(a + b, L, H)
    F = L // 2 + 1
    low = np.arange(F) < 24
    ya = oracle.istft(X, np.abs(X) * low[None, :], L, H, len(n))
    yb = oracle.istft(X, np.abs(X) * (~low)[None, :], L, H, len(n))
    mid = slice(L, len(n) - L)
    for y, src, other in ((ya, a, b), (yb, b, a)):
        err = y[mid] - src[mid]
        assert np.sum(err ** 2) <= 0.01 * np.sum(src[mid].astype(np.float64) ** 2)
    np.testing.assert_allclose(ya[mid] + yb[mid], (a + b)[mid], atol=1e-6)   # masks sum to the mixture
