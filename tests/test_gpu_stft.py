"""GPU parity of the spectrogram front end and the resynthesis back end (libnfhmm nfhmm_stft / nfhmm_istft,
SURVEY §8(f) NEXT-4) against the FP64 DFT-definition oracle (oracle/stft_oracle.c, pinned in
tests/test_stft_oracle.py), plus the round trip and an end-to-end separation of two synthetic band-limited
sources (STFT -> N-HMM training per source -> VB separation -> resynthesis with the mixture phase).

Tolerances: an FP32 radix-2 FFT of length L carries ~log2(L) eps relative error per bin against the FP64
DFT: rel-L2 <= 1e-6 for X and V; the resynthesis (two FFTs, one overlap-add) rel-L2 <= 2e-6."""
import numpy as np
import pytest

from tests.gpu_common import compare

pytestmark = pytest.mark.gpu


def signals(n_sig, n, seed):
    rng = np.random.default_rng(seed)
    return rng.standard_normal((n_sig, n)).astype(np.float32)


@pytest.mark.parametrize("L,H,n,n_sig", [(1024, 256, 16000, 2), (64, 16, 1000, 3), (256, 256, 2048, 1), (8, 2, 40, 2)])
def test_stft_matches_oracle(oracle, L, H, n, n_sig):
    from paper_1206_6468_b200.nfhmm import stft
    x = signals(n_sig, n, L + n)
    g = stft(x, win=L, hop=H, gain=3.0)
    for i in range(n_sig):
        X, V = oracle.stft(x[i], L, H, gain=3.0)
        compare(f"stft:L{L}H{H}/sig{i}", "X", np.stack([g["X"][i].real, g["X"][i].imag], -1),
                np.stack([X.real, X.imag], -1), 1e-6)
        compare(f"stft:L{L}H{H}/sig{i}", "V", g["V"][i], V, 1e-6)


@pytest.mark.parametrize("L,H,T,S", [(1024, 256, 40, 2), (64, 16, 30, 3), (16, 8, 9, 1)])
def test_istft_matches_oracle(oracle, L, H, T, S):
    from paper_1206_6468_b200.nfhmm import istft
    rng = np.random.default_rng(L * T)
    n = (T - 1) * H + L
    x = rng.standard_normal(n).astype(np.float32)
    X, _ = oracle.stft(x, L, H)                      # the mixture STFT (from the oracle, cast to complex64)
    X32 = X.astype(np.complex64)
    M = (rng.random((S, T, L // 2 + 1)) * 5).astype(np.float32)
    y = istft(X32[None], M[None], n, win=L, hop=H, gain=2.0)
    # samples covered only by a window's tails (sum_t w^2 < 1e-2 of its maximum, at the signal's two ends)
    # are ill-conditioned: the FP32 frames' absolute error is divided by w^2 (~1e-10 next to a window's
    # zero); they are compared separately with a bound scaled by that amplification
    w = 0.5 - 0.5 * np.cos(2 * np.pi * np.arange(L) / L)
    den = np.zeros(n)
    for t in range(T):
        den[t * H:t * H + L] += w * w
    ok = den >= 1e-2 * den.max()
    for s in range(S):
        ref = oracle.istft(X32.astype(np.complex128), M[s].astype(np.float64) / 2.0, L, H, n)
        compare(f"istft:L{L}H{H}T{T}/src{s}", "y (sum w^2 >= 1e-2 max)", y[0, s][ok], ref[ok], 2e-6)
        edge = ~ok & (den > 0)
        scale = np.abs(ref[ok]).max()
        assert np.all(np.abs(y[0, s][edge] - ref[edge]) <= 1e-5 * scale * den.max() / den[edge])


def test_round_trip_paper_analysis():
    """P:219 analysis (1024 / 256 at 16 kHz): istft(stft(x), |X|) = x wherever the windows cover x."""
    from paper_1206_6468_b200.nfhmm import istft, stft
    x = signals(2, 16000, 7)
    g = stft(x, 1024, 256, gain=1.0)
    y = istft(g["X"], g["V"][:, None], 16000, 1024, 256, gain=1.0)
    cover = slice(1024, 16000 - 1024)
    for i in range(2):
        err = np.linalg.norm(y[i, 0, cover] - x[i, cover]) / np.linalg.norm(x[i, cover])
        assert err <= 2e-6, err


def test_end_to_end_separation_of_band_limited_sources():
    """Two synthetic 'speakers' in different bands (harmonic stacks switching between 3 pitches, i.e. a
    3-state chain each), 16 kHz, the paper's analysis: GPU STFT -> counts -> per-source N-HMM EM training on
    the isolated sources -> VB separation of the 0 dB mixture -> resynthesis with the mixture phase
    (P:201).  Each output is closer to its own source than to the other (SDR gain > 10 dB)."""
    from paper_1206_6468_b200.nfhmm import NFHMM, NHMMTrainer, istft, stft
    fs, n, L, H = 16000, 32000, 1024, 256
    rng = np.random.default_rng(11)
    t = np.arange(n) / fs

    def speaker(f0s, band):
        y = np.zeros(n)
        seg = 4000
        for s0 in range(0, n, seg):
            f0 = f0s[rng.integers(len(f0s))]
            for h in range(1, 6):
                if f0 * h < band:
                    y[s0:s0 + seg] += np.sin(2 * np.pi * f0 * h * t[s0:s0 + seg]) / h
        return (y / np.abs(y).max()).astype(np.float32)

    a = speaker([200.0, 250.0, 300.0], 1800.0)
    b = speaker([2600.0, 3000.0, 3400.0], 8000.0)
    gain = 50.0
    spec = stft(np.stack([a, b, a + b]), L, H, gain=gain)
    V = spec["V"]
    T, F = V.shape[1], V.shape[2]
    N, K = 3, 4
    # EM start: random dictionaries, near-uniform chain
    b0 = rng.dirichlet(np.ones(F), size=(2, N, K)).astype(np.float32)
    a0 = (np.full((2, N, N), 1.0 / N) + 0.1 * np.eye(N)[None]).astype(np.float32)
    a0 /= a0.sum(-1, keepdims=True)
    p0 = np.full((2, N), 1.0 / N, np.float32)
    tr = NHMMTrainer(F, T, N, K, n_src=2, max_iters=30)
    tr.set_data(np.ascontiguousarray(V[:2]))
    tr.set_params(b0, a0, p0)
    tr.em(30)
    m = tr.get()
    tr.close()
    assert np.all(np.diff(m["loglik"], axis=1) >= -1e-6 * np.abs(m["loglik"][:, 1:]))
    dict_ = np.ascontiguousarray(np.concatenate([m["dict"][0:1], m["dict"][1:2]], 0))   # [S=2][N][K][F]
    h = NFHMM(F, T, 2, N, K, n_mix=1)
    h.set_model(dict_, m["trans"], m["prior"])
    h.set_observations(np.ascontiguousarray(V[2:3]))
    h.vb_iterate(30)
    vstar = h.separate()                                   # [1][2][T][F]
    h.close()
    y = istft(spec["X"][2:3], vstar, n, L, H, gain=gain)  # [1][2][n]
    cover = slice(L, n - L)

    def sdr(est, ref):
        return 10 * np.log10(np.sum(ref.astype(np.float64) ** 2) / np.sum((est - ref).astype(np.float64) ** 2))

    for s, src, other in ((0, a, b), (1, b, a)):
        got, base = sdr(y[0, s, cover], src[cover]), sdr((a + b)[cover], src[cover])
        assert got - base >= 10.0, (s, got, base)
