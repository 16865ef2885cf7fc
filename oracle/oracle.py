"""ctypes wrapper over liboracle.so (oracle/nfhmm_oracle.c).

ORACLE -- TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs may import this module.  The product package
(paper_1206_6468_b200) never imports it.

Every function is a thin marshalling layer over the C oracle; all arithmetic is in the C file,
which cites PAPER.md for each step.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "nfhmm_oracle.c")
_SRCS = [_SRC, os.path.join(_HERE, "nhmm_em_oracle.c"),   # VB iteration; N-HMM EM training (NEXT-3)
         os.path.join(_HERE, "stft_oracle.c")]                   # STFT front end / resynthesis (NEXT-4)
_LIB = os.path.join(_HERE, "liboracle.so")

OR_OK, OR_EINVAL, OR_EZEROSUPPORT, OR_ENUMERIC = 0, -1, -5, -6


def build(force: bool = False) -> str:
    """Compile the oracle: plain gcc -O2, IEEE FP64, no -ffast-math, no threads, no BLAS."""
    if force or not os.path.exists(_LIB) or any(os.path.getmtime(_LIB) < os.path.getmtime(f) for f in _SRCS):
        subprocess.check_call(["gcc", "-O2", "-std=c99", "-fPIC", "-shared", "-o", _LIB, *_SRCS, "-lm"])
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        d, i, P = ctypes.c_double, ctypes.c_int, ctypes.c_void_p
        L.or_digamma.restype = d
        L.or_digamma.argtypes = [d]
        L.or_prior_alpha.argtypes = [i, i, i, d, P, P]
        L.or_forward_backward.argtypes = [i, i, P, P, P, P, P]
        L.or_z_hat.argtypes = [i, i, i, i, i, P, P, P]
        L.or_z_alpha_step.argtypes = [i, i, i, i, i, d, P, P, P, P, P, P, P]
        L.or_surrogate.argtypes = [i, i, i, i, P, P]
        L.or_d_step.argtypes = [i, i, i, d, P, P, P, P, P]
        L.or_dirichlet_entropy.restype = d
        L.or_dirichlet_entropy.argtypes = [i, P]
        L.or_bound.restype = d
        L.or_bound.argtypes = [i, i, i, i, d, d, P, P]
        L.or_separate.argtypes = [i, i, i, i, i, P, P, P, P, P]
        L.or_vb_run.argtypes = [i, i, i, i, i, d, P, P, P, P, i, i, P, P, P, P, P]
        L.or_fb_pairwise.argtypes = [i, i, P, P, P, P, P, P]
        L.or_nhmm_loglik.argtypes = [i, i, i, i, P, P, P, P]
        L.or_nhmm_em_step.argtypes = [i, i, i, i, P, P, P, P, P, P]
        L.or_stft.argtypes = [P, i, i, i, d, P, P]
        L.or_istft.argtypes = [P, P, i, i, i, P, i]
        _lib = L
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def _f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


class OracleError(RuntimeError):
    pass


def _check(st):
    if st != OR_OK:
        raise OracleError(f"oracle status {st}")


def digamma(x: float) -> float:
    return lib().or_digamma(float(x))


def prior_alpha(S, N, K, gamma, states):
    st = np.ascontiguousarray(states, dtype=np.int32)
    out = np.empty(S * N * K)
    _check(lib().or_prior_alpha(S, N, K, gamma, _p(st), _p(out)))
    return out


def forward_backward(loglik, A, pi):
    """loglik [T][N], A [N][N] row-stochastic, pi [N] -> (marginals [T][N], logZ)."""
    ll, A, pi = _f64(loglik), _f64(A), _f64(pi)
    T, N = ll.shape
    marg = np.empty((T, N))
    lz = ctypes.c_double()
    _check(lib().or_forward_backward(T, N, _p(ll), _p(A), _p(pi), _p(marg), ctypes.byref(lz)))
    return marg, lz.value


def z_hat(beta, alpha, dims):
    F, T, S, N, K = dims
    b, a = _f32(beta), _f64(alpha)
    z = np.empty((T, F, S * N * K))
    _check(lib().or_z_hat(F, T, S, N, K, _p(b), _p(a), _p(z)))
    return z


def z_alpha_step(beta, V, alpha, d_hat, dims, gamma=1.0):
    """Returns (alpha_new [T][Kt], V_hat [T][F], data_term)."""
    F, T, S, N, K = dims
    b, v, a, d = _f32(beta), _f32(V), _f64(alpha), _f64(d_hat)
    an = np.empty((T, S * N * K))
    vh = np.empty((T, F))
    dt = ctypes.c_double()
    _check(lib().or_z_alpha_step(F, T, S, N, K, gamma, _p(b), _p(v), _p(a), _p(d), _p(an), _p(vh),
                                 ctypes.byref(dt)))
    return an, vh, dt.value


def surrogate(alpha, dims):
    F, T, S, N, K = dims
    a = _f64(alpha)
    phi = np.empty((S, T, N))
    _check(lib().or_surrogate(T, S, N, K, _p(a), _p(phi)))
    return phi


def d_step(phi, trans, prior, dims, gamma=1.0):
    F, T, S, N, K = dims
    ph, tr, pr = _f64(phi), _f32(trans), _f32(prior)
    d = np.empty((S, T, N))
    lz = np.empty(S)
    _check(lib().or_d_step(T, S, N, gamma, _p(tr), _p(pr), _p(ph), _p(d), _p(lz)))
    return d, lz


def dirichlet_entropy(a):
    a = _f64(a)
    return lib().or_dirichlet_entropy(a.size, _p(a))


def bound(data_term, alpha, logZ, dims, gamma=1.0):
    F, T, S, N, K = dims
    a, lz = _f64(alpha), _f64(logZ)
    return lib().or_bound(T, S, N, K, gamma, data_term, _p(a), _p(lz))


def separate(beta, V, alpha, dims):
    """Returns (V_src [S][T][F], V_star [S][T][F])."""
    F, T, S, N, K = dims
    b, v, a = _f32(beta), _f32(V), _f64(alpha)
    vs = np.empty((S, T, F))
    vst = np.empty((S, T, F))
    _check(lib().or_separate(F, T, S, N, K, _p(b), _p(v), _p(a), _p(vs), _p(vst)))
    return vs, vst


def vb_run(beta, trans, prior, V, dims, n_iters, gamma=1.0, state=None):
    """Full VB run.  beta [S][N][K][F], trans [S][N][N], prior [S][N], V [T][F] (float32 inputs).
    Returns dict(alpha [T][Kt], d_hat [S][T][N], V_hat [T][F], free_energy [n_iters], logZ [S])."""
    F, T, S, N, K = dims
    Kt = S * N * K
    b, tr, pr, v = _f32(beta), _f32(trans), _f32(prior), _f32(V)
    if state is None:
        alpha = np.empty((T, Kt))
        d = np.empty((S, T, N))
        init = 0
    else:
        alpha, d = _f64(state[0]).copy(), _f64(state[1]).copy()
        init = 1
    vh = np.empty((T, F))
    fe = np.empty(max(n_iters, 1))
    lz = np.empty(S)
    _check(lib().or_vb_run(F, T, S, N, K, gamma, _p(b), _p(tr), _p(pr), _p(v), n_iters, init,
                           _p(alpha), _p(d), _p(vh), _p(fe), _p(lz)))
    return dict(alpha=alpha, d_hat=d, V_hat=vh, free_energy=fe[:n_iters], logZ=lz)


# ---- N-HMM maximum-likelihood EM (nhmm_em_oracle.c) ----------------------------------

def fb_pairwise(loglik, A, pi):
    """Returns (marg [T][N], xi_sum [N][N] = sum_{t>=1} xi_t, logZ)."""
    ll, A, pi = _f64(loglik), _f64(A), _f64(pi)
    T, N = ll.shape
    marg = np.empty((T, N))
    xi = np.empty((N, N))
    lz = ctypes.c_double()
    _check(lib().or_fb_pairwise(T, N, _p(ll), _p(A), _p(pi), _p(marg), _p(xi), ctypes.byref(lz)))
    return marg, xi, lz.value


def nhmm_loglik(V, beta, theta):
    """V [T][F], beta [N][K][F], theta [T][N][K] -> loglik [T][N]."""
    v, b, th = _f64(V), _f64(beta), _f64(theta)
    T, F = v.shape
    N, K, _ = b.shape
    ll = np.empty((T, N))
    _check(lib().or_nhmm_loglik(F, T, N, K, _p(v), _p(b), _p(th), _p(ll)))
    return ll


def nhmm_em(V, beta, theta, A, pi, n_iters):
    """n_iters EM iterations from (beta [N][K][F], theta [T][N][K], A [N][N], pi [N]); returns
    dict(beta, theta, A, pi, loglik [n_iters]) -- loglik[i] is the log evidence of the parameters
    iteration i started from."""
    v = _f64(V)
    b, th, a, p = _f64(beta).copy(), _f64(theta).copy(), _f64(A).copy(), _f64(pi).copy()
    T, F = v.shape
    N, K, _ = b.shape
    ll = np.empty(n_iters)
    for i in range(n_iters):
        lz = ctypes.c_double()
        _check(lib().or_nhmm_em_step(F, T, N, K, _p(v), _p(b), _p(th), _p(a), _p(p), ctypes.byref(lz)))
        ll[i] = lz.value
    return dict(beta=b, theta=th, A=a, pi=p, loglik=ll)


# ---- STFT front end and resynthesis (stft_oracle.c) -------------------------------------

def stft(x, win, hop, gain=1.0):
    """x [n_samples] (one signal) -> (X [T][F] complex128, V [T][F] = gain |X|)."""
    xs = _f32(x)
    n = xs.shape[0]
    T = 1 + (n - win) // hop
    F = win // 2 + 1
    X = np.empty((T, F, 2))
    V = np.empty((T, F))
    _check(lib().or_stft(_p(xs), n, win, hop, float(gain), _p(X), _p(V)))
    return X[..., 0] + 1j * X[..., 1], V


def istft(X, M, win, hop, n_samples):
    """X [T][F] complex mixture STFT, M [T][F] magnitudes -> y [n_samples] (mixture phase, weighted OLA)."""
    Xc = np.asarray(X)
    Xr = np.ascontiguousarray(np.stack([Xc.real, Xc.imag], -1), dtype=np.float64)
    Mm = _f64(M)
    T = Xr.shape[0]
    y = np.empty(n_samples)
    _check(lib().or_istft(_p(Xr), _p(Mm), T, win, hop, _p(y), n_samples))
    return y
