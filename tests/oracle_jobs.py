"""Full-size oracle runs for the parity tests, spread over the host cores (test infrastructure).

The oracle (oracle/nfhmm_oracle.c) is single-threaded; a full-size run of config 2 or 4 takes from
minutes to an hour on one core.  The z/alpha step (Eq. 7 then Eq. 6) and Eq. 8 are
frame-local, the Dirichlet entropy of the bound is a sum over frames, and only the forward-backward
 couples frames.  `vb_run_frames` therefore runs EXACTLY the sequence of or_vb_run (z/alpha step
-> bound of the previous state -> Eq. 8 -> forward-backward per source; trailing z-step; DESIGN R5-R8)
with the frame-local oracle calls (or_z_alpha_step, or_surrogate, or_bound) cut into frame chunks and
run in worker processes, and the forward-backward (or_d_step) on the whole chain.  Only the FP64
summation order of the data term and of the per-frame bound terms differs from or_vb_run (chunk partials
added in chunk order); `tests/test_oracle_jobs.py` pins the two together on small inputs.

No arithmetic of the method lives here: every number comes from an oracle/ call.  Nothing here touches
the CUDA path.
"""
from __future__ import annotations

import multiprocessing as mp
import os
from concurrent.futures import ProcessPoolExecutor

import numpy as np

_CACHE: dict[str, np.ndarray] = {}


def _load(path):
    if path not in _CACHE:
        _CACHE[path] = np.load(path)
    return _CACHE[path]


def _z_chunk(args):
    beta_path, V, alpha, d, dims, gamma, want_vh = args
    from oracle import oracle
    an, vh, data = oracle.z_alpha_step(_load(beta_path), V, alpha, d, dims, gamma)
    return an, (vh if want_vh else None), data


def _surrogate_chunk(args):
    alpha, dims = args
    from oracle import oracle
    return oracle.surrogate(alpha, dims)


def _bound_chunk(args):
    alpha, dims, gamma = args
    from oracle import oracle
    S = dims[2]
    # or_bound with a zero data term and zero log Z: the chunk's Dirichlet entropies + T_c * c_prior
    return oracle.bound(0.0, alpha, np.zeros(S), dims, gamma)


def _separate_chunk(args):
    beta_path, V, alpha, dims = args
    from oracle import oracle
    return oracle.separate(_load(beta_path), V, alpha, dims)


def make_pool(workers=None):
    """Spawned workers (the parent may hold a CUDA context; the children only load the oracle)."""
    workers = workers or max(1, os.cpu_count() or 1)
    return ProcessPoolExecutor(max_workers=workers, mp_context=mp.get_context("spawn"))


def save_beta(beta, directory, name):
    path = os.path.join(directory, f"beta_{name}.npy")
    np.save(path, np.ascontiguousarray(beta, np.float32))
    return path


def _cuts(T, chunks):
    chunks = max(1, min(chunks, T))
    return [(i * T // chunks, (i + 1) * T // chunks) for i in range(chunks)]


def vb_run_frames(ex, beta_path, trans, prior, V, dims, n_iters, gamma=1.0, chunks=32, separate=True,
                  snapshot_first=True):
    """or_vb_run's sequence with frame-chunked oracle calls on executor `ex` (see module docstring).
    Returns dict(alpha, d_hat, V_hat, free_energy [n_iters], logZ) of the final state, plus
    first=dict(alpha, d_hat, V_hat, free_energy) after sweep 1 (snapshot_first) and V_src / V_star
    (separate, Section 4)."""
    from oracle import oracle
    F, T, S, N, K = dims
    Kt = S * N * K
    V = np.ascontiguousarray(V, np.float32)
    cuts = _cuts(T, chunks)
    sub = lambda t0, t1: (F, t1 - t0, S, N, K)   # noqa: E731

    def z_step(alpha, d, want_vh):
        jobs = [(beta_path, V[t0:t1], alpha[t0:t1], np.ascontiguousarray(d[:, t0:t1]), sub(t0, t1), gamma, want_vh)
                for t0, t1 in cuts]
        res = list(ex.map(_z_chunk, jobs))
        an = np.concatenate([r[0] for r in res])
        vh = np.concatenate([r[1] for r in res]) if want_vh else None
        data = 0.0
        for r in res:
            data += r[2]
        return an, vh, data

    def bound(data, alpha, logZ):
        parts = list(ex.map(_bound_chunk, [(alpha[t0:t1], sub(t0, t1), gamma) for t0, t1 in cuts]))
        L = data
        for p in parts:
            L += p
        for s in range(S):
            L += logZ[s]
        return L

    def phi_of(alpha):
        parts = list(ex.map(_surrogate_chunk, [(alpha[t0:t1], sub(t0, t1)) for t0, t1 in cuts]))
        return np.concatenate(parts, axis=1)

    alpha = np.full((T, Kt), 1.0 + gamma / N)           # DESIGN R5
    d = np.full((S, T, N), 1.0 / N)
    logZ = np.zeros(S)
    fe = np.empty(n_iters)
    first = None
    for it in range(1, n_iters + 1):
        an, vh, data = z_step(alpha, d, want_vh=(it == 2 and snapshot_first))
        if it >= 2:
            fe[it - 2] = bound(data, alpha, logZ)
        if it == 2 and snapshot_first:
            first = dict(alpha=alpha, d_hat=d, V_hat=vh, free_energy=fe[:1].copy())
        alpha = an
        d, logZ = oracle.d_step(phi_of(alpha), trans, prior, dims, gamma)
    _, vh, data = z_step(alpha, d, want_vh=True)
    if n_iters >= 1:
        fe[n_iters - 1] = bound(data, alpha, logZ)
    out = dict(alpha=alpha, d_hat=d, V_hat=vh, free_energy=fe, logZ=logZ)
    if n_iters == 1 and snapshot_first:
        first = dict(alpha=alpha, d_hat=d, V_hat=vh, free_energy=fe[:1].copy())
    out["first"] = first
    if separate:
        parts = list(ex.map(_separate_chunk, [(beta_path, V[t0:t1], alpha[t0:t1], sub(t0, t1)) for t0, t1 in cuts]))
        out["V_src"] = np.concatenate([p[0] for p in parts], axis=1)
        out["V_star"] = np.concatenate([p[1] for p in parts], axis=1)
    return out
