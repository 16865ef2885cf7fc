"""Seeded synthetic inputs shared by the CUDA path's tests/bench and the CPU oracle.

This module holds ONLY the generative sampling of BASELINE.json's configs (the N-HMM generative
process of PAPER.md §2.1/§2.2, applied per source and summed), and none of the
inference arithmetic.  It is the one module both sides may import (task rule ③).

Recipe (BASELINE.json configs 0-4), per source s:
  1. dictionary columns beta_s(n, j) ~ Dirichlet(c_dict) over F bins (c_dict = 1, or 0.5 for cfg 4);
  2. transition rows A_s[i] ~ Dirichlet(1) + boost * e_i, renormalised (boost 8 / 8 / 20 / 8 / 30);
  3. pi_s uniform;
  4. state path D_1 ~ pi_s, D_t ~ A_s[D_{t-1}];
  5. weights w_t ~ Dirichlet(1) over the K elements of the active dictionary;
  6. mass m_t ~ LogNormal(0, 0.5);
  7. X_s[t] = m_t * sum_j w_tj beta_s(D_t, j).
Then V[t] ~ Multinomial(C, sum_s X_s[t] / sum_l sum_s X_s[t, l]), C = 1e4 (cfg 0) or 1e5 (others).
Model key = (seed_c, 0xFFFFFFFF); mixture m key = (seed_c, m) so every mixture is generated the same
way on any rank (sharding invariance).  seed_c = 12066468 + c.
"""
from __future__ import annotations

import dataclasses
import os
from concurrent.futures import ProcessPoolExecutor

import numpy as np

SEED_BASE = 12066468


@dataclasses.dataclass(frozen=True)
class Config:
    name: str
    S: int
    N: int
    K: int
    F: int
    T: int
    M: int
    iters: int
    counts: int
    diag_boost: float
    dict_conc: float

    @property
    def Kt(self) -> int:
        return self.S * self.N * self.K

    @property
    def dims(self):
        return (self.F, self.T, self.S, self.N, self.K)


CONFIGS = {
    0: Config("tiny", 2, 4, 3, 33, 50, 1, 20, 10_000, 8.0, 1.0),
    1: Config("paper-typical", 2, 40, 10, 513, 1000, 1, 100, 100_000, 8.0, 1.0),
    2: Config("three-sources", 3, 40, 10, 513, 2000, 1, 100, 100_000, 20.0, 1.0),
    3: Config("batched", 2, 40, 10, 513, 2000, 256, 50, 100_000, 8.0, 1.0),
    4: Config("large", 4, 100, 20, 1025, 8000, 64, 50, 100_000, 30.0, 0.5),
}


def config(c: int, **override) -> Config:
    return dataclasses.replace(CONFIGS[c], **override) if override else CONFIGS[c]


def seed_of(c: int) -> int:
    return SEED_BASE + c


@dataclasses.dataclass
class Model:
    beta: np.ndarray    # [S][N][K][F] float32, each column sums to 1
    trans: np.ndarray   # [S][N][N] float32, row i = P(next = j | current = i)
    prior: np.ndarray   # [S][N] float32


def make_model(cfg: Config, seed: int) -> Model:
    rng = np.random.default_rng([seed, 0xFFFFFFFF])
    S, N, K, F = cfg.S, cfg.N, cfg.K, cfg.F
    beta = rng.dirichlet(np.full(F, cfg.dict_conc), size=(S, N, K))
    # Dirichlet(<1) can underflow to exact zeros in float64; keep every bin strictly positive so the
    # mixture has full support (V > 0 with V_hat = 0 would be a zero-support error).
    beta = np.maximum(beta, 1e-30)
    beta /= beta.sum(-1, keepdims=True)
    trans = rng.dirichlet(np.ones(N), size=(S, N)) + cfg.diag_boost * np.eye(N)[None]
    trans /= trans.sum(-1, keepdims=True)
    prior = np.full((S, N), 1.0 / N)
    return Model(beta.astype(np.float32), trans.astype(np.float32), prior.astype(np.float32))


@dataclasses.dataclass
class Mixture:
    V: np.ndarray        # [T][F] float32 integer-valued counts
    paths: np.ndarray    # [S][T] int32 true state paths
    sources: np.ndarray  # [S][T][F] float32 true (pre-multinomial) source spectra X_s


def make_mixture(cfg: Config, model: Model, seed: int, m: int, with_truth: bool = False) -> Mixture:
    rng = np.random.default_rng([seed, m])
    S, N, K, F, T = cfg.S, cfg.N, cfg.K, cfg.F, cfg.T
    beta = model.beta.astype(np.float64)
    trans = model.trans.astype(np.float64)
    X = np.zeros((S, T, F))
    paths = np.zeros((S, T), dtype=np.int32)
    for s in range(S):
        cum = np.cumsum(trans[s], axis=1)
        u = rng.random(T)
        d = int(np.searchsorted(np.cumsum(model.prior[s].astype(np.float64)), u[0] * model.prior[s].sum(), side="right"))
        d = min(d, N - 1)
        paths[s, 0] = d
        for t in range(1, T):
            d = min(int(np.searchsorted(cum[d], u[t] * cum[d, -1], side="right")), N - 1)
            paths[s, t] = d
        w = rng.dirichlet(np.ones(K), size=T)                   # [T][K]
        mass = rng.lognormal(0.0, 0.5, size=T)                  # [T]
        X[s] = mass[:, None] * np.einsum("tj,tjf->tf", w, beta[s, paths[s]])
    P = X.sum(0)
    P /= P.sum(-1, keepdims=True)
    V = rng.multinomial(cfg.counts, P).astype(np.float32)
    if with_truth:
        return Mixture(V, paths, X.astype(np.float32))
    return Mixture(V, paths, np.zeros((0,), np.float32))


def _mix_worker(args):
    cfg, model, seed, m = args
    return make_mixture(cfg, model, seed, m).V


def make_batch(cfg: Config, model: Model, seed: int, mixtures, workers: int | None = None) -> np.ndarray:
    """V for the given mixture ids, stacked [len(mixtures)][T][F] float32 (process pool if many)."""
    mixtures = list(mixtures)
    if workers is None:
        workers = min(len(mixtures), os.cpu_count() or 1, 32)
    if workers <= 1 or len(mixtures) <= 2:
        return np.stack([make_mixture(cfg, model, seed, m).V for m in mixtures])
    with ProcessPoolExecutor(max_workers=workers) as ex:
        out = list(ex.map(_mix_worker, [(cfg, model, seed, m) for m in mixtures], chunksize=1))
    return np.stack(out)


# ---- N-HMM EM training inputs ------------------------------------------------------
# Isolated-source training spectrograms: source s of config c's model sampled ALONE through the same
# generative process (steps 1-7 above with S = 1, key (seed_c, 0xE0000000 + s)), i.e. the "training data
# of each speaker" the separation models are learned from.  EM start (the paper does not state
# one): dictionaries ~ Dirichlet(1) over F, transition rows Dirichlet(1) + 1 on the diagonal
# (near-uniform with a small boost), uniform pi, uniform weights (passed as NULL).

def make_training_data(cfg: Config, model: Model, seed: int, T: int | None = None) -> np.ndarray:
    """[S][T][F] float32: one isolated-source spectrogram per source of cfg's model."""
    T = T or cfg.T
    out = []
    for s in range(cfg.S):
        c1 = dataclasses.replace(cfg, S=1, T=T)
        m1 = Model(model.beta[s:s + 1], model.trans[s:s + 1], model.prior[s:s + 1])
        out.append(make_mixture(c1, m1, seed, 0xE0000000 + s).V)
    return np.stack(out).astype(np.float32)


def make_em_init(cfg: Config, seed: int):
    """(dict [S][N][K][F], trans [S][N][N], prior [S][N]) float32 starting point for EM."""
    rng = np.random.default_rng([seed, 0xE1000000])
    S, N, K, F = cfg.S, cfg.N, cfg.K, cfg.F
    beta = rng.dirichlet(np.ones(F), size=(S, N, K))
    beta = np.maximum(beta, 1e-30)
    beta /= beta.sum(-1, keepdims=True)
    trans = rng.dirichlet(np.ones(N), size=(S, N)) + np.eye(N)[None]
    trans /= trans.sum(-1, keepdims=True)
    prior = np.full((S, N), 1.0 / N)
    return beta.astype(np.float32), trans.astype(np.float32), prior.astype(np.float32)
