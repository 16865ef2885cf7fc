"""GPU parity at BASELINE.json's full sizes, in the launch configuration bench.py times (one handle over
all mixtures of the config, the default tensor-core engine).  The oracle checks sampled mixtures (or,
for config 4, sampled frames of the first sweep, whose alpha depends only on its own frame because
d^0 is uniform: Eq. 6 with R5); every mixture is checked against invariants that hold at any size."""
import numpy as np
import pytest

from paper_1206_6468_b200 import synth
from tests.gpu_common import rel_l2, run_gpu, run_oracle

pytestmark = pytest.mark.gpu


def full_inputs(c):
    cfg = synth.config(c)
    seed = synth.seed_of(c)
    model = synth.make_model(cfg, seed)
    V = synth.make_batch(cfg, model, seed, range(cfg.M))
    return cfg, model, V


def check_invariants(cfg, V, g):
    np.testing.assert_allclose(g["d_hat"].sum(-1), 1.0, atol=5e-6)
    assert (g["alpha_hat"] >= 1.0).all()
    np.testing.assert_allclose(g["alpha_hat"].sum(-1), V.sum(-1) + cfg.Kt + cfg.S * cfg.K, rtol=5e-6)
    fe = g["free_energy"]
    assert np.isfinite(fe).all()
    assert (np.diff(fe, axis=1) >= -1e-6 * np.abs(fe[:, 1:])).all()


def test_cfg1_paper_typical_full():
    cfg, model, V = full_inputs(1)
    g1 = run_gpu(cfg, model, V, 1, separate=False)
    o1 = run_oracle(cfg, model, V[0], 1, separate=False)
    for key, okey in (("d_hat", "d_hat"), ("V_hat", "V_hat"), ("alpha_hat", "alpha")):
        assert rel_l2(g1[key][0], o1[okey]) <= 1e-5, key
    iters = 50
    g = run_gpu(cfg, model, V, iters)
    o = run_oracle(cfg, model, V[0], iters)
    assert rel_l2(g["V_star"][0], o["V_star"]) <= 1e-3
    assert np.all(np.abs(g["free_energy"][0] - o["free_energy"]) <= 1e-5 * np.abs(o["free_energy"]))
    check_invariants(cfg, V, g)
    g100 = run_gpu(cfg, model, V, cfg.iters, separate=False)          # the config's 100 sweeps
    check_invariants(cfg, V, g100)


def test_cfg2_three_sources_full_first_sweep():
    cfg, model, V = full_inputs(2)
    g1 = run_gpu(cfg, model, V, 1, separate=False)
    o1 = run_oracle(cfg, model, V[0], 1, separate=False)
    for key, okey in (("d_hat", "d_hat"), ("V_hat", "V_hat"), ("alpha_hat", "alpha")):
        assert rel_l2(g1[key][0], o1[okey]) <= 1e-5, key
    g = run_gpu(cfg, model, V, cfg.iters, separate=False)
    check_invariants(cfg, V, g)


def test_cfg3_batched_full_sampled_mixtures():
    cfg, model, V = full_inputs(3)
    g1 = run_gpu(cfg, model, V, 1, separate=False)
    for m in (0, 255):
        o1 = run_oracle(cfg, model, V[m], 1, separate=False)
        for key, okey in (("d_hat", "d_hat"), ("V_hat", "V_hat"), ("alpha_hat", "alpha")):
            assert rel_l2(g1[key][m], o1[okey]) <= 1e-5, (m, key)
        assert abs(g1["free_energy"][m, 0] - o1["free_energy"][0]) <= 1e-5 * abs(o1["free_energy"][0])
    g = run_gpu(cfg, model, V, cfg.iters)
    check_invariants(cfg, V, g)
    np.testing.assert_allclose(g["V_star"].sum(1), V, rtol=1e-5, atol=2e-3)


def test_cfg4_large_full_sampled_frames():
    from oracle import oracle
    cfg, model, V = full_inputs(4)
    g1 = run_gpu(cfg, model, V, 1, separate=False)
    rng = np.random.default_rng(4)
    for m in (0, 63):
        ts = np.sort(rng.choice(cfg.T, size=24, replace=False))
        sub = V[m][ts]
        dims = (cfg.F, len(ts), cfg.S, cfg.N, cfg.K)
        a0 = np.full((len(ts), cfg.Kt), 1.0 + 1.0 / cfg.N)
        d0 = np.full((cfg.S, len(ts), cfg.N), 1.0 / cfg.N)
        a1, _, _ = oracle.z_alpha_step(model.beta, sub, a0, d0, dims, 1.0)        # alpha_1 (frame-local)
        _, vh1, _ = oracle.z_alpha_step(model.beta, sub, a1, d0, dims, 1.0)       # V_hat of alpha_1
        assert rel_l2(g1["alpha_hat"][m][ts], a1) <= 1e-5
        assert rel_l2(g1["V_hat"][m][ts], vh1) <= 1e-5
    np.testing.assert_allclose(g1["d_hat"].sum(-1), 1.0, atol=5e-6)
    np.testing.assert_allclose(g1["alpha_hat"].sum(-1), V.sum(-1) + cfg.Kt + cfg.S * cfg.K, rtol=5e-6)
