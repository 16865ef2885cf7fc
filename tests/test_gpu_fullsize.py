"""GPU parity at BASELINE.json's full sizes, in the launch configuration bench.py times: one handle over
ALL mixtures of the config, the default options (tensor-core engine, bound on, the caller's current
stream), the config's own sweep count.  So config 3 runs the path bench.py times (512,000 frames:
eager launches, the sequential forward-backward beside the reconstruction GEMM, the wide tiles).

Tolerance points (BASELINE.json north_star):
  after sweep 1:             d_hat, V_hat, alpha_hat rel-L2 <= 1e-5; L_1 rel <= 1e-5
  after the config's sweeps: V_star and V_src rel-L2 <= 1e-3; L_i rel <= 1e-5 at EVERY sweep i
Coverage (the oracle checks sampled mixtures; invariants are checked on every mixture):
  cfg 1 (1 x 1000, 100 sweeps) and cfg 2 (1 x 2000, S = 3, 100 sweeps): the whole run;
  cfg 3 (256 x 2000, 50 sweeps): mixtures 0, 128, 255 (first, middle, last row tile of the batch);
  cfg 4 (64 x 8000, S = 4, N = 100, K = 20, F = 1025): sweep 1 at full size on mixtures 0 and 63, and
        50 sweeps of all 64 mixtures at T = 200 (oracle: mixtures 0 and 63).
The oracle runs are submitted to a process pool over the host cores at module start
(tests/oracle_jobs.py, pinned equal to or_vb_run in tests/test_oracle_jobs.py) and overlap the GPU
runs.  Every comparison is logged (rel-L2 and max-abs) to the parity record (tests/gpu_common.record).
"""
import os
import tempfile
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

from paper_1206_6468_b200 import synth
from tests import oracle_jobs
from tests.gpu_common import compare, record

pytestmark = pytest.mark.gpu

TOL1 = 1e-5
TOL_VSTAR = 1e-3
TOL_L = 1e-5

# (job key) -> (config, override, mixtures, sweeps)
JOBS = {
    "cfg4_full_sweep1": (4, {}, (0, 63), 1),
    "cfg2_full": (2, {}, (0,), 100),
    "cfg3_full": (3, {}, (0, 128, 255), 50),
    "cfg4_T200": (4, {"T": 200}, (0, 63), 50),
    "cfg1_full": (1, {}, (0,), 100),
}


@pytest.fixture(scope="module")
def oracle_runs():
    """{job: {m: future of the oracle result}} -- submitted once, longest first."""
    from oracle import oracle
    oracle.build()
    tmp = tempfile.mkdtemp(prefix="nfhmm_oracle_")
    ex = oracle_jobs.make_pool(os.cpu_count())
    drivers = ThreadPoolExecutor(max_workers=16)
    futs = {}
    for job, (c, over, mixtures, sweeps) in JOBS.items():
        cfg = synth.config(c, **over)
        seed = synth.seed_of(c)
        model = synth.make_model(cfg, seed)
        bp = oracle_jobs.save_beta(model.beta, tmp, job)
        futs[job] = {}
        for m in mixtures:
            V = synth.make_mixture(cfg, model, seed, m).V
            futs[job][m] = drivers.submit(oracle_jobs.vb_run_frames, ex, bp, model.trans, model.prior, V, cfg.dims,
                                          sweeps, 1.0, 64, sweeps > 1)
    yield futs
    drivers.shutdown(wait=True, cancel_futures=True)
    ex.shutdown(wait=True, cancel_futures=True)


def full_inputs(c, **over):
    cfg = synth.config(c, **over)
    seed = synth.seed_of(c)
    model = synth.make_model(cfg, seed)
    V = synth.make_batch(cfg, model, seed, range(cfg.M))
    return cfg, model, V


def run_gpu_full(cfg, model, V, iters, mixtures, separate=True):
    """One handle over every mixture (bench.py's launch configuration).  Outputs stay on the device;
    returns the sampled mixtures' arrays on the host plus all-mixture invariant checks."""
    import torch
    from paper_1206_6468_b200.nfhmm import NFHMM, nfhmm_posteriors
    M, S, T, N, F, Kt = V.shape[0], cfg.S, cfg.T, cfg.N, cfg.F, cfg.Kt
    dev = "cuda:0"
    h = NFHMM(cfg.F, cfg.T, cfg.S, cfg.N, cfg.K, n_mix=M, max_iters=max(iters, 1))
    h.set_model(model.beta, model.trans, model.prior)
    Vd = torch.from_numpy(np.ascontiguousarray(V)).to(dev)
    h.set_observations(Vd)
    h.vb_iterate(iters)
    d = torch.empty((M, S, T, N), dtype=torch.float32, device=dev)
    a = torch.empty((M, T, Kt), dtype=torch.float32, device=dev)
    vh = torch.empty((M, T, F), dtype=torch.float32, device=dev)
    fe = np.empty((M, h.max_iters), np.float64)
    it = nfhmm_posteriors(h.h, d, a, vh, fe)
    assert it == iters
    fe = fe[:, :iters]
    # invariants on every mixture (any size): sum_n d = 1; alpha >= 1; sum_k alpha = v_t + Kt + gamma S K
    # (R19); L finite and non-decreasing (coordinate ascent)
    assert float((d.sum(-1) - 1.0).abs().max()) <= 5e-6
    assert float(a.min()) >= 1.0
    mass = Vd.sum(-1, dtype=torch.float64) + Kt + S * cfg.K
    assert float(((a.sum(-1, dtype=torch.float64) - mass).abs() / mass).max()) <= 5e-6
    assert np.isfinite(fe).all()
    assert (np.diff(fe, axis=1) >= -1e-6 * np.abs(fe[:, 1:])).all()
    out = {m: dict(d_hat=d[m].cpu().numpy(), alpha_hat=a[m].cpu().numpy(), V_hat=vh[m].cpu().numpy(),
                   free_energy=fe[m]) for m in mixtures}
    del a, vh
    if separate:
        vst = torch.empty((M, S, T, F), dtype=torch.float32, device=dev)
        vs = torch.empty((M, S, T, F), dtype=torch.float32, device=dev)
        h.separate_into(vst, vs)
        # Section 4 mass: sum_s V* = V on every mixture
        assert float((vst.sum(1) - Vd).abs().max()) <= 2e-3 + 1e-5 * float(Vd.max())
        for m in mixtures:
            out[m]["V_star"] = vst[m].cpu().numpy()
            out[m]["V_src"] = vs[m].cpu().numpy()
        del vst, vs
    out["launches"] = h.kernel_launches()
    h.close()
    del d, Vd
    torch.cuda.empty_cache()
    return out


def check_first_sweep(tag, g, o1):
    """g: GPU arrays after sweep 1 of mixture m; o1: oracle state after sweep 1."""
    compare(tag, "d_hat", g["d_hat"], o1["d_hat"], TOL1)
    compare(tag, "V_hat", g["V_hat"], o1["V_hat"], TOL1)
    compare(tag, "alpha_hat", g["alpha_hat"], o1["alpha"], TOL1)
    rel = abs(g["free_energy"][0] - o1["free_energy"][0]) / abs(o1["free_energy"][0])
    record(tag, "L_1", rel=rel, tol=TOL_L)
    assert rel <= TOL_L, (tag, rel)


def check_final(tag, g, on):
    compare(tag, "V_star", g["V_star"], on["V_star"], TOL_VSTAR)
    compare(tag, "V_src", g["V_src"], on["V_src"], TOL_VSTAR)
    fe_g, fe_o = g["free_energy"], on["free_energy"]
    assert fe_g.shape == fe_o.shape
    rel = np.abs(fe_g - fe_o) / np.abs(fe_o)
    record(tag, "L_every_sweep", rel=float(rel.max()), tol=TOL_L, sweeps=int(len(fe_o)))
    assert float(rel.max()) <= TOL_L, (tag, float(rel.max()), int(rel.argmax()))


def _full_run(job, oracle_runs):
    c, over, mixtures, sweeps = JOBS[job]
    cfg, model, V = full_inputs(c, **over)
    g1 = run_gpu_full(cfg, model, V, 1, mixtures, separate=False)
    gn = run_gpu_full(cfg, model, V, sweeps, mixtures) if sweeps > 1 else None
    for m in mixtures:
        on = oracle_runs[job][m].result(timeout=3600)
        check_first_sweep(f"{job}/m{m}/sweep1", g1[m], on["first"])
        if gn is not None:
            check_final(f"{job}/m{m}/sweep{sweeps}", gn[m], on)


def test_cfg1_paper_typical_full(oracle_runs):
    _full_run("cfg1_full", oracle_runs)


def test_cfg2_three_sources_full(oracle_runs):
    _full_run("cfg2_full", oracle_runs)


def test_cfg3_batched_full_bench_path(oracle_runs):
    _full_run("cfg3_full", oracle_runs)


def test_cfg4_large_T200_all_mixtures_50_sweeps(oracle_runs):
    _full_run("cfg4_T200", oracle_runs)


def test_cfg4_large_full_first_sweep(oracle_runs):
    _full_run("cfg4_full_sweep1", oracle_runs)
