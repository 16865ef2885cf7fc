"""The frame-chunked oracle driver used by the full-size parity tests (tests/oracle_jobs.py) computes
what or_vb_run computes: same state after every sweep, same bound trace, same separation.  Only the FP64
order of the chunk partial sums differs, so values agree to ~1e-15 relative."""
import numpy as np
import pytest

from paper_1206_6468_b200 import synth
from tests import oracle_jobs


@pytest.fixture(scope="module")
def pool():
    ex = oracle_jobs.make_pool(4)
    yield ex
    ex.shutdown()


@pytest.mark.parametrize("c,T,iters,chunks,gamma", [(0, 50, 6, 7, 1.0), (0, 23, 1, 4, 2.5), (2, 9, 3, 3, 1.0)])
def test_frame_chunked_driver_equals_vb_run(oracle, pool, tmp_path, c, T, iters, chunks, gamma):
    cfg = synth.config(c, T=T, F=min(synth.config(c).F, 40), N=min(synth.config(c).N, 5), counts=3000)
    seed = synth.seed_of(c)
    model = synth.make_model(cfg, seed)
    V = synth.make_mixture(cfg, model, seed, 0).V
    bp = oracle_jobs.save_beta(model.beta, str(tmp_path), f"c{c}")
    got = oracle_jobs.vb_run_frames(pool, bp, model.trans, model.prior, V, cfg.dims, iters, gamma, chunks=chunks)
    ref = oracle.vb_run(model.beta, model.trans, model.prior, V, cfg.dims, iters, gamma)
    for key in ("alpha", "d_hat", "V_hat", "logZ"):
        np.testing.assert_allclose(got[key], ref[key], rtol=1e-12, atol=0, err_msg=key)
    np.testing.assert_allclose(got["free_energy"], ref["free_energy"], rtol=1e-13)
    one = oracle.vb_run(model.beta, model.trans, model.prior, V, cfg.dims, 1, gamma)
    for key in ("alpha", "d_hat", "V_hat", "free_energy"):
        np.testing.assert_allclose(got["first"][key], one[key], rtol=1e-12, err_msg="first " + key)
    vs, vst = oracle.separate(model.beta, V, ref["alpha"], cfg.dims)
    np.testing.assert_allclose(got["V_src"], vs, rtol=1e-12)
    np.testing.assert_allclose(got["V_star"], vst, rtol=1e-12)
