"""Multi-process run of the LIBRARY (not the oracle): two ranks, each driving libnfhmm on its shard of a
batched configuration (the mixture sharding of bench.py --gpus N), gather the free-energy
traces and posteriors over torch.distributed (gloo: both ranks share the one GPU of the test box, and
their kernels never wait on each other), and compare with one rank running every mixture: the per-mixture
results are bitwise identical (fixed-order reductions; the sharding invariant of SURVEY §8(e))."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_1206_6468_b200 import dist as pdist
from paper_1206_6468_b200 import synth

pytestmark = pytest.mark.gpu

CASE = dict(T=150, M=5, counts=5000)
ITERS = 6


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _run_lib(cfg, model, V, iters):
    from paper_1206_6468_b200.nfhmm import NFHMM
    h = NFHMM(cfg.F, cfg.T, cfg.S, cfg.N, cfg.K, n_mix=V.shape[0], max_iters=iters)
    h.set_model(model.beta, model.trans, model.prior)
    h.set_observations(np.ascontiguousarray(V))
    h.vb_iterate(iters)
    p = h.posteriors(alpha_hat=False, V_hat=False)
    vst = h.separate()
    h.close()
    return p["free_energy"], p["d_hat"], vst


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg = synth.config(3, **CASE)
    seed = synth.seed_of(3)
    model = synth.make_model(cfg, seed)
    mine = pdist.shard(cfg.M, world, rank)
    V = synth.make_batch(cfg, model, seed, mine, workers=1)
    fe, d, vst = _run_lib(cfg, model, V, ITERS)
    fe_all = pdist.gather_mixtures(fe, cfg.M)
    d_all = pdist.gather_mixtures(d.reshape(len(mine), -1), cfg.M)
    v_all = pdist.gather_mixtures(vst.reshape(len(mine), -1), cfg.M)
    if rank == 0:
        q.put((fe_all, d_all, v_all))
    dist.barrier()
    dist.destroy_process_group()


def test_two_ranks_on_the_library_gather_bitwise_equal_to_one_rank():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    fe_all, d_all, v_all = q.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    cfg = synth.config(3, **CASE)
    seed = synth.seed_of(3)
    model = synth.make_model(cfg, seed)
    V = synth.make_batch(cfg, model, seed, range(cfg.M), workers=1)
    fe, d, vst = _run_lib(cfg, model, V, ITERS)
    np.testing.assert_array_equal(fe_all, fe)
    np.testing.assert_array_equal(d_all, d.reshape(cfg.M, -1).astype(np.float64))
    np.testing.assert_array_equal(v_all, vst.reshape(cfg.M, -1).astype(np.float64))
