"""Multi-process (world size 2, gloo, CPU) tests of the sharding / gather plumbing of bench.py's N > 1
path.  The per-mixture compute here is the CPU oracle (tests may call it); what is tested is that every
mixture lands on exactly one rank, is generated identically there, and comes back in global order."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_1206_6468_b200 import dist as pdist
from paper_1206_6468_b200 import synth


def test_shard_partitions_exactly():
    for M in (0, 1, 3, 256, 64, 7):
        for world in (1, 2, 3, 4, 8):
            got = [m for r in range(world) for m in pdist.shard(M, world, r)]
            assert got == list(range(M))
            sizes = [len(pdist.shard(M, world, r)) for r in range(world)]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        pdist.shard(4, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, M, iters, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import oracle
    cfg = synth.config(0, M=M, T=20)
    seed = synth.seed_of(0)
    model = synth.make_model(cfg, seed)
    mine = pdist.shard(M, world, rank)
    traces = []
    for m in mine:
        V = synth.make_mixture(cfg, model, seed, m).V
        traces.append(oracle.vb_run(model.beta, model.trans, model.prior, V, cfg.dims, iters)["free_energy"])
    local = np.array(traces).reshape(len(mine), iters)
    full = pdist.gather_mixtures(local, M)
    tmax = pdist.max_over_ranks(float(rank + 1))
    if rank == 0:
        q.put((full, tmax))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("M", [3, 4])
def test_gloo_world2_gather_matches_single_process(M):
    iters = 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, M, iters, q)) for r in range(2)]
    for p in procs:
        p.start()
    full, tmax = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert tmax == 2.0
    from oracle import oracle
    cfg = synth.config(0, M=M, T=20)
    seed = synth.seed_of(0)
    model = synth.make_model(cfg, seed)
    ref = np.array([oracle.vb_run(model.beta, model.trans, model.prior, synth.make_mixture(cfg, model, seed, m).V,
                                  cfg.dims, iters)["free_energy"] for m in range(M)])
    np.testing.assert_array_equal(full, ref)   # same mixtures, same order, bitwise


def test_mixture_generation_is_rank_independent():
    cfg = synth.config(3, T=30, M=5)
    seed = synth.seed_of(3)
    model = synth.make_model(cfg, seed)
    a = synth.make_batch(cfg, model, seed, range(5), workers=1)
    b = np.concatenate([synth.make_batch(cfg, model, seed, pdist.shard(5, 2, r), workers=1) for r in range(2)])
    np.testing.assert_array_equal(a, b)
    assert (a.sum(-1) == cfg.counts).all()
