"""Quick per-kernel timing + first-sweep accuracy on a config-3-shaped batch (development helper, GPU).

  python scripts/perf_quick.py [--mixtures 64] [--iters 10] [--math tc] [--config 3]

Prints ms per launch of each kernel class (CUDA events bracketing each launch, nfhmm_profile_*).
Accuracy against the oracle is checked by tests/ only (the oracle is test infrastructure).
"""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_1206_6468_b200 import synth  # noqa: E402
from paper_1206_6468_b200.nfhmm import NFHMM  # noqa: E402


ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=3)
ap.add_argument("--mixtures", type=int, default=64)
ap.add_argument("--T", type=int, default=None)
ap.add_argument("--iters", type=int, default=10)
ap.add_argument("--math", default="tc")
ap.add_argument("--kernels", default="", help="comma list of classes to time alone with nfhmm_bench_kernel")
a = ap.parse_args()

over = dict(M=a.mixtures)
if a.T:
    over["T"] = a.T
cfg = synth.config(a.config, **over)
seed = synth.seed_of(a.config)
model = synth.make_model(cfg, seed)
V = synth.make_batch(cfg, model, seed, range(cfg.M))
h = NFHMM(cfg.F, cfg.T, cfg.S, cfg.N, cfg.K, n_mix=cfg.M, math=a.math)
h.set_model(model.beta, model.trans, model.prior)
h.set_observations(V)
if a.kernels:   # time the named kernel classes alone and stop (works under NFHMM_TC_DEBUG experiments)
    for k in a.kernels.split(","):
        print(f"alone: {k:10s} ms/launch {h.bench_kernel(k, 10):8.3f}")
    sys.exit(0)
h.vb_iterate(2)
h.reset()
h.profile_enable(True)
h.vb_iterate(a.iters)
prof = h.profile_read()
frames = cfg.M * cfg.T
tot = 0.0
for n, (ms, cnt) in prof.items():
    if cnt:
        tot += ms
        print(f"{n:10s} launches {cnt:4d}  ms/launch {ms / cnt:8.3f}")
print(f"total {tot:.2f} ms for {a.iters} sweeps -> {frames * a.iters / tot * 1e3 / 1e6:.2f} M frame-iter/s")
h.close()
