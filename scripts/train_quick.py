"""Timing of the N-HMM EM trainer on an isolated-source batch (development helper, GPU).
  python scripts/train_quick.py [--config 1] [--T 2000] [--iters 10]"""
import argparse, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1206_6468_b200 import synth
from paper_1206_6468_b200.nfhmm import NHMMTrainer
ap = argparse.ArgumentParser(); ap.add_argument("--config", type=int, default=1); ap.add_argument("--T", type=int, default=2000)
ap.add_argument("--iters", type=int, default=10); a = ap.parse_args()
cfg = synth.config(a.config); seed = synth.seed_of(a.config); model = synth.make_model(cfg, seed)
V = synth.make_training_data(cfg, model, seed, a.T); b0, a0, p0 = synth.make_em_init(cfg, seed)
tr = NHMMTrainer(cfg.F, a.T, cfg.N, cfg.K, n_src=cfg.S, max_iters=a.iters + 2)
tr.set_data(torch.from_numpy(V).cuda()); tr.set_params(b0, a0, p0); tr.em(2)
tr.set_params(b0, a0, p0)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); tr.em(a.iters); e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1)
print(f"S={cfg.S} N={cfg.N} K={cfg.K} F={cfg.F} T={a.T}: {ms / a.iters:.3f} ms per EM iteration -> "
      f"{cfg.S * a.T * a.iters / ms * 1e3 / 1e6:.3f} M frame-iterations/s; loglik {tr.get()['loglik'][:, -1]}")
