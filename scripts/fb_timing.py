"""Standalone FB timing at config 3 through three methods (profile events, bench_kernel, overlap off)."""
import sys, time
sys.path.insert(0, '.')
import numpy as np, torch
from paper_1206_6468_b200 import synth
from paper_1206_6468_b200.nfhmm import NFHMM
cfg = synth.config(3); seed = synth.seed_of(3); model = synth.make_model(cfg, seed)
V = synth.make_batch(cfg, model, seed, range(cfg.M))
h = NFHMM(cfg.F, cfg.T, cfg.S, cfg.N, cfg.K, n_mix=cfg.M, max_iters=64)
h.set_model(model.beta, model.trans, model.prior); h.set_observations(torch.from_numpy(V).cuda())
h.vb_iterate(3)
for cls in ("fb", "dirichlet", "recon", "backproj"):
    print(cls, "bench_kernel ms", h.bench_kernel(cls, 20))
h.vb_iterate(3)
h.profile_enable(True); h.vb_iterate(10); p = h.profile_read(); h.profile_enable(False)
print({k: (round(v[0] / max(v[1], 1), 4), v[1]) for k, v in p.items()})
vst = torch.empty((cfg.M, cfg.S, cfg.T, cfg.F), dtype=torch.float32, device="cuda")
for rep in range(2):
    h.profile_enable(True)
    h.reset(); h.vb_iterate_async(50); h.separate_into(vst)
    torch.cuda.synchronize()
    p = h.profile_read(); h.profile_enable(False)
    print("bench-like", {k: (round(v[0] / max(v[1], 1), 4), v[1]) for k, v in p.items()})
h2 = NFHMM(cfg.F, cfg.T, cfg.S, cfg.N, cfg.K, n_mix=cfg.M, max_iters=64, free_energy=False)
h2.set_model(model.beta, model.trans, model.prior); h2.set_observations(torch.from_numpy(V).cuda())
h2.profile_enable(True); h2.vb_iterate(10); p = h2.profile_read(); h2.profile_enable(False)
print("bound off", {k: (round(v[0] / max(v[1], 1), 4), v[1]) for k, v in p.items()})
