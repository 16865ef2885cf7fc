"""Isolate the Dirichlet kernel's psi/exp accuracy: V_hat(GPU) vs beta . exp(psi(alpha_gpu) - psi(sum alpha_gpu))
evaluated in float64 (debug helper)."""
import sys
import numpy as np
from scipy.special import digamma
sys.path.insert(0, ".")
from tests.gpu_common import make_inputs, rel_l2, run_gpu

for c, ov in [(1, dict(T=200)), (3, dict(T=300, M=1))]:
    cfg, model, V = make_inputs(c, **ov)
    for math in ("simt", "tc"):
        g = run_gpu(cfg, model, V, 2, math=math, separate=False)
        a = g["alpha_hat"][0].astype(np.float64)
        th = np.exp(digamma(a) - digamma(a.sum(1, keepdims=True)))
        vh = th @ model.beta.reshape(cfg.Kt, cfg.F).astype(np.float64)
        print(c, math, "V_hat vs exact-from-gpu-alpha", rel_l2(g["V_hat"][0], vh), flush=True)
