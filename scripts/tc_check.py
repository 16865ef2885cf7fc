"""Quick numerics check of the tcgen05 3xTF32 path vs the SIMT path and the oracle (debug helper)."""
import sys, time
import numpy as np
sys.path.insert(0, ".")
from tests.gpu_common import make_inputs, rel_l2, run_gpu, run_oracle

for c, ov, iters in [(0, {}, 1), (1, dict(T=200), 1), (3, dict(T=300, M=2), 3), (2, dict(T=100), 2)]:
    cfg, model, V = make_inputs(c, **ov)
    t = time.time()
    g = {m: run_gpu(cfg, model, V, iters, math=m) for m in ("simt", "tc")}
    o = run_oracle(cfg, model, V[0], iters)
    for m in ("simt", "tc"):
        print(f"cfg{c} {ov} iters={iters} {m}: dhat {rel_l2(g[m]['d_hat'][0], o['d_hat']):.2e} "
              f"vhat {rel_l2(g[m]['V_hat'][0], o['V_hat']):.2e} alpha {rel_l2(g[m]['alpha_hat'][0], o['alpha']):.2e} "
              f"L {np.max(np.abs(g[m]['free_energy'][0]-o['free_energy'])/np.abs(o['free_energy'])):.2e} "
              f"vstar {rel_l2(g[m]['V_star'][0], o['V_star']):.2e}", flush=True)
