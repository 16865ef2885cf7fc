"""Shared helpers of the GPU parity tests: run the CUDA path (through the C-ABI) and the oracle on the
same seeded synthetic inputs.  Inputs come only from paper_1206_6468_b200.synth; expected values only
from oracle/ (never from the CUDA path)."""
import json
import os

import numpy as np

from paper_1206_6468_b200 import synth

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def rel_l2(x, ref):
    x = np.asarray(x, np.float64)
    ref = np.asarray(ref, np.float64)
    den = np.linalg.norm(ref.ravel())
    return float(np.linalg.norm((x - ref).ravel()) / (den if den > 0 else 1.0))


def make_inputs(c, **override):
    cfg = synth.config(c, **override)
    seed = synth.seed_of(c)
    model = synth.make_model(cfg, seed)
    V = synth.make_batch(cfg, model, seed, range(cfg.M), workers=1)
    return cfg, model, V


def run_gpu(cfg, model, V, iters, gamma=1.0, separate=True, max_iters=1024, device_io=False, split=None,
            math="tc", guard=False):
    """Run the CUDA path: set_model, set_observations, vb_iterate(iters) (optionally split into several
    calls), posteriors (+ separate).  Returns dict of host numpy arrays."""
    import torch
    from paper_1206_6468_b200.nfhmm import NFHMM
    M = V.shape[0]
    h = NFHMM(cfg.F, cfg.T, cfg.S, cfg.N, cfg.K, n_mix=M, gamma=gamma, max_iters=max_iters, math=math)
    if device_io:
        h.set_model(torch.from_numpy(model.beta).cuda(), torch.from_numpy(model.trans).cuda(),
                    torch.from_numpy(model.prior).cuda())
        h.set_observations(torch.from_numpy(np.ascontiguousarray(V)).cuda())
    else:
        h.set_model(model.beta, model.trans, model.prior)
        h.set_observations(np.ascontiguousarray(V))
    for n in (split or [iters]):
        h.vb_iterate(n)
    out = h.posteriors()
    if separate:
        vst, vs = h.separate(V_src=True)
        out["V_star"], out["V_src"] = vst, vs
    out["launches"] = h.kernel_launches()
    if guard:   # NFHMM_GUARD zones of the workspace (include/nfhmm.h nfhmm_guard_check)
        out["guard"] = h.guard_check()
    h.close()
    return out


def run_oracle(cfg, model, Vm, iters, gamma=1.0, separate=True):
    from oracle import oracle
    r = oracle.vb_run(model.beta, model.trans, model.prior, Vm, cfg.dims, iters, gamma)
    if separate:
        vs, vst = oracle.separate(model.beta, Vm, r["alpha"], cfg.dims)
        r["V_src"], r["V_star"] = vs, vst
    return r


RECORD_PATH = os.environ.get("NFHMM_PARITY_LOG", os.path.join(ROOT, "gpurun_out", "parity_records.jsonl"))


def record(tag, quantity, **vals):
    """Append one parity measurement (JSON line) to the parity record and print it."""
    line = dict(tag=tag, quantity=quantity, **{k: (float(v) if isinstance(v, (np.floating, float)) else v)
                                                for k, v in vals.items()})
    print("PARITY", json.dumps(line))
    try:
        os.makedirs(os.path.dirname(RECORD_PATH), exist_ok=True)
        with open(RECORD_PATH, "a") as f:
            f.write(json.dumps(line) + "\n")
    except OSError:
        pass


def compare(tag, quantity, x, ref, tol):
    """rel-L2 gate (DESIGN R13) with max-abs and max-relative logged beside it."""
    x = np.asarray(x, np.float64)
    ref = np.asarray(ref, np.float64)
    r = rel_l2(x, ref)
    diff = np.abs(x - ref)
    mx = float(diff.max()) if diff.size else 0.0
    scale = float(np.abs(ref).max()) if ref.size else 0.0
    record(tag, quantity, rel_l2=r, max_abs=mx, max_abs_over_max_ref=(mx / scale if scale > 0 else 0.0), tol=tol)
    assert r <= tol, (tag, quantity, r)
    return r
