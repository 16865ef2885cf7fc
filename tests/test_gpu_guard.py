"""Bounds checking of the CUDA path without compute-sanitizer (closed on this pool: DESIGN §9).

With NFHMM_GUARD set, every workspace piece is followed (and the first preceded) by a zone of 0xA5
bytes that starts at the piece's exact byte count; nfhmm_guard_check counts zone bytes a kernel or copy
overwrote (include/nfhmm.h).  Each launch path of the sweep -- tensor-core and SIMT engines, split-K,
CTA pairs, the deferred back-projection beside the multi-chain / parallel-in-time / wide recursions,
CUDA graphs, the fused and frame-tile Dirichlet variants, 3xTF32 products, ragged edge shapes -- runs
with guards, and must (1) leave every zone intact and (2) produce results bitwise equal to an unguarded
handle, so no kernel reads past a piece either (a read of a zone sees 0xA5 instead of the 0 padding).
Caller-owned device outputs are checked the same way from Python: views into sentinel-filled buffers.
"""
import numpy as np
import pytest

from tests.gpu_common import make_inputs, run_gpu

pytestmark = pytest.mark.gpu

GUARD = "4096"
KEYS = ("d_hat", "alpha_hat", "V_hat", "free_energy", "V_star", "V_src")

# (name, config, input overrides, sweeps, environment switches, engine)
CASES = [
    ("cfg0-graphs-pfb-splitk", 0, dict(), 20, {}, "tc"),
    ("cfg0-simt", 0, dict(), 6, {}, "simt"),
    ("cfg1-T1000-splitk-pfb", 1, dict(), 4, {}, "tc"),
    ("cfg2-T300-S3", 2, dict(T=300), 4, {}, "tc"),
    ("cfg3-M34-overlap-defer-multichain", 3, dict(M=34, T=2000), 3, {}, "tc"),
    ("cfg3-M19-pair-oddtiles", 3, dict(M=19, T=500), 3, {"NFHMM_OVERLAP": "0"}, "tc"),
    ("cfg3-M8-tf32", 3, dict(M=8, T=300), 3, {"NFHMM_RECON": "tf32", "NFHMM_BACKPROJ": "tf32"}, "tc"),
    ("cfg3-M6-fused-dirichlet", 3, dict(M=6, T=300), 3, {"NFHMM_FUSED": "1"}, "tc"),
    ("cfg3-M6-tile-dirichlet", 3, dict(M=6, T=300), 3, {"NFHMM_DIRICHLET": "tile"}, "tc"),
    ("cfg3-M40-tc-fb", 3, dict(M=40, T=64), 3, {"NFHMM_FB_MULTI": "2"}, "tc"),
    ("cfg4-T200-wide-fb", 4, dict(M=2, T=200), 2, {}, "tc"),
    ("edge-F9-T257", 0, dict(S=3, N=2, K=3, F=9, T=257, counts=500), 6, {}, "tc"),
    ("edge-T1", 0, dict(S=1, N=3, K=2, F=17, T=1, counts=500), 6, {}, "tc"),
    ("edge-N33-K1", 0, dict(S=2, N=33, K=1, F=40, T=31, counts=500), 6, {}, "simt"),
]


@pytest.mark.parametrize("name,c,over,iters,env,math", CASES, ids=[c[0] for c in CASES])
def test_guard_zones_intact_and_results_unchanged(name, c, over, iters, env, math, monkeypatch):
    cfg, model, V = make_inputs(c, **over)
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    monkeypatch.delenv("NFHMM_GUARD", raising=False)
    plain = run_gpu(cfg, model, V, iters, math=math)
    monkeypatch.setenv("NFHMM_GUARD", GUARD)
    guarded = run_gpu(cfg, model, V, iters, math=math, guard=True)
    checked, bad, msg = guarded["guard"]
    assert checked > 0
    assert bad == 0, f"{name}: {msg}"
    for key in KEYS:
        assert np.array_equal(plain[key], guarded[key]), f"{name}: {key} differs with guard zones"


def test_guard_check_detects_overwrites(monkeypatch):
    """Positive control: bytes written into the leading zone and the trailing one are counted."""
    import torch
    from paper_1206_6468_b200.nfhmm import NFHMM
    cfg, model, V = make_inputs(0)
    monkeypatch.setenv("NFHMM_GUARD", GUARD)
    h = NFHMM(cfg.F, cfg.T, cfg.S, cfg.N, cfg.K, n_mix=V.shape[0])
    h.set_model(model.beta, model.trans, model.prior)
    h.set_observations(np.ascontiguousarray(V))
    h.vb_iterate(2)
    checked, bad, _ = h.guard_check()
    assert checked >= 2 * int(GUARD) and bad == 0
    h.workspace[5] = 0
    h.workspace[-1] = 7
    h.workspace[-2] = 0xA5          # unchanged value: not counted
    torch.cuda.synchronize()
    checked2, bad2, msg = h.guard_check()
    assert checked2 == checked and bad2 == 2
    assert "piece -1" in msg
    h.close()


def _sentinel(shape, dtype, pad=4096):
    import torch
    n = int(np.prod(shape))
    buf = torch.full((pad + n + pad,), float("nan"), dtype=dtype, device="cuda")
    return buf, buf[pad:pad + n].view(*shape)


def test_device_outputs_written_only_inside_their_extent():
    """posteriors / separate into caller-owned device buffers write exactly their extents (views into
    NaN-filled buffers keep every NaN outside the view) and equal the host-buffer outputs."""
    import torch
    from paper_1206_6468_b200.nfhmm import NFHMM, nfhmm_posteriors, nfhmm_separate
    cfg, model, V = make_inputs(0, S=3, N=2, K=3, F=9, T=257, counts=500)
    M, S, T, N, F, Kt = V.shape[0], cfg.S, cfg.T, cfg.N, cfg.F, cfg.S * cfg.N * cfg.K
    h = NFHMM(F, T, S, N, cfg.K, n_mix=M, max_iters=8)
    h.set_model(model.beta, model.trans, model.prior)
    h.set_observations(np.ascontiguousarray(V))
    h.vb_iterate(5)
    host = h.posteriors()
    vst_h, vs_h = h.separate(V_src=True)
    outs = {"d": _sentinel((M, S, T, N), torch.float32), "a": _sentinel((M, T, Kt), torch.float32),
            "v": _sentinel((M, T, F), torch.float32), "fe": _sentinel((M, 8), torch.float64),
            "vst": _sentinel((M, S, T, F), torch.float32), "vs": _sentinel((M, S, T, F), torch.float32)}
    nfhmm_posteriors(h.h, outs["d"][1], outs["a"][1], outs["v"][1], outs["fe"][1])
    nfhmm_separate(h.h, outs["vst"][1], outs["vs"][1])
    torch.cuda.synchronize()
    for k, (buf, view) in outs.items():
        pad = buf.numel() - view.numel()
        assert torch.isnan(buf[:4096]).all() and torch.isnan(buf[4096 + view.numel():]).all(), k
        assert pad == 8192
    assert np.array_equal(outs["d"][1].cpu().numpy(), host["d_hat"])
    assert np.array_equal(outs["a"][1].cpu().numpy(), host["alpha_hat"])
    assert np.array_equal(outs["v"][1].cpu().numpy(), host["V_hat"])
    assert np.array_equal(outs["fe"][1].cpu().numpy()[:, :5], host["free_energy"])
    assert np.array_equal(outs["vst"][1].cpu().numpy(), vst_h)
    assert np.array_equal(outs["vs"][1].cpu().numpy(), vs_h)
    h.close()


@pytest.mark.parametrize("win,hop,n", [(1024, 256, 16000 + 77), (64, 48, 1000), (8, 8, 8)])
def test_stft_istft_device_outputs_inside_their_extent(win, hop, n):
    """nfhmm_stft / nfhmm_istft into caller-owned device buffers (views into NaN-filled buffers, ragged
    signal lengths): nothing outside the views changes, and the views equal the host-buffer outputs."""
    import torch
    from paper_1206_6468_b200 import nfhmm as nf
    lib = nf.library()
    rng = np.random.default_rng(1206)
    x = rng.standard_normal((3, n)).astype(np.float32)
    T, F = 1 + (n - win) // hop, win // 2 + 1
    ref = nf.stft(x, win=win, hop=hop, gain=3.0)
    xd = torch.from_numpy(x).cuda()
    Xb, Xv = _sentinel((3, T, F, 2), torch.float32)
    Vb, Vv = _sentinel((3, T, F), torch.float32)
    st = lib.nfhmm_stft(xd.data_ptr(), 3, n, win, hop, 3.0, Xv.data_ptr(), Vv.data_ptr(), 0,
                        nf._stream_ptr(None, 0))
    assert st == 0
    torch.cuda.synchronize()
    for buf, view in ((Xb, Xv), (Vb, Vv)):
        assert torch.isnan(buf[:4096]).all() and torch.isnan(buf[4096 + view.numel():]).all()
    assert np.array_equal(Xv.cpu().numpy().view(np.complex64)[..., 0], ref["X"])
    assert np.array_equal(Vv.cpu().numpy(), ref["V"])
    M = np.stack([ref["V"] * 0.25, ref["V"] * 0.75], axis=1).astype(np.float32)      # [3][2][T][F]
    y_ref = nf.istft(ref["X"], M, n, win=win, hop=hop, gain=3.0)
    yb, yv = _sentinel((3, 2, n), torch.float32)
    st = lib.nfhmm_istft(Xv.data_ptr(), torch.from_numpy(M).cuda().data_ptr(), 3, 2, T, win, hop, 3.0,
                         yv.data_ptr(), n, 0, nf._stream_ptr(None, 0))
    assert st == 0
    torch.cuda.synchronize()
    assert torch.isnan(yb[:4096]).all() and torch.isnan(yb[4096 + yv.numel():]).all()
    assert np.array_equal(yv.cpu().numpy(), y_ref)


@pytest.mark.parametrize("c,over", [(0, {}), (4, dict(T=40, N=70, K=4, F=65)), (0, dict(T=1))])
def test_trainer_device_outputs_inside_their_extent(c, over):
    """nhmm_train_get into caller-owned device buffers (views into NaN-filled buffers): nothing outside
    the views changes, and the views equal the host-buffer outputs (N-HMM EM training, NEXT-3)."""
    import ctypes
    import torch
    from paper_1206_6468_b200 import nfhmm as nf
    from paper_1206_6468_b200 import synth
    cfg = synth.config(c, **over)
    seed = synth.seed_of(c)
    model = synth.make_model(cfg, seed)
    V = synth.make_training_data(cfg, model, seed)
    b0, a0, p0 = synth.make_em_init(cfg, seed)
    S, T, N, K, F = V.shape[0], V.shape[1], cfg.N, cfg.K, cfg.F
    tr = nf.NHMMTrainer(F, T, N, K, n_src=S, max_iters=4)
    tr.set_data(V)
    tr.set_params(b0, a0, p0)
    tr.em(3)
    host = tr.get()
    outs = [_sentinel((S, N, K, F), torch.float32), _sentinel((S, N, N), torch.float32),
            _sentinel((S, N), torch.float32), _sentinel((S, T, N, K), torch.float32),
            _sentinel((S, 4), torch.float64)]
    it = ctypes.c_int32()
    st = nf.library().nhmm_train_get(tr.h, *[v.data_ptr() for _, v in outs], ctypes.byref(it))
    assert st == 0 and it.value == 3
    torch.cuda.synchronize()
    for buf, view in outs:
        assert torch.isnan(buf[:4096]).all() and torch.isnan(buf[4096 + view.numel():]).all()
    for (_, view), key in zip(outs, ("dict", "trans", "prior", "weights")):
        assert np.array_equal(view.cpu().numpy(), host[key]), key
    assert np.array_equal(outs[4][1].cpu().numpy()[:, :3], host["loglik"])
    tr.close()


@pytest.mark.parametrize("c,over,iters", [(3, dict(M=34, T=2000), 3), (1, dict(), 6), (3, dict(M=19, T=500), 4)])
def test_repeated_runs_are_bitwise_identical(c, over, iters):
    """Race detection without racecheck: the launch paths with concurrency between CTAs or streams (the
    recursion beside the capped contractions on a side stream, CUDA graphs, CTA pairs sharing multicast
    images and commit barriers, atomicMax row maxima, split-K partials, the parallel-in-time scan) run
    four times on fresh handles; a data race would show up as run-to-run differences in some output."""
    cfg, model, V = make_inputs(c, **over)
    runs = [run_gpu(cfg, model, V, iters) for _ in range(4)]
    for r in runs[1:]:
        for key in KEYS:
            assert np.array_equal(runs[0][key], r[key]), key
