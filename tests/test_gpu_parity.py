"""GPU parity: the CUDA path (through the C-ABI) against the FP64 oracle on the same seeded inputs.

Tolerances (BASELINE.json north_star):
  after 1 sweep:             d_hat, V_hat (and alpha_hat) rel-L2 <= 1e-5
  after the config's sweeps: V_star rel-L2 <= 1e-3, free energy rel <= 1e-5 (every sweep)
  every sweep (GPU):         free energy non-decreasing within 1e-6 |L|
Sizes span several 128-frame tiles with a ragged tail; configs 1-4 are run at reduced T / M here and
at full size in test_gpu_fullsize.py.
"""
import numpy as np
import pytest

from tests.gpu_common import compare, make_inputs, rel_l2, run_gpu, run_oracle

pytestmark = pytest.mark.gpu

TOL1 = 1e-5
TOL_VSTAR = 1e-3
TOL_L = 1e-5


MATHS = ["tc", "simt"]


def check_parity(cfg, model, V, iters, gamma=1.0, mixtures=None, tol1=TOL1, math="tc"):
    g1 = run_gpu(cfg, model, V, 1, gamma=gamma, separate=False, math=math)
    gn = run_gpu(cfg, model, V, iters, gamma=gamma, math=math)
    tag = f"{cfg.name}:S{cfg.S}N{cfg.N}K{cfg.K}F{cfg.F}T{cfg.T}M{V.shape[0]}:g{gamma}:{math}"
    for m in (mixtures if mixtures is not None else range(V.shape[0])):
        o1 = run_oracle(cfg, model, V[m], 1, gamma=gamma, separate=False)
        compare(f"{tag}/m{m}/sweep1", "d_hat", g1["d_hat"][m], o1["d_hat"], tol1)
        compare(f"{tag}/m{m}/sweep1", "V_hat", g1["V_hat"][m], o1["V_hat"], tol1)
        compare(f"{tag}/m{m}/sweep1", "alpha_hat", g1["alpha_hat"][m], o1["alpha"], tol1)
        assert abs(g1["free_energy"][m, 0] - o1["free_energy"][0]) <= TOL_L * abs(o1["free_energy"][0])
        on = run_oracle(cfg, model, V[m], iters, gamma=gamma)
        compare(f"{tag}/m{m}/sweep{iters}", "V_star", gn["V_star"][m], on["V_star"], TOL_VSTAR)
        compare(f"{tag}/m{m}/sweep{iters}", "V_src", gn["V_src"][m], on["V_src"], TOL_VSTAR)
        fe_g, fe_o = gn["free_energy"][m], on["free_energy"]
        assert fe_g.shape == fe_o.shape
        assert np.all(np.abs(fe_g - fe_o) <= TOL_L * np.abs(fe_o)), np.max(np.abs(fe_g - fe_o) / np.abs(fe_o))
        assert np.all(np.diff(fe_g) >= -1e-6 * np.abs(fe_g[1:]))
    return g1, gn


@pytest.mark.parametrize("math", MATHS)
def test_cfg0_tiny_full(math):
    cfg, model, V = make_inputs(0)
    g1, gn = check_parity(cfg, model, V, cfg.iters, math=math)
    assert gn["iters_done"] == cfg.iters


@pytest.mark.parametrize("math", MATHS)
def test_cfg1_reduced_T200(math):
    cfg, model, V = make_inputs(1, T=200)
    check_parity(cfg, model, V, 30, math=math)


@pytest.mark.parametrize("math", MATHS)
def test_cfg2_three_sources_reduced(math):
    cfg, model, V = make_inputs(2, T=150)
    check_parity(cfg, model, V, 20, math=math)


@pytest.mark.parametrize("math", MATHS)
def test_cfg3_batched_reduced_multi_mixture(math):
    cfg, model, V = make_inputs(3, T=300, M=3)
    check_parity(cfg, model, V, 15, math=math)


@pytest.mark.parametrize("math", MATHS)
def test_cfg4_large_reduced(math):
    cfg, model, V = make_inputs(4, T=40, M=2)
    check_parity(cfg, model, V, 4, mixtures=[1], math=math)


@pytest.mark.parametrize("gamma", [0.0, 2.5])
@pytest.mark.parametrize("math", MATHS)
def test_gamma_values(gamma, math):
    cfg, model, V = make_inputs(0, T=70)
    check_parity(cfg, model, V, 10, gamma=gamma, math=math)


@pytest.mark.parametrize("shape", [dict(S=1, N=3, K=2, F=17, T=1), dict(S=1, N=1, K=1, F=5, T=9),
                                   dict(S=2, N=1, K=5, F=64, T=129), dict(S=2, N=33, K=1, F=40, T=31),
                                   dict(S=3, N=2, K=3, F=9, T=257)])
@pytest.mark.parametrize("math", MATHS)
def test_edge_shapes(shape, math):
    cfg, model, V = make_inputs(0, counts=500, **shape)
    check_parity(cfg, model, V, 6, math=math)


def test_empty_frames_and_sharding_invariance():
    """Frames with V = 0 are legal (alpha = prior pseudo-counts); per-mixture results are bitwise the
    same whether a mixture runs alone or batched with others (the multi-GPU sharding invariant)."""
    cfg, model, V = make_inputs(3, T=150, M=3, counts=2000)
    V[1, 10:20] = 0.0
    batched = run_gpu(cfg, model, V, 5)
    for m in range(3):
        single = run_gpu(cfg, model, V[m:m + 1], 5)
        for key in ("d_hat", "alpha_hat", "V_hat", "free_energy", "V_star", "V_src"):
            np.testing.assert_array_equal(batched[key][m], single[key][0], err_msg=key)
    o = run_oracle(cfg, model, V[1], 5)
    assert rel_l2(batched["V_star"][1], o["V_star"]) <= TOL_VSTAR
    np.testing.assert_allclose(batched["V_star"][1].sum(0), V[1], rtol=1e-5, atol=1e-3)


@pytest.mark.parametrize("c,over", [(0, {}), (1, dict(T=300)), (3, dict(M=6, T=120))])
def test_resume_equals_single_call_and_device_io(c, over):
    """Sweeps split over several calls equal one call, bitwise, and device I/O equals host I/O.  Covers the
    CUDA-graph replays with the recursion beside the contractions and the deferred back-projection (config 0
    and the batch: sequential recursion; config 1: parallel in time), whose state crosses call boundaries."""
    cfg, model, V = make_inputs(c, **over)
    a = run_gpu(cfg, model, V, 7)
    b = run_gpu(cfg, model, V, 7, split=[3, 1, 3])
    c = run_gpu(cfg, model, V, 7, device_io=True)
    for key in ("d_hat", "alpha_hat", "V_hat", "free_energy", "V_star"):
        np.testing.assert_array_equal(a[key], b[key], err_msg=key)
        np.testing.assert_array_equal(a[key], c[key], err_msg=key)


def test_invariants_on_gpu_outputs():
    cfg, model, V = make_inputs(1, T=257)
    g = run_gpu(cfg, model, V, 10)
    np.testing.assert_allclose(g["d_hat"].sum(-1), 1.0, atol=2e-6)
    assert (g["alpha_hat"] >= 1.0).all()
    Kt = cfg.Kt
    np.testing.assert_allclose(g["alpha_hat"].sum(-1), V.sum(-1) + Kt + cfg.S * cfg.K, rtol=2e-6)
    np.testing.assert_allclose(g["V_star"].sum(1), V, rtol=1e-5, atol=1e-3)
    np.testing.assert_allclose(g["V_src"].sum((1, 3)), V.sum(-1), rtol=1e-5)


def test_errors_are_explicit():
    import torch
    from paper_1206_6468_b200.nfhmm import NFHMM, NFHMMError, NFHMM_EINVAL, NFHMM_ESTATE, NFHMM_EZEROSUPPORT
    cfg, model, V = make_inputs(0)
    h = NFHMM(cfg.F, cfg.T, cfg.S, cfg.N, cfg.K)
    with pytest.raises(NFHMMError) as e:
        h.vb_iterate(1)
    assert e.value.status == NFHMM_ESTATE
    bad = model.beta.copy()
    bad[0, 0, 0, 0] += 0.5
    with pytest.raises(NFHMMError) as e:
        h.set_model(bad, model.trans, model.prior)
    assert e.value.status == NFHMM_EINVAL
    h.set_model(model.beta, model.trans, model.prior)
    Vn = V.copy()
    Vn[0, 3, 4] = -1.0
    with pytest.raises(NFHMMError) as e:
        h.set_observations(Vn)
        h.vb_iterate(1)
    assert e.value.status == NFHMM_EINVAL
    # zero support: a bin no dictionary element covers, with counts in it
    zb = model.beta.copy()
    zb[..., 0] = 0.0
    zb /= zb.sum(-1, keepdims=True)
    h2 = NFHMM(cfg.F, cfg.T, cfg.S, cfg.N, cfg.K)
    h2.set_model(zb, model.trans, model.prior)
    Vz = V.copy()
    Vz[0, :, 0] = 3.0
    with pytest.raises(NFHMMError) as e:
        h2.set_observations(Vz)
        h2.vb_iterate(1)
    assert e.value.status == NFHMM_EZEROSUPPORT
    h.close()
    h2.close()


def test_bench_kernel_instrumentation_resets_state():
    """nfhmm_bench_kernel (per-kernel timing) leaves the handle reset: a run after it equals a fresh run
    bitwise; classes outside RECON..FB and reps < 1 are rejected."""
    from paper_1206_6468_b200.nfhmm import NFHMM, NFHMMError, NFHMM_EINVAL
    cfg, model, V = make_inputs(3, T=150, M=2, counts=2000)
    ref = run_gpu(cfg, model, V, 4, separate=False)
    h = NFHMM(cfg.F, cfg.T, cfg.S, cfg.N, cfg.K, n_mix=2)
    h.set_model(model.beta, model.trans, model.prior)
    h.set_observations(np.ascontiguousarray(V))
    h.vb_iterate(2)
    for cls in ("recon", "backproj", "dirichlet", "fb"):
        assert h.bench_kernel(cls, 3) > 0.0
    for bad in (("elbo", 1), ("recon", 0)):
        with pytest.raises(NFHMMError) as e:
            h.bench_kernel(*bad)
        assert e.value.status == NFHMM_EINVAL
    h.vb_iterate(4)
    out = h.posteriors()
    h.close()
    for key in ("d_hat", "alpha_hat", "V_hat", "free_energy"):
        np.testing.assert_array_equal(out[key], ref[key], err_msg=key)


@pytest.mark.parametrize("c,over", [(1, dict(T=400)), (2, dict(T=333)), (3, dict(T=250, M=2))])
def test_parallel_in_time_fb_matches_sequential(c, over, monkeypatch):
    """the chunked (parallel-in-time) forward-backward that few-chain handles use agrees with
    the sequential recursion (same products, another association order) and with the oracle."""
    cfg, model, V = make_inputs(c, **over)
    par = run_gpu(cfg, model, V, 6)
    monkeypatch.setenv("NFHMM_FB_PARALLEL", "0")
    seq = run_gpu(cfg, model, V, 6)
    for key in ("d_hat", "alpha_hat", "V_hat", "V_star"):
        assert rel_l2(par[key], seq[key]) <= 2e-6, key
    assert np.all(np.abs(par["free_energy"] - seq["free_energy"]) <= 1e-7 * np.abs(seq["free_energy"]))
    o = run_oracle(cfg, model, V[0], 6)
    assert rel_l2(par["V_star"][0], o["V_star"]) <= TOL_VSTAR
    assert np.all(np.abs(par["free_energy"][0] - o["free_energy"]) <= TOL_L * np.abs(o["free_energy"]))


@pytest.mark.parametrize("c,over", [(0, {}), (1, dict(T=300)), (3, dict(T=200, M=3))])
def test_fused_dirichlet_epilogue_matches_separate_kernel(c, over, monkeypatch):
    """Opt-in engine (NFHMM_FUSED=1): the Dirichlet element step in the back-projection GEMM's epilogue
    gives the separate kernel's results (same per-element arithmetic, other summation order of the Eq. 8
    block sums and of the bound terms) and the oracle's."""
    cfg, model, V = make_inputs(c, **over)
    sep = run_gpu(cfg, model, V, 5)
    monkeypatch.setenv("NFHMM_FUSED", "1")
    fus = run_gpu(cfg, model, V, 5)
    for key in ("d_hat", "alpha_hat", "V_hat", "V_star"):
        assert rel_l2(fus[key], sep[key]) <= 2e-6, key
    # the fused engine's back-projection is 3xTF32, the default's 3xFP16: the bound's data term moves by
    # ~1e-7 relative (round 2 measured L vs the oracle after one sweep: 2.1e-7 for 3xTF32, 8e-8 for 3xFP16)
    assert np.all(np.abs(fus["free_energy"] - sep["free_energy"]) <= 1e-6 * np.abs(sep["free_energy"]))
    o = run_oracle(cfg, model, V[0], 5)
    assert rel_l2(fus["V_star"][0], o["V_star"]) <= TOL_VSTAR
    assert np.all(np.abs(fus["free_energy"][0] - o["free_energy"]) <= TOL_L * np.abs(o["free_energy"]))


@pytest.mark.parametrize("c,over", [(0, {}), (2, dict(T=150))])
def test_frame_tile_dirichlet_variant_matches(c, over, monkeypatch):
    """Opt-in NFHMM_DIRICHLET=tile (frame-tile Dirichlet kernel: bulk copies, per-(frame, source) work
    spread over the CTA) agrees with the default kernel and the oracle."""
    cfg, model, V = make_inputs(c, **over)
    ref = run_gpu(cfg, model, V, 5)
    monkeypatch.setenv("NFHMM_DIRICHLET", "tile")
    tile = run_gpu(cfg, model, V, 5)
    for key in ("d_hat", "alpha_hat", "V_hat", "V_star"):
        assert rel_l2(tile[key], ref[key]) <= 2e-6, key
    assert np.all(np.abs(tile["free_energy"] - ref["free_energy"]) <= 1e-7 * np.abs(ref["free_energy"]))
    o = run_oracle(cfg, model, V[0], 5)
    assert rel_l2(tile["V_star"][0], o["V_star"]) <= TOL_VSTAR


@pytest.mark.parametrize("c,over", [(4, dict(T=120, M=2)), (4, dict(T=97, M=1, N=70))])
def test_wide_forward_backward_matches_one_warp_kernel(c, over, monkeypatch):
    """N > 64: the multi-warp forward-backward (a CTA of ceil(N/32) warps per chain and direction, A in
    registers) agrees with the one-warp kernel (A in shared memory) and with the oracle."""
    cfg, model, V = make_inputs(c, **over)
    wide = run_gpu(cfg, model, V, 4)
    monkeypatch.setenv("NFHMM_FB_WIDE", "0")
    one = run_gpu(cfg, model, V, 4)
    for key in ("d_hat", "alpha_hat", "V_hat", "V_star"):
        assert rel_l2(wide[key], one[key]) <= 2e-6, key
    assert np.all(np.abs(wide["free_energy"] - one["free_energy"]) <= 1e-7 * np.abs(one["free_energy"]))
    o = run_oracle(cfg, model, V[0], 4)
    assert rel_l2(wide["V_star"][0], o["V_star"]) <= TOL_VSTAR
    assert np.all(np.abs(wide["free_energy"][0] - o["free_energy"]) <= TOL_L * np.abs(o["free_energy"]))


@pytest.mark.parametrize("graphs", ["0", "1"])
def test_fb_overlap_is_bitwise_neutral(graphs, monkeypatch):
    """Large batches run the forward-backward beside the reconstruction GEMM (grid capped at num_SMs - 32,
    side stream, fork/join; also inside CUDA graphs): every tile and recursion is computed exactly as
    without the overlap, so the results are bitwise identical."""
    cfg, model, V = make_inputs(3, M=34, T=2000)          # 68,000 frames > 65,536: overlap on by default
    monkeypatch.setenv("NFHMM_GRAPHS", graphs)
    ov = run_gpu(cfg, model, V, 3, separate=False)
    monkeypatch.setenv("NFHMM_OVERLAP", "0")
    seq = run_gpu(cfg, model, V, 3, separate=False)
    for key in ("d_hat", "alpha_hat", "V_hat", "free_energy"):
        assert np.array_equal(ov[key], seq[key]), key


def test_cta_pair_multicast_is_bitwise_neutral(monkeypatch):
    """Many row tiles: the contractions run as clusters of two CTAs that share every dictionary image by
    TMA multicast (each fetches half).  297 row tiles (odd: the last pair's second CTA computes on zero
    fill past the end and stores nothing) -- bitwise equal to the unpaired kernel, and the last mixture
    (whose frames end in the unpaired tail) matches the oracle after one sweep and after four."""
    cfg, model, V = make_inputs(3, M=19, T=2000)          # 38,000 frames = 297 row tiles of 128
    paired = run_gpu(cfg, model, V, 4)
    one = run_gpu(cfg, model, V, 1, separate=False)
    monkeypatch.setenv("NFHMM_TC_PAIR", "0")
    single = run_gpu(cfg, model, V, 4)
    for key in ("d_hat", "alpha_hat", "V_hat", "V_star", "free_energy"):
        assert np.array_equal(paired[key], single[key]), key
    m = V.shape[0] - 1
    o1 = run_oracle(cfg, model, V[m], 1, separate=False)
    for key, okey in (("d_hat", "d_hat"), ("V_hat", "V_hat"), ("alpha_hat", "alpha")):
        compare(f"pair:{cfg.name}:M19/m{m}/sweep1", key, one[key][m], o1[okey], TOL1)
    o = run_oracle(cfg, model, V[m], 4)
    assert rel_l2(paired["V_star"][m], o["V_star"]) <= TOL_VSTAR
    assert np.all(np.abs(paired["free_energy"][m] - o["free_energy"]) <= TOL_L * np.abs(o["free_energy"]))


@pytest.mark.parametrize("c,over", [(3, dict(T=40, M=21)), (0, dict(T=60, M=20)), (2, dict(T=30, M=13)),
                                    (3, dict(T=35, M=37, N=24))])
def test_multi_chain_forward_backward(c, over, monkeypatch):
    """> 32 chains: the multi-chain forward-backward (C chains of one source per warp, the N = 32 Q + R
    remainder states spread over the lanes; M not a multiple of C leaves a partly empty group) agrees
    with the one-chain-per-warp kernel and with the oracle."""
    cfg, model, V = make_inputs(c, **over)
    monkeypatch.setenv("NFHMM_FB_MULTI", "1")   # (the default for <= 64 chains is the one-chain kernel)
    multi = run_gpu(cfg, model, V, 4)
    if cfg.N % 8 == 0 and V.shape[0] >= 16:   # tensor-core variant (16 chains per warp, mma.sync 3xTF32)
        monkeypatch.setenv("NFHMM_FB_MULTI", "2")
        tcv = run_gpu(cfg, model, V, 4)
        for key in ("d_hat", "alpha_hat", "V_hat", "V_star"):
            assert rel_l2(tcv[key], multi[key]) <= 2e-6, key
    monkeypatch.setenv("NFHMM_FB_MULTI", "0")
    one = run_gpu(cfg, model, V, 4)
    for key in ("d_hat", "alpha_hat", "V_hat", "V_star"):
        assert rel_l2(multi[key], one[key]) <= 2e-6, key
    assert np.all(np.abs(multi["free_energy"] - one["free_energy"]) <= 1e-7 * np.abs(one["free_energy"]))
    for m in (0, V.shape[0] - 1):
        o1 = run_oracle(cfg, model, V[m], 1, separate=False)
        g1 = run_gpu(cfg, model, V, 1, separate=False) if m == 0 else g1
        compare(f"multi-fb:{cfg.name}:M{V.shape[0]}/m{m}/sweep1", "d_hat", g1["d_hat"][m], o1["d_hat"], TOL1)
        o = run_oracle(cfg, model, V[m], 4)
        assert rel_l2(multi["V_star"][m], o["V_star"]) <= TOL_VSTAR
        assert np.all(np.abs(multi["free_energy"][m] - o["free_energy"]) <= TOL_L * np.abs(o["free_energy"]))


@pytest.mark.parametrize("chunk", [None, "32"])
def test_long_single_chain_parallel_scan_fits(chunk, monkeypatch):
    """One long chain with N = 64 (the parallel-in-time FB's largest state bucket): T = 20,000 frames.
    With NFHMM_FB_CHUNK=32 the phase-2 scan would need 625 chunks' row scales in shared memory (> 227 KB);
    fb_pick_chunks grows the chunk length until it fits instead of failing the sweep."""
    if chunk:
        monkeypatch.setenv("NFHMM_FB_CHUNK", chunk)
    cfg, model, V = make_inputs(0, S=1, N=64, K=3, F=33, T=20000, M=1, counts=300)
    check_parity(cfg, model, V, 3)


@pytest.mark.parametrize("c,over", [(0, {}), (1, dict(T=300)), (3, dict(T=200, M=3)), (4, dict(T=40, M=2))])
def test_recon_tf32_variant_matches_3xfp16(c, over, monkeypatch):
    """The default reconstruction runs 3xFP16 products (theta~ scaled by 2^15, dictionary rows by powers of two;
    DESIGN "3xFP16 reconstruction"); NFHMM_RECON=tf32 selects the 3xTF32 products.  Both keep ~22 significant
    bits per product, so they agree with each other and with the oracle."""
    cfg, model, V = make_inputs(c, **over)
    h16 = run_gpu(cfg, model, V, 5)
    monkeypatch.setenv("NFHMM_BACKPROJ", "tf32")     # 3xFP16 reconstruction, 3xTF32 back-projection on R'
    mixed = run_gpu(cfg, model, V, 5)
    monkeypatch.setenv("NFHMM_RECON", "tf32")        # both 3xTF32 (plain R)
    tf = run_gpu(cfg, model, V, 5)
    for other in (mixed, tf):
        for key in ("d_hat", "alpha_hat", "V_hat", "V_star"):
            assert rel_l2(h16[key], other[key]) <= 3e-6, key
        # (the data term sum V log V_hat moves by ~1e-7 relative with V_hat's ~1e-6 rounding differences)
        assert np.all(np.abs(h16["free_energy"] - other["free_energy"]) <= 1e-6 * np.abs(other["free_energy"]))
    monkeypatch.delenv("NFHMM_RECON")
    monkeypatch.delenv("NFHMM_BACKPROJ")
    o1 = run_oracle(cfg, model, V[0], 1, separate=False)
    g1 = run_gpu(cfg, model, V[:1], 1, separate=False)
    compare(f"recon-h16:{cfg.name}/m0/sweep1", "V_hat", g1["V_hat"][0], o1["V_hat"], TOL1)
    compare(f"recon-h16:{cfg.name}/m0/sweep1", "d_hat", g1["d_hat"][0], o1["d_hat"], TOL1)
    o = run_oracle(cfg, model, V[0], 5)
    assert rel_l2(h16["V_star"][0], o["V_star"]) <= TOL_VSTAR
    assert np.all(np.abs(h16["free_energy"][0] - o["free_energy"]) <= TOL_L * np.abs(o["free_energy"]))


def test_recon_3xfp16_extreme_dynamic_range():
    """Range stress for the 3xFP16 contractions: very sparse dictionaries (Dirichlet(0.05): entries down
    to ~1e-30 beside ~1), frame masses from 1 to 10^7 counts (theta~ down to ~1e-8), silent frames and
    counts in a bin no dictionary covers.
    Products below the FP16 range of a row carry at most 2^-38 of that row's largest term (DESIGN), so
    sweep-1 parity holds at the north-star tolerance."""
    cfg, model, V = make_inputs(0, S=2, N=4, K=3, F=65, T=150, counts=1000)
    rng = np.random.default_rng(1206)
    beta = rng.dirichlet(np.full(cfg.F, 0.05), size=cfg.S * cfg.N * cfg.K).astype(np.float32)
    beta = np.maximum(beta, np.float32(1e-30))
    beta /= beta.sum(1, keepdims=True)
    model.beta[...] = beta.reshape(model.beta.shape)
    mass = 10.0 ** rng.uniform(0, 7, size=cfg.T)
    V0 = np.zeros((1, cfg.T, cfg.F), np.float32)
    W = rng.dirichlet(np.ones(cfg.S * cfg.N * cfg.K), size=cfg.T) @ beta
    for t in range(cfg.T):
        V0[0, t] = rng.multinomial(int(mass[t]), W[t] / W[t].sum())
    V0[0, 5:8] = 0.0
    # mispredicted bins: counts where every dictionary is ~0 (R = V / V_hat huge: the back-projection's
    # per-row A scale is set by these entries, the rest of the row sits far below its maximum)
    l_bad = int(np.argmin(beta.max(0)))
    V0[0, 20:30, l_bad] += np.float32(3.0)
    o1 = run_oracle(cfg, model, V0[0], 1, separate=False)
    g1 = run_gpu(cfg, model, V0, 1, separate=False)
    for key, ref in (("V_hat", o1["V_hat"]), ("d_hat", o1["d_hat"]), ("alpha_hat", o1["alpha"])):
        compare(f"recon-h16-range/m0/sweep1", key, g1[key][0], ref, TOL1)
    o = run_oracle(cfg, model, V0[0], 8)
    g = run_gpu(cfg, model, V0, 8)
    assert rel_l2(g["V_star"][0], o["V_star"]) <= TOL_VSTAR
    assert np.all(np.abs(g["free_energy"][0] - o["free_energy"]) <= TOL_L * np.abs(o["free_energy"]))
