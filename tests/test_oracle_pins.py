"""Pins for the CPU oracle (oracle/nfhmm_oracle.c) against things other than itself.

Each pin comes from the paper, SPEC's hand-checked examples (tests/golden/spec_hand_cases.json),
closed forms, textbook/library routines (scipy.special.digamma/gammaln, path enumeration), or
invariants the mathematics fixes.  The strongest pins are independent of the update equations:
  * the bound L computed from its DEFINITION (E_q[log P] + H[q], explicit z, enumerated q(D))
    equals the oracle's closed form;
  * each coordinate update is a stationary point of that directly-evaluated bound (a wrong sign,
    dropped term or transposed operand in Eq. 6/7/8 or the FB breaks stationarity);
  * L is a lower bound on the exact evidence log P(f) (enumerated Dirichlet-multinomial integrals);
  * L is non-decreasing across sweeps.
"""
import itertools
import json
import math
import os

import numpy as np
import pytest
from scipy.special import digamma as sp_digamma, gammaln

GOLDEN = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_hand_cases.json")))


# ----------------------------------------------------------------------------------------------
# tiny random instances
# ----------------------------------------------------------------------------------------------
def tiny_instance(rng, S, N, K, F, T, counts, conc=1.0):
    beta = rng.dirichlet(np.full(F, conc), size=(S, N, K)).astype(np.float32)
    beta = (beta / beta.sum(-1, keepdims=True)).astype(np.float32)
    trans = (rng.dirichlet(np.ones(N), size=(S, N)) + 2.0 * np.eye(N)).astype(np.float64)
    trans = (trans / trans.sum(-1, keepdims=True)).astype(np.float32)
    prior = rng.dirichlet(np.ones(N), size=S).astype(np.float32)
    V = np.stack([rng.multinomial(counts, rng.dirichlet(np.ones(F))) for _ in range(T)]).astype(np.float32)
    return beta, trans, prior, V


def kidx(S, N, K):
    """(s, n) of every global element k (S:250 ordering)."""
    k = np.arange(S * N * K)
    blk = k // K
    return blk // N, blk % N


# ----------------------------------------------------------------------------------------------
# digamma
# ----------------------------------------------------------------------------------------------
@pytest.mark.parametrize("case", GOLDEN["digamma"])
def test_digamma_golden(oracle, case):
    assert abs(oracle.digamma(case["x"]) - case["value"]) <= case["tol"]


def test_digamma_recurrence_harmonic_and_lgamma_derivative(oracle):
    euler = 0.5772156649015329
    for n in range(1, 40):                                   # psi(n) = -gamma_E + H_{n-1}
        H = sum(1.0 / i for i in range(1, n))
        assert abs(oracle.digamma(float(n)) - (-euler + H)) < 1e-13 * max(1, abs(H))
    rng = np.random.default_rng(0)
    for x in rng.uniform(0.05, 300.0, size=200):
        assert abs(oracle.digamma(x + 1) - oracle.digamma(x) - 1.0 / x) < 1e-12 * max(1.0, 1.0 / x)
        h = 1e-5 * max(1.0, x)
        fd = (math.lgamma(x + h) - math.lgamma(x - h)) / (2 * h)  # psi = d lnGamma / dx
        assert abs(oracle.digamma(x) - fd) < 1e-7 * max(1.0, abs(fd))
        assert abs(oracle.digamma(x) - sp_digamma(x)) < 1e-13 * max(1.0, abs(sp_digamma(x)))
    assert abs(oracle.digamma(100.0) - (math.log(100.0) - 1 / 200)) < 1e-4


# ----------------------------------------------------------------------------------------------
# Eq. 1 / P:111 and hand cases of Eqs. 6/7
# ----------------------------------------------------------------------------------------------
@pytest.mark.parametrize("case", GOLDEN["prior_alpha"])
def test_prior_alpha_golden(oracle, case):
    a = oracle.prior_alpha(case["S"], case["N"], case["K"], case["gamma"], case["states"])
    np.testing.assert_array_equal(a, np.array(case["alpha"], float))


@pytest.mark.parametrize("case", GOLDEN["update_alpha"])
def test_update_alpha_golden(oracle, case):
    dims = (case["F"], case["T"], case["S"], case["N"], case["K"])
    an, _, _ = oracle.z_alpha_step(np.array(case["beta"]), np.array(case["V"]), np.array(case["alpha_in"]),
                                   np.array(case["d_hat"]), dims, case["gamma"])
    np.testing.assert_allclose(an, np.array(case["alpha_out"]), rtol=0, atol=1e-12)


@pytest.mark.parametrize("case", GOLDEN["z_hat"])
def test_z_hat_golden(oracle, case):
    dims = (case["F"], case["T"], case["S"], case["N"], case["K"])
    z = oracle.z_hat(np.array(case["beta"]), np.array(case["alpha"]), dims)
    np.testing.assert_allclose(z[0, case["l"]], case["z"], atol=1e-7)   # float32 beta storage


def test_z_hat_normalised_uniform_and_single_element(oracle):
    rng = np.random.default_rng(1)
    S, N, K, F, T = 2, 2, 3, 5, 4
    beta, _, _, _ = tiny_instance(rng, S, N, K, F, T, 10)
    alpha = rng.uniform(1, 5, size=(T, S * N * K))
    z = oracle.z_hat(beta, alpha, (F, T, S, N, K))
    np.testing.assert_allclose(z.sum(-1), 1.0, atol=1e-12)
    ub = np.full((S, N, K, F), 1.0 / F, np.float32)
    zu = oracle.z_hat(ub, np.full((T, S * N * K), 2.5), (F, T, S, N, K))
    np.testing.assert_allclose(zu, 1.0 / (S * N * K), atol=1e-12)
    z1 = oracle.z_hat(np.full((1, 1, 1, F), 1.0 / F, np.float32), np.full((T, 1), 7.0), (F, T, 1, 1, 1))
    np.testing.assert_allclose(z1, 1.0, atol=0)


def test_update_alpha_linear_in_V(oracle):
    rng = np.random.default_rng(2)
    S, N, K, F, T = 2, 3, 2, 6, 3
    beta, _, _, V = tiny_instance(rng, S, N, K, F, T, 20)
    alpha = rng.uniform(1, 4, size=(T, S * N * K))
    d = rng.dirichlet(np.ones(N), size=(S, T))
    a1, _, _ = oracle.z_alpha_step(beta, V, alpha, d, (F, T, S, N, K), 1.0)
    a10, _, _ = oracle.z_alpha_step(beta, V * 10, alpha, d, (F, T, S, N, K), 1.0)
    prior = 1.0 + d[kidx(S, N, K)[0], :, kidx(S, N, K)[1]].T
    np.testing.assert_allclose(a10 - prior, 10 * (a1 - prior), rtol=1e-12)


# ----------------------------------------------------------------------------------------------
# forward-backward vs brute-force path enumeration
# ----------------------------------------------------------------------------------------------
def brute_chain(loglik, A, pi):
    T, N = loglik.shape
    marg = np.zeros((T, N))
    tot = 0.0
    for path in itertools.product(range(N), repeat=T):
        p = pi[path[0]] * math.exp(loglik[0, path[0]])
        for t in range(1, T):
            p *= A[path[t - 1], path[t]] * math.exp(loglik[t, path[t]])
        tot += p
        for t in range(T):
            marg[t, path[t]] += p
    return marg / tot, math.log(tot)


def test_fb_fixed_table(oracle):
    g = GOLDEN["fb_fixed_table"]
    ll, A, pi = np.array(g["loglik"]), np.array(g["A_rowstochastic"]), np.array(g["pi"])
    m, lz = oracle.forward_backward(ll, A, pi)
    bm, blz = brute_chain(ll, A, pi)
    np.testing.assert_allclose(m, bm, atol=1e-12)
    assert abs(lz - blz) < 1e-12


@pytest.mark.parametrize("T,N", [(1, 1), (1, 3), (2, 2), (3, 3), (5, 2), (5, 3), (6, 3)])
def test_fb_brute_force(oracle, T, N):
    rng = np.random.default_rng(10 * T + N)
    for _ in range(5):
        A = rng.dirichlet(np.ones(N), size=N)
        pi = rng.dirichlet(np.ones(N))
        ll = rng.normal(0, 3, size=(T, N)) - 50.0
        m, lz = oracle.forward_backward(ll, A, pi)
        bm, blz = brute_chain(ll, A, pi)
        np.testing.assert_allclose(m, bm, atol=1e-12)
        assert abs(lz - blz) < 1e-12 * max(1, abs(blz))


def test_fb_special_cases(oracle):
    rng = np.random.default_rng(3)
    ll = rng.normal(size=(7, 1))
    m, lz = oracle.forward_backward(ll, np.ones((1, 1)), np.ones(1))          # S:128 N = 1
    np.testing.assert_allclose(m, 1.0)
    assert abs(lz - ll.sum()) < 1e-12
    m, _ = oracle.forward_backward(np.tile([[-1.3, -1.3]], (6, 1)), np.full((2, 2), 0.5), np.full(2, 0.5))
    np.testing.assert_allclose(m, 0.5, atol=1e-15)                          # S:129 symmetry
    ll = rng.normal(size=(8, 3))
    c = rng.normal(size=(8, 1)) * 100
    A = rng.dirichlet(np.ones(3), size=3)
    pi = rng.dirichlet(np.ones(3))
    m1, z1 = oracle.forward_backward(ll, A, pi)
    m2, z2 = oracle.forward_backward(ll + c, A, pi)                          # S:134 shift invariance
    np.testing.assert_allclose(m1, m2, atol=1e-12)
    assert abs(z2 - z1 - c.sum()) < 1e-9
    P = np.roll(np.eye(3), 1, axis=1)                                       # S:135 permutation chain
    m, _ = oracle.forward_backward(ll, P, np.array([0.0, 1.0, 0.0]))
    traj = [(1 + t) % 3 for t in range(8)]
    np.testing.assert_allclose(m, np.eye(3)[traj], atol=1e-12)
    with pytest.raises(oracle.OracleError):                                 # S:126 zero evidence
        oracle.forward_backward(np.array([[0.0, -np.inf]]), np.eye(2), np.array([0.0, 1.0]))


def test_fb_long_chain_stable(oracle):
    rng = np.random.default_rng(4)
    T, N = 3000, 5
    ll = rng.normal(0, 30, size=(T, N)) - 1000.0
    A = rng.dirichlet(np.ones(N), size=N)
    m, lz = oracle.forward_backward(ll, A, np.full(N, 1 / N))
    assert np.isfinite(m).all() and np.isfinite(lz)
    np.testing.assert_allclose(m.sum(1), 1.0, atol=1e-12)


# ----------------------------------------------------------------------------------------------
# the bound from its definition (independent of Eqs. 6-8 and of the oracle's closed form)
# ----------------------------------------------------------------------------------------------
def direct_bound(beta, trans, prior, V, dims, gamma, alpha, z, qD):
    """L = E_q[log P(Z, theta, D, f)] + H[q], evaluated term by term from the generative model
    (Eq. 1) with q(theta_t) = Dir(alpha_t), q(Z) = z [T][F][Kt] (per quantum,
    grouped by frequency P:171), q(D^s) = full distribution over paths qD[s] {path: prob}."""
    F, T, S, N, K = dims
    Kt = S * N * K
    b = beta.reshape(Kt, F).astype(np.float64)
    Elog = sp_digamma(alpha) - sp_digamma(alpha.sum(1, keepdims=True))        # E[log theta]
    L = 0.0
    # chain prior and entropy, per source
    marg = np.zeros((S, T, N))
    for s in range(S):
        for path, q in qD[s].items():
            if q <= 0:
                continue
            lp = math.log(prior[s, path[0]]) + sum(math.log(trans[s, path[t - 1], path[t]]) for t in range(1, T))
            L += q * (lp - math.log(q))
            for t in range(T):
                marg[s, t, path[t]] += q
    # E[log Dir(theta_t; alpha(D_t))] with alpha(D) = prior Dirichlet of Eq. 1 (sum over joint states)
    for t in range(T):
        for states in itertools.product(range(N), repeat=S):
            w = np.prod([marg[s, t, states[s]] for s in range(S)])
            if w == 0:
                continue
            a = np.ones(Kt)
            for s in range(S):
                blk = s * N + states[s]
                a[blk * K:(blk + 1) * K] += gamma
            L += w * (gammaln(a.sum()) - gammaln(a).sum() + ((a - 1) * Elog[t]).sum())
    # quanta: E[log theta_z + log beta_f(z)] - E[log q(z)]
    for t in range(T):
        for l in range(F):
            if V[t, l] == 0:
                continue
            zz = z[t, l]
            nz = zz > 0
            L += V[t, l] * (zz[nz] * (Elog[t][nz] + np.log(b[nz, l]) - np.log(zz[nz]))).sum()
    # Dirichlet entropy of q(theta_t)
    for t in range(T):
        a = alpha[t]
        a0 = a.sum()
        H = gammaln(a).sum() - gammaln(a0) + (a0 - Kt) * sp_digamma(a0) - ((a - 1) * sp_digamma(a)).sum()
        L += H
    return L


def enum_qD(phi_s, trans_s, prior_s, gamma):
    """q(D) proportional to P(D) exp(gamma sum_t phi_{t,D_t}) by explicit enumeration."""
    T, N = phi_s.shape
    w = {}
    for path in itertools.product(range(N), repeat=T):
        lp = math.log(prior_s[path[0]]) + sum(math.log(trans_s[path[t - 1], path[t]]) for t in range(1, T))
        lp += gamma * sum(phi_s[t, path[t]] for t in range(T))
        w[path] = lp
    m = max(w.values())
    tot = sum(math.exp(v - m) for v in w.values())
    return {p: math.exp(v - m) / tot for p, v in w.items()}


def direct_phi(alpha, dims):
    F, T, S, N, K = dims
    Elog = sp_digamma(alpha) - sp_digamma(alpha.sum(1, keepdims=True))
    return Elog.reshape(T, S, N, K).sum(-1).transpose(1, 0, 2)               # [S][T][N]


def direct_z(beta, alpha, dims):
    F, T, S, N, K = dims
    b = beta.reshape(S * N * K, F).astype(np.float64)
    Elog = sp_digamma(alpha) - sp_digamma(alpha.sum(1, keepdims=True))
    u = b.T[None] * np.exp(Elog)[:, None, :]                                 # [T][F][Kt]
    return u / u.sum(-1, keepdims=True)


TINY = [(2, 2, 1, 3, 3, 5, 1.0), (2, 2, 2, 4, 3, 8, 1.0), (1, 3, 2, 4, 4, 6, 1.0),
        (3, 2, 1, 3, 2, 4, 2.0), (2, 3, 1, 3, 3, 5, 0.5)]


@pytest.mark.parametrize("S,N,K,F,T,counts,gamma", TINY)
def test_bound_closed_form_equals_definition(oracle, S, N, K, F, T, counts, gamma):
    rng = np.random.default_rng(S * 100 + N * 10 + K + F)
    beta, trans, prior, V = tiny_instance(rng, S, N, K, F, T, counts)
    dims = (F, T, S, N, K)
    for iters in (1, 2, 4):
        r = oracle.vb_run(beta, trans, prior, V, dims, iters, gamma)
        alpha = r["alpha"]
        phi = direct_phi(alpha, dims)
        qD = [enum_qD(phi[s], trans[s].astype(float), prior[s].astype(float), gamma) for s in range(S)]
        z = direct_z(beta, alpha, dims)
        Ld = direct_bound(beta, trans.astype(float), prior.astype(float), V, dims, gamma, alpha, z, qD)
        assert abs(r["free_energy"][-1] - Ld) <= 1e-10 * abs(Ld), (iters, r["free_energy"][-1], Ld)
        # the oracle's d_hat are the marginals of the enumerated q(D)
        for s in range(S):
            m = np.zeros((T, N))
            for p, q in qD[s].items():
                for t in range(T):
                    m[t, p[t]] += q
            np.testing.assert_allclose(r["d_hat"][s], m, atol=1e-11)
        # V_hat from the trailing z-step: kappa_tl = sum_k beta_l(k) exp(Elog_k)
        Elog = sp_digamma(alpha) - sp_digamma(alpha.sum(1, keepdims=True))
        np.testing.assert_allclose(r["V_hat"], np.exp(Elog) @ beta.reshape(-1, F).astype(float), rtol=1e-12)


@pytest.mark.parametrize("S,N,K,F,T,counts,gamma", TINY[:3])
def test_updates_are_stationary_points_of_the_bound(oracle, S, N, K, F, T, counts, gamma):
    """Each coordinate update maximises the directly-evaluated bound in its own factor:
    numerical gradients of L w.r.t. that factor's free parameters vanish at the update."""
    rng = np.random.default_rng(7 + S + N + K)
    beta, trans, prior, V = tiny_instance(rng, S, N, K, F, T, counts)
    trans, prior = trans.astype(float), prior.astype(float)
    dims = (F, T, S, N, K)
    r0 = oracle.vb_run(beta, trans, prior, V, dims, 2, gamma)
    a_prev, d_prev = r0["alpha"], r0["d_hat"]
    z_prev = direct_z(beta, a_prev, dims)
    phi_prev = direct_phi(a_prev, dims)
    qD_prev = [enum_qD(phi_prev[s], trans[s], prior[s], gamma) for s in range(S)]
    # alpha-step (Eq. 6): alpha_new maximises L(z_prev, alpha, qD_prev)
    a_new, _, _ = oracle.z_alpha_step(beta, V, a_prev, d_prev, dims, gamma)
    f = lambda a: direct_bound(beta, trans, prior, V, dims, gamma, a, z_prev, qD_prev)
    base = f(a_new)
    for _ in range(6):
        t, k = rng.integers(T), rng.integers(S * N * K)
        h = 1e-5 * a_new[t, k]
        ap, am = a_new.copy(), a_new.copy()
        ap[t, k] += h
        am[t, k] -= h
        g = (f(ap) - f(am)) / (2 * h)
        assert abs(g) < 1e-5 * max(1.0, abs(base) / a_new.size), g
        assert f(ap) <= base + 1e-9 and f(am) <= base + 1e-9
    # z-step (Eq. 7): z(alpha_new) maximises L(z, alpha_new, qD) over each simplex
    z_new = direct_z(beta, a_new, dims)
    fz = lambda z: direct_bound(beta, trans, prior, V, dims, gamma, a_new, z, qD_prev)
    basez = fz(z_new)
    for _ in range(6):
        t, l = rng.integers(T), rng.integers(F)
        if V[t, l] == 0:
            continue
        dlt = rng.normal(size=S * N * K)
        dlt -= dlt.mean()
        zp, zm = z_new.copy(), z_new.copy()
        eps = 1e-6 * z_new[t, l].min() / np.abs(dlt).max()
        zp[t, l] += eps * dlt
        zm[t, l] -= eps * dlt
        assert abs(fz(zp) - fz(zm)) / (2 * eps) < 1e-5 * V[t, l]
        assert fz(zp) <= basez + 1e-9 and fz(zm) <= basez + 1e-9
    # D-step: q(D) = enumerated FB posterior maximises L over path distributions (Eq. 4/5)
    phi_new = direct_phi(a_new, dims)
    qD = [enum_qD(phi_new[s], trans[s], prior[s], gamma) for s in range(S)]
    fq = lambda q: direct_bound(beta, trans, prior, V, dims, gamma, a_new, z_prev, q)
    baseq = fq(qD)
    for _ in range(4):
        s = rng.integers(S)
        paths = [p for p, q in qD[s].items() if q > 1e-3]    # a tangent direction on the simplex
        dlt = rng.normal(size=len(paths))
        dlt -= dlt.mean()
        eps = 1e-4 * min(qD[s][p] for p in paths) / np.abs(dlt).max()
        qp = [dict(q) for q in qD]
        qm = [dict(q) for q in qD]
        for p, dd in zip(paths, dlt):
            qp[s][p] += eps * dd
            qm[s][p] -= eps * dd
        assert abs(fq(qp) - fq(qm)) / (2 * eps) < 1e-6
        assert fq(qp) <= baseq + 1e-9 and fq(qm) <= baseq + 1e-9
    # and the oracle's D-step marginals come from exactly that q(D)
    oph = oracle.surrogate(a_new, dims)
    np.testing.assert_allclose(oph, phi_new, atol=1e-12)                    # Eq. 8 vs scipy digamma
    d_new, _ = oracle.d_step(oph, trans.astype(np.float32), prior.astype(np.float32), dims, gamma)
    for s in range(S):
        m = np.zeros((T, N))
        for p, q in qD[s].items():
            for t in range(T):
                m[t, p[t]] += q
        np.testing.assert_allclose(d_new[s], m, atol=1e-11)


def exact_log_evidence(beta, trans, prior, V, dims, gamma):
    """log P(f) of the ordered quanta (DESIGN R8): enumerate joint state paths; per frame
    P(f_t | D_t) = sum over element assignments of prod beta * B(alpha(D)+c)/B(alpha(D))."""
    F, T, S, N, K = dims
    Kt = S * N * K
    b = beta.reshape(Kt, F).astype(np.float64)
    frame_lik = {}
    for t in range(T):
        quanta = [l for l in range(F) for _ in range(int(V[t, l]))]
        for states in itertools.product(range(N), repeat=S):
            a = np.ones(Kt)
            for s in range(S):
                blk = s * N + states[s]
                a[blk * K:(blk + 1) * K] += gamma
            lB = lambda x: gammaln(x).sum() - gammaln(x.sum())
            tot = 0.0
            for zs in itertools.product(range(Kt), repeat=len(quanta)):
                c = np.bincount(np.array(zs, dtype=int), minlength=Kt) if zs else np.zeros(Kt)
                pb = np.prod([b[z, l] for z, l in zip(zs, quanta)]) if zs else 1.0
                tot += pb * math.exp(lB(a + c) - lB(a))
            frame_lik[(t, states)] = tot
    total = 0.0
    for joint in itertools.product(itertools.product(range(N), repeat=S), repeat=T):
        p = 1.0
        for s in range(S):
            p *= prior[s, joint[0][s]]
            for t in range(1, T):
                p *= trans[s, joint[t - 1][s], joint[t][s]]
        for t in range(T):
            p *= frame_lik[(t, joint[t])]
        total += p
    return math.log(total)


@pytest.mark.parametrize("seed", range(4))
def test_bound_below_exact_evidence(oracle, seed):
    rng = np.random.default_rng(100 + seed)
    S, N, K, F, T = 2, 2, 1, 3, 3
    beta, trans, prior, V = tiny_instance(rng, S, N, K, F, T, 3)
    dims = (F, T, S, N, K)
    logp = exact_log_evidence(beta, trans.astype(float), prior.astype(float), V, dims, 1.0)
    r = oracle.vb_run(beta, trans, prior, V, dims, 30, 1.0)
    assert (r["free_energy"] <= logp + 1e-9).all(), (r["free_energy"].max(), logp)
    assert r["free_energy"][-1] > logp - 10.0   # and not vacuous


@pytest.mark.parametrize("S,N,K,F,T,counts,gamma", TINY + [(2, 4, 3, 12, 30, 2000, 1.0)])
def test_bound_monotone(oracle, S, N, K, F, T, counts, gamma):
    rng = np.random.default_rng(11 + S * N * K * F)
    beta, trans, prior, V = tiny_instance(rng, S, N, K, F, T, counts)
    r = oracle.vb_run(beta, trans, prior, V, (F, T, S, N, K), 25, gamma)
    fe = r["free_energy"]
    assert (np.diff(fe) >= -1e-12 * np.abs(fe[1:])).all(), np.diff(fe).min()


# ----------------------------------------------------------------------------------------------
# invariants and special cases
# ----------------------------------------------------------------------------------------------
def test_mass_and_normalisation_invariants(oracle):
    rng = np.random.default_rng(5)
    S, N, K, F, T, C = 2, 4, 3, 20, 15, 500
    beta, trans, prior, V = tiny_instance(rng, S, N, K, F, T, C)
    dims = (F, T, S, N, K)
    r = oracle.vb_run(beta, trans, prior, V, dims, 5, 1.0)
    Kt = S * N * K
    np.testing.assert_allclose(r["alpha"].sum(1), V.sum(1) + Kt + 1.0 * S * K, rtol=1e-12)   # mass
    assert (r["alpha"] >= 1.0).all()
    np.testing.assert_allclose(r["d_hat"].sum(-1), 1.0, atol=1e-12)
    vs, vst = oracle.separate(beta, V, r["alpha"], dims)
    np.testing.assert_allclose(vst.sum(0), V, rtol=1e-12, atol=1e-12)     # S:401 conservation
    # reconstructed mass = v_t (up to the float32 rounding of the column sums of beta)
    colsum = beta.reshape(Kt, F).astype(float).sum(1)
    Et = r["alpha"] / r["alpha"].sum(1, keepdims=True)
    np.testing.assert_allclose(vs.sum((0, 2)), V.sum(1) * (Et @ colsum), rtol=1e-12)
    np.testing.assert_allclose(vs.sum((0, 2)), V.sum(1), rtol=1e-6)


def test_gamma_zero_decouples_chain(oracle):
    """gamma = 0 (needs DESIGN R1): q(D^s) is the chain prior, d_t = pi A^{t-1}."""
    rng = np.random.default_rng(6)
    S, N, K, F, T = 2, 3, 2, 6, 7
    beta, trans, prior, V = tiny_instance(rng, S, N, K, F, T, 50)
    r = oracle.vb_run(beta, trans, prior, V, (F, T, S, N, K), 3, 0.0)
    for s in range(S):
        p = prior[s].astype(float)
        for t in range(T):
            np.testing.assert_allclose(r["d_hat"][s, t], p, atol=1e-12)
            p = p @ trans[s].astype(float)


def test_N1_is_textbook_lda_estep(oracle):
    """N = 1: d = 1 and each frame is the LDA variational E-step with fixed topics and symmetric
    Dirichlet prior 1 + gamma (Blei et al. 2003 eqs. 6-7)."""
    rng = np.random.default_rng(8)
    S, N, K, F, T = 2, 1, 3, 7, 4
    beta, trans, prior, V = tiny_instance(rng, S, N, K, F, T, 40)
    gamma, iters = 1.0, 6
    r = oracle.vb_run(beta, trans, prior, V, (F, T, S, N, K), iters, gamma)
    np.testing.assert_allclose(r["d_hat"], 1.0)
    topics = beta.reshape(S * K, F).astype(float)          # beta[k][w]
    for t in range(T):
        g = np.full(S * K, 1.0 + gamma / N)                  # initial variational Dirichlet
        for _ in range(iters):                               # Blei et al.: phi_nk ∝ beta_k,w exp(psi(g_k))
            ph = topics * np.exp(sp_digamma(g))[:, None]
            ph /= ph.sum(0, keepdims=True)
            g = (1.0 + gamma) + (ph * V[t][None]).sum(1)   # g_k = alpha_k + sum_n phi_nk
        np.testing.assert_allclose(r["alpha"][t], g, rtol=1e-12)


def test_identical_sources_split_evenly(oracle):
    rng = np.random.default_rng(9)
    S, N, K, F, T = 2, 3, 2, 8, 6
    beta, trans, prior, V = tiny_instance(rng, S, N, K, F, T, 100)
    beta[1], trans[1], prior[1] = beta[0], trans[0], prior[0]
    r = oracle.vb_run(beta, trans, prior, V, (F, T, S, N, K), 8, 1.0)
    _, vst = oracle.separate(beta, V, r["alpha"], (F, T, S, N, K))
    np.testing.assert_allclose(vst[0], V / 2, rtol=1e-12)
    np.testing.assert_allclose(vst[1], V / 2, rtol=1e-12)


def test_disjoint_supports_attribute_mass(oracle):
    """S:308 / S:578: sources on disjoint frequency halves; frames where only source 0 sounds put
    >= 95% of E[theta] on source 0's elements."""
    rng = np.random.default_rng(12)
    S, N, K, F, T = 2, 3, 2, 16, 10
    beta = np.zeros((S, N, K, F))
    beta[0, :, :, :F // 2] = rng.dirichlet(np.ones(F // 2), size=(N, K))
    beta[1, :, :, F // 2:] = rng.dirichlet(np.ones(F // 2), size=(N, K))
    beta = np.maximum(beta, 1e-12)
    beta = (beta / beta.sum(-1, keepdims=True)).astype(np.float32)
    trans = np.full((S, N, N), 1.0 / N, np.float32)
    prior = np.full((S, N), 1.0 / N, np.float32)
    V = np.zeros((T, F), np.float32)
    for t in range(T):
        p = beta[0, rng.integers(N)].astype(float).T @ rng.dirichlet(np.ones(K))
        if t % 2:
            p = p + beta[1, rng.integers(N)].astype(float).T @ rng.dirichlet(np.ones(K))
        V[t] = rng.multinomial(10_000, p / p.sum())
    r = oracle.vb_run(beta, trans, prior, V, (F, T, S, N, K), 20, 1.0)
    Et = r["alpha"] / r["alpha"].sum(1, keepdims=True)
    share0 = Et[:, : N * K].sum(1)
    assert (share0[0::2] >= 0.95).all(), share0
    # Section 4 attributes each bin to the source whose reconstruction explains it: with
    # disjoint supports source s's V_src is (up to the 1e-12 floor) zero off its half, so V*^(0) = V on
    # the lower half and V*^(1) = V on the upper half of EVERY frame, and on source-0-only frames
    # V*^(0) carries >= 95% of the frame's mass (an s <-> S-1-s swap of the outputs fails both).
    vsrc, vst = oracle.separate(beta, V, r["alpha"], (F, T, S, N, K))
    h = F // 2
    np.testing.assert_allclose(vst[0][:, :h], V[:, :h], rtol=1e-6, atol=1e-6)
    np.testing.assert_allclose(vst[1][:, h:], V[:, h:], rtol=1e-6, atol=1e-6)
    assert np.abs(vst[0][:, h:]).max() <= 1e-6 * V.max()
    assert np.abs(vst[1][:, :h]).max() <= 1e-6 * V.max()
    assert vsrc[0][:, h:].max() <= 1e-8 * vsrc[0].max() and vsrc[1][:, :h].max() <= 1e-8 * vsrc[1].max()
    vt = V.sum(1)
    assert (vst[0].sum(1)[0::2] >= 0.95 * vt[0::2]).all()
    assert (vst[1].sum(1)[0::2] <= 0.05 * vt[0::2]).all()


def test_S1_d_is_fb_of_surrogate(oracle):
    """S = 1 (BJ:5 "reduces to the single-source N-HMM", structural reading S:307): d equals an
    independent enumeration of the single chain posterior on gamma*phi(alpha); V* = V exactly."""
    rng = np.random.default_rng(13)
    S, N, K, F, T = 1, 3, 2, 5, 5
    beta, trans, prior, V = tiny_instance(rng, S, N, K, F, T, 30)
    dims = (F, T, S, N, K)
    r = oracle.vb_run(beta, trans, prior, V, dims, 4, 1.0)
    phi = direct_phi(r["alpha"], dims)
    bm, _ = brute_chain(phi[0], trans[0].astype(float), prior[0].astype(float))
    np.testing.assert_allclose(r["d_hat"][0], bm, atol=1e-12)
    _, vst = oracle.separate(beta, V, r["alpha"], dims)
    np.testing.assert_allclose(vst[0], V, rtol=1e-15)


def test_zero_support_is_an_error(oracle):
    S, N, K, F, T = 1, 1, 1, 3, 1
    beta = np.array([[[[0.5, 0.5, 0.0]]]], np.float32)
    V = np.array([[1.0, 0.0, 2.0]], np.float32)
    with pytest.raises(oracle.OracleError):
        oracle.vb_run(beta, np.ones((1, 1, 1), np.float32), np.ones((1, 1), np.float32), V, (F, T, S, N, K), 1)
