"""Pins of the N-HMM EM oracle (oracle/nhmm_em_oracle.c) against things other than
itself: exhaustive path enumeration, brute-force evidence, SPEC's closed-form and fixed-point examples
(S:182-183), and EM's ascent property.  CPU only."""
import itertools

import numpy as np
import pytest

from oracle import oracle


def brute_fb(loglik, A, pi):
    """Enumerate all N^T state paths: marginals, pairwise sums and the log evidence."""
    T, N = loglik.shape
    marg = np.zeros((T, N))
    xi = np.zeros((N, N))
    Z = 0.0
    for path in itertools.product(range(N), repeat=T):
        w = pi[path[0]] * np.exp(loglik[0, path[0]])
        for t in range(1, T):
            w *= A[path[t - 1], path[t]] * np.exp(loglik[t, path[t]])
        Z += w
        for t in range(T):
            marg[t, path[t]] += w
        for t in range(1, T):
            xi[path[t - 1], path[t]] += w
    return marg / Z, xi / Z, np.log(Z)


def brute_evidence(V, beta, theta, A, pi):
    """log P(V) of the N-HMM with per-frame weights theta: sum over state paths of
    pi A ... prod_t prod_l (sum_z theta_t(d)_z beta_l(d, z))^V_lt (multinomial coefficient omitted)."""
    T, F = V.shape
    N = beta.shape[0]
    em = np.zeros((T, N))
    for t in range(T):
        for d in range(N):
            lh = theta[t, d] @ beta[d]                   # [F]
            em[t, d] = np.sum(np.where(V[t] > 0, V[t] * np.log(np.where(V[t] > 0, lh, 1.0)), 0.0))
    return brute_fb(em, A, pi)[2]


def random_instance(rng, T, F, N, K, counts=6):
    V = rng.integers(0, counts, size=(T, F)).astype(float)
    V[:, 0] += 1.0                                       # every frame non-empty
    beta = rng.dirichlet(np.ones(F), size=(N, K))
    theta = rng.dirichlet(np.ones(K), size=(T, N))
    A = rng.dirichlet(np.ones(N), size=N) + 2.0 * np.eye(N)
    A /= A.sum(1, keepdims=True)
    pi = rng.dirichlet(np.ones(N))
    return V, beta, theta, A, pi


@pytest.mark.parametrize("T,N", [(1, 2), (3, 2), (4, 3), (5, 3)])
def test_pairwise_posteriors_match_path_enumeration(T, N):
    rng = np.random.default_rng(100 + 10 * T + N)
    ll = rng.normal(size=(T, N)) * 3.0
    A = rng.dirichlet(np.ones(N), size=N)
    pi = rng.dirichlet(np.ones(N))
    m, xi, lz = oracle.fb_pairwise(ll, A, pi)
    bm, bxi, blz = brute_fb(ll, A, pi)
    np.testing.assert_allclose(m, bm, rtol=0, atol=1e-12)
    np.testing.assert_allclose(xi, bxi, rtol=0, atol=1e-12)
    assert abs(lz - blz) <= 1e-12 * max(1.0, abs(blz))
    # marginalising the pairwise sums over either index gives the adjacent marginals
    np.testing.assert_allclose(xi.sum(1), m[:-1].sum(0), atol=1e-12)
    np.testing.assert_allclose(xi.sum(0), m[1:].sum(0), atol=1e-12)


def test_estep_evidence_matches_brute_force_and_em_ascends():
    """The log evidence each EM iteration reports is the brute-force evidence of the parameters it
    started from, and that evidence never decreases."""
    rng = np.random.default_rng(7)
    V, beta, theta, A, pi = random_instance(rng, T=5, F=6, N=3, K=2)
    cur = (beta.copy(), theta.copy(), A.copy(), pi.copy())
    prev = -np.inf
    for it in range(6):
        bf = brute_evidence(V, *cur)
        r = oracle.nhmm_em(V, *cur, 1)
        assert abs(r["loglik"][0] - bf) <= 1e-10 * abs(bf), it
        assert bf >= prev - 1e-10 * abs(bf), it
        prev = bf
        cur = (r["beta"], r["theta"], r["A"], r["pi"])
        # normalisation invariants of the M-step
        np.testing.assert_allclose(r["beta"].sum(-1), 1.0, atol=1e-12)
        np.testing.assert_allclose(r["theta"].sum(-1), 1.0, atol=1e-12)
        np.testing.assert_allclose(r["A"].sum(-1), 1.0, atol=1e-12)
        assert abs(r["pi"].sum() - 1.0) <= 1e-12


def test_em_monotone_on_larger_random_instance():
    rng = np.random.default_rng(11)
    V, beta, theta, A, pi = random_instance(rng, T=40, F=20, N=4, K=3, counts=30)
    r = oracle.nhmm_em(V, beta, theta, A, pi, 15)
    assert np.all(np.diff(r["loglik"]) >= -1e-9 * np.abs(r["loglik"][1:]))


def test_single_element_closed_form():
    """N = 1, K = 1 -- beta is the normalised row-sum profile of V after one step."""
    rng = np.random.default_rng(3)
    T, F = 9, 11
    V = rng.integers(0, 20, size=(T, F)).astype(float)
    beta = rng.dirichlet(np.ones(F), size=(1, 1))
    r = oracle.nhmm_em(V, beta, np.ones((T, 1, 1)), np.ones((1, 1)), np.ones(1), 2)
    prof = V.sum(0) / V.sum()
    np.testing.assert_allclose(r["beta"][0, 0], prof, rtol=0, atol=1e-14)
    # the second iteration starts from the ML solution: its evidence is sum V log(profile)
    assert abs(r["loglik"][1] - np.sum(V[V > 0] * np.log(np.broadcast_to(prof, V.shape)[V > 0]))) <= 1e-10 * abs(r["loglik"][1])


def test_fixed_point_single_element_data():
    """data proportional to one dictionary element, model already at that element -> unchanged."""
    rng = np.random.default_rng(5)
    T, F, N, K = 6, 8, 2, 2
    beta = rng.dirichlet(np.ones(F), size=(N, K))
    V = np.outer(rng.integers(1, 9, size=T), beta[0, 1] * 64.0)   # every frame ∝ beta(0, 1)
    theta = np.zeros((T, N, K))
    theta[:, :, 1] = 1.0                                         # weights on element 1 of every dictionary
    A = np.array([[1.0, 0.0], [0.0, 1.0]])
    pi = np.array([1.0, 0.0])                                    # the chain sits in dictionary 0
    r = oracle.nhmm_em(V, beta, theta, A, pi, 2)
    np.testing.assert_allclose(r["beta"][0, 1], beta[0, 1], rtol=0, atol=1e-12)
    np.testing.assert_allclose(r["theta"][:, 0], theta[:, 0], atol=1e-12)
    np.testing.assert_allclose(r["pi"], pi, atol=1e-12)
    assert abs(r["loglik"][1] - r["loglik"][0]) <= 1e-12 * abs(r["loglik"][0])
