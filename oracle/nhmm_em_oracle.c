/*
 * nhmm_em_oracle.c -- plain, slow, single-threaded FP64 CPU oracle for maximum-likelihood EM training
 * of the single-source N-HMM (Mysore & Sahani, arXiv 1206.6468, Section 2.1).
 *
 * ORACLE -- TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  The product path
 * (paper_1206_6468_b200/, libnfhmm.so) never links, imports or calls it, and it shares no code,
 * header, table or constant with the CUDA path.
 *
 * Citation keys as in nfhmm_oracle.c ("P:n" = PAPER.md line n, "S:n" = SPEC.md line n).
 *
 * The model: state D_t | D_{t-1} ~ rho(D_{t-1}); per quantum an element Z_t ~ theta_t(D_t),
 * a frequency F_t ~ beta(D_t, Z_t).  "maximum-likelihood (ML) values of all these parameters may be
 * found by the EM algorithm"; the paper gives no equations, so the steps follow SPEC's em_step
 * and the standard derivation, in this order:
 *   E-step  lhat_{t,d}(l) = sum_z theta_t(d)_z beta_l(d,z);
 *           loglik_{t,d}  = sum_l V_lt log lhat_{t,d}(l)     (multinomial, no coefficient: constant in d);
 *           forward-backward over the chain -> gamma_t(d), xi_t(i,j), log evidence;
 *           P(z | l, t, d) = theta_t(d)_z beta_l(d,z) / lhat_{t,d}(l);
 *   M-step  theta_t(d)_z  ∝ sum_l V_lt P(z | l, t, d);
 *           beta_l(d,z)   ∝ sum_t gamma_t(d) V_lt P(z | l, t, d);
 *           rho(i -> j)   ∝ sum_{t>=1} xi_t(i,j);  pi = gamma_0;
 *           beta and rho floored at 1e-12, then renormalised (SPEC's decision S:214: "Floor of 1e-12
 *           applied to beta and rho after each M-step, then renormalize ... prevents absorbing zeros that
 *           would freeze EM"), and pi likewise (DESIGN R21: pi = gamma_0 puts all its mass on one state
 *           after a few iterations; if that state's emission ratio at frame 0 underflows, the evidence is
 *           exactly 0 and EM stops -- the absorbing zero S:214 guards against, on the chain's other
 *           parameter).  A sum with no weight at all (an element no frame, or a chain
 *           row no transition, gave any posterior mass to -- exactly 0 in FP64) keeps its previous value:
 *           0/0 has no ML solution.
 * (theta's update carries no gamma: gamma_t(d) is constant in z for fixed (t, d) and cancels in the
 * normalisation.)  Every step is the exact maximiser of the expected complete-data log-likelihood,
 * so the returned log evidence is non-decreasing across iterations.
 *
 * Layouts (row-major, FP64): V [T][F]; beta [N][K][F] (beta_l(d,z) = beta[(d*K + z)*F + l]);
 * theta [T][N][K]; A [N][N] row-stochastic (A[i][j] = P(D_t = j | D_{t-1} = i), DESIGN R4); pi [N].
 *
 * Parity pins: tests/test_nhmm_oracle.py (pairwise posteriors vs path enumeration; the E-step's log
 * evidence vs brute-force enumeration; EM ascent of the brute-force evidence; the N = K = 1 closed
 * form; the fixed point of S:180).
 */
#include <math.h>
#include <stdlib.h>
#include <string.h>

#define OR_OK 0
#define OR_EINVAL (-1)
#define OR_EZEROSUPPORT (-5)
#define OR_ENUMERIC (-6)

/* Scaled forward-backward with pairwise posteriors (Rabiner 1989, scaled form):
 *   e_t(n) = exp(loglik_t(n) - max_n loglik_t(n)),  a_0 = pi .* e_0 / c_0,  a_t = (a_{t-1} A) .* e_t / c_t,
 *   b_{T-1} = 1,  b_t(i) = sum_j A[i][j] e_{t+1}(j) b_{t+1}(j) / c_{t+1};
 *   marg_t(n) = a_t(n) b_t(n);  xi_t(i,j) = a_{t-1}(i) A[i][j] e_t(j) b_t(j) / c_t  (t >= 1);
 *   logZ = sum_t (log c_t + max_n loglik_t(n)).
 * xi_sum [N][N] = sum_{t>=1} xi_t(i,j) (nullable). */
int or_fb_pairwise(int T, int N, const double *loglik, const double *A, const double *pi, double *marg,
                   double *xi_sum, double *logZ) {
    double *fw = (double *)malloc(sizeof(double) * (size_t)T * N);
    double *bw = (double *)malloc(sizeof(double) * (size_t)T * N);
    double *e = (double *)malloc(sizeof(double) * (size_t)T * N);
    double *c = (double *)malloc(sizeof(double) * (size_t)T);
    double *mx = (double *)malloc(sizeof(double) * (size_t)T);
    int status = OR_OK;
    if (!fw || !bw || !e || !c || !mx) { status = OR_EINVAL; goto done; }
    for (int t = 0; t < T; ++t) {
        double m = -INFINITY;
        for (int n = 0; n < N; ++n) if (loglik[t * N + n] > m) m = loglik[t * N + n];
        if (!isfinite(m)) { status = OR_ENUMERIC; goto done; }
        mx[t] = m;
        for (int n = 0; n < N; ++n) e[t * N + n] = exp(loglik[t * N + n] - m);
    }
    for (int t = 0; t < T; ++t) {
        double ct = 0.0;
        for (int j = 0; j < N; ++j) {
            double p = 0.0;
            if (t == 0) p = pi[j];
            else for (int i = 0; i < N; ++i) p += fw[(t - 1) * N + i] * A[i * N + j];
            fw[t * N + j] = p * e[t * N + j];
            ct += fw[t * N + j];
        }
        if (!(ct > 0.0)) { status = OR_ENUMERIC; goto done; }
        c[t] = ct;
        for (int j = 0; j < N; ++j) fw[t * N + j] /= ct;
    }
    for (int n = 0; n < N; ++n) bw[(T - 1) * N + n] = 1.0;
    for (int t = T - 2; t >= 0; --t)
        for (int i = 0; i < N; ++i) {
            double acc = 0.0;
            for (int j = 0; j < N; ++j) acc += A[i * N + j] * e[(t + 1) * N + j] * bw[(t + 1) * N + j];
            bw[t * N + i] = acc / c[t + 1];
        }
    {
        double lz = 0.0;
        for (int t = 0; t < T; ++t) {
            double z = 0.0;
            for (int n = 0; n < N; ++n) { marg[t * N + n] = fw[t * N + n] * bw[t * N + n]; z += marg[t * N + n]; }
            for (int n = 0; n < N; ++n) marg[t * N + n] /= z;
            lz += log(c[t]) + mx[t];
        }
        *logZ = lz;
    }
    if (xi_sum) {
        for (int k = 0; k < N * N; ++k) xi_sum[k] = 0.0;
        for (int t = 1; t < T; ++t)
            for (int i = 0; i < N; ++i)
                for (int j = 0; j < N; ++j)
                    xi_sum[i * N + j] += fw[(t - 1) * N + i] * A[i * N + j] * e[t * N + j] * bw[t * N + j] / c[t];
    }
done:
    free(fw); free(bw); free(e); free(c); free(mx);
    return status;
}

/* E-step emission: loglik [T][N], loglik_{t,d} = sum_{l: V_lt > 0} V_lt log lhat_{t,d}(l).
 * Returns OR_EZEROSUPPORT when V_lt > 0 with lhat_{t,d}(l) = 0 for every d (no state can explain it). */
int or_nhmm_loglik(int F, int T, int N, int K, const double *V, const double *beta, const double *theta,
                   double *loglik) {
    for (int t = 0; t < T; ++t) {
        int any = 0;
        for (int d = 0; d < N; ++d) {
            double ll = 0.0;
            for (int l = 0; l < F; ++l) {
                const double v = V[t * F + l];
                if (v <= 0.0) continue;
                double lh = 0.0;
                for (int z = 0; z < K; ++z) lh += theta[(t * N + d) * K + z] * beta[(d * K + z) * F + l];
                ll += lh > 0.0 ? v * log(lh) : -INFINITY;
            }
            loglik[t * N + d] = ll;
            if (ll > -INFINITY) any = 1;
        }
        if (!any) return OR_EZEROSUPPORT;
    }
    return OR_OK;
}

/* S:214 (DESIGN R21): floor at 1e-12, then renormalise. */
static void floor_renorm(double *p, int n) {
    double s = 0.0;
    for (int i = 0; i < n; ++i) {
        if (p[i] < 1e-12) p[i] = 1e-12;
        s += p[i];
    }
    for (int i = 0; i < n; ++i) p[i] /= s;
}

/* One EM iteration (order of the file header).  beta, theta, A, pi are updated in place; *loglik_out is
 * the log evidence of the parameters the iteration started from. */
int or_nhmm_em_step(int F, int T, int N, int K, const double *V, double *beta, double *theta, double *A,
                    double *pi, double *loglik_out) {
    double *ll = (double *)malloc(sizeof(double) * (size_t)T * N);
    double *g = (double *)malloc(sizeof(double) * (size_t)T * N);
    double *xi = (double *)malloc(sizeof(double) * (size_t)N * N);
    double *nb = (double *)calloc((size_t)N * K * F, sizeof(double));
    double *nt = (double *)malloc(sizeof(double) * (size_t)T * N * K);
    int st = OR_OK;
    if (!ll || !g || !xi || !nb || !nt) { st = OR_EINVAL; goto done; }
    st = or_nhmm_loglik(F, T, N, K, V, beta, theta, ll);
    if (st) goto done;
    st = or_fb_pairwise(T, N, ll, A, pi, g, xi, loglik_out);
    if (st) goto done;
    /* responsibilities P(z | l, t, d) and the two M-step sums */
    for (int t = 0; t < T; ++t)
        for (int d = 0; d < N; ++d) {
            const double *th = theta + (size_t)(t * N + d) * K;
            double *ntd = nt + (size_t)(t * N + d) * K;
            for (int z = 0; z < K; ++z) ntd[z] = 0.0;
            for (int l = 0; l < F; ++l) {
                const double v = V[t * F + l];
                if (v <= 0.0) continue;
                double lh = 0.0;
                for (int z = 0; z < K; ++z) lh += th[z] * beta[(d * K + z) * F + l];
                if (!(lh > 0.0)) continue;   /* this state cannot explain the quantum: weight 0 */
                for (int z = 0; z < K; ++z) {
                    const double pz = th[z] * beta[(d * K + z) * F + l] / lh;   /* P(z | l, t, d) */
                    ntd[z] += v * pz;
                    nb[(d * K + z) * F + l] += g[t * N + d] * v * pz;
                }
            }
        }
    /* M-step */
    for (int t = 0; t < T; ++t)
        for (int d = 0; d < N; ++d) {
            double s = 0.0;
            for (int z = 0; z < K; ++z) s += nt[(size_t)(t * N + d) * K + z];
            if (s > 0.0)   /* an empty frame (or a state with no support) keeps its weights */
                for (int z = 0; z < K; ++z) theta[(size_t)(t * N + d) * K + z] = nt[(size_t)(t * N + d) * K + z] / s;
        }
    for (int dz = 0; dz < N * K; ++dz) {
        double s = 0.0;
        for (int l = 0; l < F; ++l) s += nb[dz * F + l];
        if (s > 0.0)
            for (int l = 0; l < F; ++l) beta[dz * F + l] = nb[dz * F + l] / s;
        floor_renorm(beta + (size_t)dz * F, F);
    }
    for (int i = 0; i < N; ++i) {
        double s = 0.0;
        for (int j = 0; j < N; ++j) s += xi[i * N + j];
        if (s > 0.0)
            for (int j = 0; j < N; ++j) A[i * N + j] = xi[i * N + j] / s;
        floor_renorm(A + (size_t)i * N, N);
    }
    for (int d = 0; d < N; ++d) pi[d] = g[d];
    floor_renorm(pi, N);   /* pi is the chain's other parameter: the same floor (DESIGN R21) */
done:
    free(ll); free(g); free(xi); free(nb); free(nt);
    return st;
}
