/*
 * nfhmm_oracle.c -- plain, slow, single-threaded FP64 CPU oracle for the variational
 * inference iteration of the Bayesian N-FHMM (Mysore & Sahani, ICML 2012, arXiv 1206.6468).
 *
 * ORACLE -- TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  The product path
 * (paper_1206_6468_b200/, libnfhmm.so) never links, imports or calls it, and it shares no code,
 * header, table or constant with the CUDA path.
 *
 * Citation keys: "P:n" = /root/reference/PAPER.md line n, "S:n" = SPEC.md line n,
 * "DESIGN Rn" = reading n listed in DESIGN.md section "Readings of the paper".
 *
 * Every function follows the paper's equations literally, in the paper's order and notation:
 *   - Eq. 7: log z_{t,l,k} = log beta_l(k) + psi(alpha_{t,k}) - psi(sum_k alpha_{t,k}) - kappa,
 *     evaluated per (t,l) with kappa the explicit log normaliser (linear domain, FP64);
 *   - Eq. 6: alpha_{t,k} = sum_l V_lt z_{t,l,k} + gamma sum_s sum_n d_{t,n}^{(s)} B_snk + 1;
 *   - Eq. 8: phi_{t,n}^{(s)} = sum_k B_snk (psi(alpha_{t,k}) - psi(sum_k alpha_{t,k}));
 *   - forward-backward per source (Rabiner 1989) on log-likelihood gamma*phi (DESIGN R1);
 *   - separation.
 * Element order: k = (s*N + n)*K + j, source-major, dictionary-major, element-minor, so
 * B_snk = 1 iff floor(k/K) == s*N+n ("do not share dictionary elements").
 *
 * Array layouts (row-major, all inputs FP32 as stored by the generator, upcast to FP64 here):
 *   beta  [S][N][K][F]   beta_l(k) = beta[k*F + l]
 *   trans [S][N][N]      trans[s][i][j] = P(D_t=j | D_{t-1}=i) (row-stochastic; DESIGN R4)
 *   prior [S][N]         pi^(s)
 *   V     [T][F]         V_lt stored as V[t*F + l]
 *   alpha [T][Kt], d_hat [S][T][N], V_hat [T][F], V_src/V_star [S][T][F]
 *
 * Parity pins: see tests/test_oracle_pins.py (every function here is pinned; none is "parity unpinned").
 */
#include <math.h>
#include <stdlib.h>
#include <string.h>

#define OR_OK 0
#define OR_EINVAL (-1)
#define OR_EZEROSUPPORT (-5)
#define OR_ENUMERIC (-6)

/* psi(x), x > 0.  Eq. 7: "psi(.) is the digamma function".
 * Recurrence psi(x) = psi(x+1) - 1/x until x >= 10, then the asymptotic series
 * psi(x) ~ ln x - 1/(2x) - sum_{n=1..7} B_{2n} / (2n x^{2n}).  Truncation < 1e-16 at x >= 10. */
double or_digamma(double x) {
    if (!(x > 0.0)) return NAN;
    double r = 0.0;
    while (x < 10.0) { r -= 1.0 / x; x += 1.0; }
    double f = 1.0 / (x * x);
    double series = f * (-1.0 / 12.0 + f * (1.0 / 120.0 + f * (-1.0 / 252.0 + f * (1.0 / 240.0 +
                    f * (-1.0 / 132.0 + f * (691.0 / 32760.0 + f * (-1.0 / 12.0)))))));
    return r + log(x) - 0.5 / x + series;
}

/* Eq. 1 / P:111: alpha_k(D_t) = 1 + gamma * sum_s sum_n delta_{t,n}^{(s)} B_snk for given states. */
int or_prior_alpha(int S, int N, int K, double gamma, const int *states, double *alpha_out) {
    int Kt = S * N * K;
    for (int k = 0; k < Kt; ++k) {
        double acc = 0.0;
        for (int s = 0; s < S; ++s)
            for (int n = 0; n < N; ++n) {
                int B = (k / K) == (s * N + n);             /* B_snk, S:250 ordering */
                int delta = (states[s] == n);               /* delta_{t,n}^{(s)} */
                acc += (double)(delta * B);
            }
        alpha_out[k] = 1.0 + gamma * acc;
    }
    return OR_OK;
}

/* Scaled forward-backward for one chain ("exact inference is efficient using the
 * forward-backward algorithm"; Rabiner 1989; stability scheme S:138: per-frame rescaling on
 * exp(loglik - rowmax)).  loglik [T][N], A [N][N] row-stochastic (A[i][j] = P(j|i)), pi [N].
 * Outputs marg [T][N] = q(D_t = n) and *logZ = log sum_paths pi A.. exp(sum_t loglik).
 * Returns OR_ENUMERIC when the evidence is zero (explicit error, not NaN). */
int or_forward_backward(int T, int N, const double *loglik, const double *A, const double *pi,
                        double *marg, double *logZ) {
    double *fw = (double *)malloc(sizeof(double) * (size_t)T * N);
    double *bw = (double *)malloc(sizeof(double) * (size_t)T * N);
    double *c = (double *)malloc(sizeof(double) * (size_t)T);
    double *e = (double *)malloc(sizeof(double) * (size_t)T * N);
    double *mx = (double *)malloc(sizeof(double) * (size_t)T);
    int status = OR_OK;
    if (!fw || !bw || !c || !e || !mx) { status = OR_EINVAL; goto done; }
    /* emissions e_t(n) = exp(loglik_t(n) - max_n loglik_t(n)) */
    for (int t = 0; t < T; ++t) {
        double m = -INFINITY;
        for (int n = 0; n < N; ++n) if (loglik[t * N + n] > m) m = loglik[t * N + n];
        if (!isfinite(m)) { status = OR_ENUMERIC; goto done; }
        mx[t] = m;
        for (int n = 0; n < N; ++n) e[t * N + n] = exp(loglik[t * N + n] - m);
    }
    /* forward: a_1 = pi .* e_1 / c_1; a_t = (a_{t-1} A) .* e_t / c_t */
    for (int t = 0; t < T; ++t) {
        double ct = 0.0;
        for (int j = 0; j < N; ++j) {
            double p;
            if (t == 0) p = pi[j];
            else {
                p = 0.0;
                for (int i = 0; i < N; ++i) p += fw[(t - 1) * N + i] * A[i * N + j];
            }
            fw[t * N + j] = p * e[t * N + j];
            ct += fw[t * N + j];
        }
        if (!(ct > 0.0)) { status = OR_ENUMERIC; goto done; }
        c[t] = ct;
        for (int j = 0; j < N; ++j) fw[t * N + j] /= ct;
    }
    /* backward: b_T = 1; b_t(i) = sum_j A[i][j] e_{t+1}(j) b_{t+1}(j) / c_{t+1} */
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
done:
    free(fw); free(bw); free(c); free(e); free(mx);
    return status;
}

/* Elog[k] = psi(alpha_k) - psi(sum_k' alpha_k') for one frame (the digamma terms of Eqs. 7, 8). */
static void expected_log_theta(int Kt, const double *alpha_t, double *elog) {
    double a0 = 0.0;
    for (int k = 0; k < Kt; ++k) a0 += alpha_t[k];
    double psi0 = or_digamma(a0);
    for (int k = 0; k < Kt; ++k) elog[k] = or_digamma(alpha_t[k]) - psi0;
}

/* Explicit z_hat [T][F][Kt] by Eq. 7 (for tiny-instance tests of Sum_k z = 1 and S:280-282). */
int or_z_hat(int F, int T, int S, int N, int K, const float *beta, const double *alpha, double *z_out) {
    int Kt = S * N * K;
    double *elog = (double *)malloc(sizeof(double) * Kt);
    for (int t = 0; t < T; ++t) {
        expected_log_theta(Kt, alpha + (size_t)t * Kt, elog);
        for (int l = 0; l < F; ++l) {
            double *z = z_out + ((size_t)t * F + l) * Kt;
            double kap = 0.0;                                   /* kappa = log sum_k exp(...) */
            for (int k = 0; k < Kt; ++k) { z[k] = (double)beta[(size_t)k * F + l] * exp(elog[k]); kap += z[k]; }
            if (!(kap > 0.0)) { free(elog); return OR_EZEROSUPPORT; }
            for (int k = 0; k < Kt; ++k) z[k] /= kap;
        }
    }
    free(elog);
    return OR_OK;
}

/* One z-step (Eq. 7) followed by one alpha-step (Eq. 6), literal per (t,l):
 *   for each t, l with V_lt > 0: z_k = beta_l(k) exp(Elog_k) / kappa_tl; cnt_k += V_lt z_k;
 *   alpha_new[t,k] = cnt_k + gamma * d_hat^{(s(k))}_{t, n(k)} + 1.
 * Also returns V_hat[t,l] = kappa_tl = sum_k beta_l(k) exp(Elog_k) (the Eq. 7 normaliser in the linear
 * domain) and data_term = sum_{t,l} V_lt log V_hat[t,l] (the z part of the bound, DESIGN R8).
 * Any of alpha_new / V_hat / data_term may be NULL. */
int or_z_alpha_step(int F, int T, int S, int N, int K, double gamma, const float *beta, const float *V,
                    const double *alpha, const double *d_hat, double *alpha_new, double *V_hat,
                    double *data_term) {
    int Kt = S * N * K;
    double *elog = (double *)malloc(sizeof(double) * Kt);
    double *th = (double *)malloc(sizeof(double) * Kt);
    double *z = (double *)malloc(sizeof(double) * Kt);
    double *cnt = (double *)malloc(sizeof(double) * Kt);
    double data = 0.0;
    int status = OR_OK;
    for (int t = 0; t < T; ++t) {
        expected_log_theta(Kt, alpha + (size_t)t * Kt, elog);
        for (int k = 0; k < Kt; ++k) { th[k] = exp(elog[k]); cnt[k] = 0.0; }
        for (int l = 0; l < F; ++l) {
            double v = (double)V[(size_t)t * F + l];
            double kap = 0.0;
            for (int k = 0; k < Kt; ++k) { z[k] = (double)beta[(size_t)k * F + l] * th[k]; kap += z[k]; }
            if (V_hat) V_hat[(size_t)t * F + l] = kap;
            if (v > 0.0) {
                if (!(kap > 0.0)) { status = OR_EZEROSUPPORT; goto done; }
                for (int k = 0; k < Kt; ++k) cnt[k] += v * (z[k] / kap);
                data += v * log(kap);
            }
        }
        if (alpha_new) {
            for (int k = 0; k < Kt; ++k) {
                int blk = k / K;                       /* = s*N + n with B_snk = 1 */
                int s = blk / N, n = blk % N;
                alpha_new[(size_t)t * Kt + k] = cnt[k] + gamma * d_hat[((size_t)s * T + t) * N + n] + 1.0;
            }
        }
    }
done:
    if (data_term) *data_term = data;
    free(elog); free(th); free(z); free(cnt);
    return status;
}

/* Eq. 8: phi [S][T][N], phi_{t,n}^{(s)} = sum_k B_snk (psi(alpha_k) - psi(sum alpha)). */
int or_surrogate(int T, int S, int N, int K, const double *alpha, double *phi) {
    int Kt = S * N * K;
    double *elog = (double *)malloc(sizeof(double) * Kt);
    for (int t = 0; t < T; ++t) {
        expected_log_theta(Kt, alpha + (size_t)t * Kt, elog);
        for (int s = 0; s < S; ++s)
            for (int n = 0; n < N; ++n) {
                double acc = 0.0;
                for (int k = 0; k < Kt; ++k) if (k / K == s * N + n) acc += elog[k];
                phi[((size_t)s * T + t) * N + n] = acc;
            }
    }
    free(elog);
    return OR_OK;
}

/* D-step: forward-backward per source on log-likelihood gamma * phi (DESIGN R1).
 * d_hat [S][T][N] out, logZ [S] out. */
int or_d_step(int T, int S, int N, double gamma, const float *trans, const float *prior,
              const double *phi, double *d_hat, double *logZ) {
    double *ll = (double *)malloc(sizeof(double) * (size_t)T * N);
    double *A = (double *)malloc(sizeof(double) * (size_t)N * N);
    double *pi = (double *)malloc(sizeof(double) * N);
    int status = OR_OK;
    for (int s = 0; s < S && status == OR_OK; ++s) {
        for (int i = 0; i < N * N; ++i) A[i] = (double)trans[(size_t)s * N * N + i];
        for (int i = 0; i < N; ++i) pi[i] = (double)prior[(size_t)s * N + i];
        for (size_t i = 0; i < (size_t)T * N; ++i) ll[i] = gamma * phi[(size_t)s * T * N + i];
        status = or_forward_backward(T, N, ll, A, pi, d_hat + (size_t)s * T * N, &logZ[s]);
    }
    free(ll); free(A); free(pi);
    return status;
}

/* Entropy of Dirichlet(alpha) over Kt elements (used in the bound, DESIGN R8):
 * H = sum_k lnGamma(a_k) - lnGamma(a0) + (a0 - Kt) psi(a0) - sum_k (a_k - 1) psi(a_k). */
double or_dirichlet_entropy(int Kt, const double *a) {
    double a0 = 0.0, h = 0.0;
    for (int k = 0; k < Kt; ++k) a0 += a[k];
    for (int k = 0; k < Kt; ++k) h += lgamma(a[k]) - (a[k] - 1.0) * or_digamma(a[k]);
    h += -lgamma(a0) + (a0 - (double)Kt) * or_digamma(a0);
    return h;
}

/* Closed-form bound at (z(alpha), alpha, q(D) = FB posterior on gamma*phi(alpha)), DESIGN R8:
 * L = sum_{t,l} V log V_hat + sum_t H_Dir(alpha_t) + sum_s log Z_s + T [lnG(Kt + gamma S K) - S K lnG(1+gamma)]. */
double or_bound(int T, int S, int N, int K, double gamma, double data_term, const double *alpha,
                const double *logZ) {
    int Kt = S * N * K;
    double L = data_term;
    for (int t = 0; t < T; ++t) L += or_dirichlet_entropy(Kt, alpha + (size_t)t * Kt);
    for (int s = 0; s < S; ++s) L += logZ[s];
    L += (double)T * (lgamma((double)Kt + gamma * S * K) - (double)S * K * lgamma(1.0 + gamma));
    return L;
}

/* Section 4: V_src[s][t][l] = v_t * sum_{k in s} beta_l(k) E[theta_{t,k}], with
 * E[theta] = alpha / sum alpha (DESIGN R9); V_star = V * V_src / sum_s' V_src (1/S where the
 * denominator is 0).  Either output may be NULL. */
int or_separate(int F, int T, int S, int N, int K, const float *beta, const float *V,
                const double *alpha, double *V_src, double *V_star) {
    int Kt = S * N * K, NK = N * K;
    double *rec = (double *)malloc(sizeof(double) * (size_t)S * F);
    for (int t = 0; t < T; ++t) {
        const double *a = alpha + (size_t)t * Kt;
        double a0 = 0.0, vt = 0.0;
        for (int k = 0; k < Kt; ++k) a0 += a[k];
        for (int l = 0; l < F; ++l) vt += (double)V[(size_t)t * F + l];
        for (int s = 0; s < S; ++s)
            for (int l = 0; l < F; ++l) {
                double acc = 0.0;
                for (int k = s * NK; k < (s + 1) * NK; ++k) acc += (double)beta[(size_t)k * F + l] * (a[k] / a0);
                rec[s * F + l] = vt * acc;
            }
        for (int l = 0; l < F; ++l) {
            double den = 0.0;
            for (int s = 0; s < S; ++s) den += rec[s * F + l];
            for (int s = 0; s < S; ++s) {
                if (V_src) V_src[((size_t)s * T + t) * F + l] = rec[s * F + l];
                if (V_star) V_star[((size_t)s * T + t) * F + l] =
                    den > 0.0 ? (double)V[(size_t)t * F + l] * rec[s * F + l] / den
                              : (double)V[(size_t)t * F + l] / (double)S;
            }
        }
    }
    free(rec);
    return OR_OK;
}

/* Full VB run ("We iterate over Eqs. 6, 7, 8, and the forward-backward algorithm for each
 * source"), order z -> alpha -> phi -> FB per sweep (DESIGN R6), initialisation alpha = 1 + gamma/N,
 * d = 1/N (DESIGN R5).  After the last sweep a trailing z-step gives V_hat_n and the data term of
 * L_n (DESIGN R7).  free_energy[i-1] = L_i for i = 1..n_iters.
 * alpha_io/d_io: if init_state != 0 they hold the starting state (resume); otherwise initialised here.
 * Outputs: alpha_io [T][Kt], d_io [S][T][N], V_hat [T][F] (nullable), free_energy [n_iters]
 * (nullable), logZ_out [S] (nullable, of the final sweep). */
int or_vb_run(int F, int T, int S, int N, int K, double gamma, const float *beta, const float *trans,
              const float *prior, const float *V, int n_iters, int init_state, double *alpha_io,
              double *d_io, double *V_hat, double *free_energy, double *logZ_out) {
    if (F < 1 || T < 1 || S < 1 || N < 1 || K < 1 || n_iters < 0) return OR_EINVAL;
    int Kt = S * N * K;
    size_t TK = (size_t)T * Kt;
    double *alpha_new = (double *)malloc(sizeof(double) * TK);
    double *phi = (double *)malloc(sizeof(double) * (size_t)S * T * N);
    double *logZ = (double *)calloc((size_t)S, sizeof(double));
    int status = OR_OK;
    if (!init_state) {
        for (size_t i = 0; i < TK; ++i) alpha_io[i] = 1.0 + gamma / (double)N;
        for (size_t i = 0; i < (size_t)S * T * N; ++i) d_io[i] = 1.0 / (double)N;
    }
    for (int it = 1; it <= n_iters; ++it) {
        double data = 0.0;
        status = or_z_alpha_step(F, T, S, N, K, gamma, beta, V, alpha_io, d_io, alpha_new, NULL, &data);
        if (status) goto done;
        if (it >= 2 && free_energy)   /* L_{it-1} uses this sweep's z-step of alpha_{it-1} */
            free_energy[it - 2] = or_bound(T, S, N, K, gamma, data, alpha_io, logZ);
        memcpy(alpha_io, alpha_new, sizeof(double) * TK);
        or_surrogate(T, S, N, K, alpha_io, phi);
        status = or_d_step(T, S, N, gamma, trans, prior, phi, d_io, logZ);
        if (status) goto done;
    }
    if (n_iters >= 1 || V_hat) {
        double data = 0.0;
        status = or_z_alpha_step(F, T, S, N, K, gamma, beta, V, alpha_io, d_io, NULL, V_hat, &data);
        if (status) goto done;
        if (n_iters >= 1 && free_energy)
            free_energy[n_iters - 1] = or_bound(T, S, N, K, gamma, data, alpha_io, logZ);
    }
    if (logZ_out) for (int s = 0; s < S; ++s) logZ_out[s] = logZ[s];
done:
    free(alpha_new); free(phi); free(logZ);
    return status;
}
