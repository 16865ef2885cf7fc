/*
 * nfhmm.h -- C-ABI of libnfhmm: B200-native (sm_100a) variational inference for the Bayesian
 * non-negative factorial HMM of Mysore & Sahani, "Variational Inference in Non-negative Factorial
 * Hidden Markov Models for Efficient Audio Source Separation", ICML 2012 (arXiv 1206.6468).
 *
 * Citation keys: "P:n" = line n of PAPER.md (the paper text), "S:n" = line n of SPEC.md,
 * "DESIGN Rn" = reading n in DESIGN.md section "Readings of the paper".
 *
 * What one call of nfhmm_vb_iterate computes, per mixture and per sweep ("We iterate over
 * Eqs. 6, 7, 8, and the forward-backward algorithm for each source"; order z -> alpha -> phi -> FB,
 * DESIGN R6):
 *   Eq. 7  z_{t,l,k} = beta_l(k) exp(psi(alpha_{t,k}) - psi(sum_k alpha_{t,k})) / V_hat_{t,l},
 *                  V_hat_{t,l} = sum_k beta_l(k) exp(psi(alpha_{t,k}) - psi(sum_k alpha_{t,k}))
 *                  (z is never materialised: only V / V_hat is needed);
 *   Eq. 6  alpha_{t,k} = sum_l V_lt z_{t,l,k} + gamma sum_{s,n} d_{t,n}^{(s)} B_snk + 1;
 *   Eq. 8  phi_{t,n}^{(s)} = sum_k B_snk (psi(alpha_{t,k}) - psi(sum_k alpha_{t,k}));
 *   forward-backward per source on log-likelihood gamma * phi (DESIGN R1) -> d;
 *   the variational bound L (closed form DESIGN R8) per sweep, FP64.
 * nfhmm_separate computes Section 4: V_src^(s) = v_t sum_{k in s} beta_l(k) E[theta_tk],
 * E[theta] = alpha / sum alpha (DESIGN R9), and V*^(s) = V V_src^(s) / sum_s' V_src^(s').
 *
 * Dimensions: F frequency bins (l), T frames (t), S sources (s), N states per source (n), K elements
 * per state dictionary; Kt = S*N*K global elements, ordered k = (s*N + n)*K + j, so
 * B_snk = 1 iff floor(k / K) == s*N + n (sources do not share elements).
 *
 * Pointers: every array argument may be a HOST pointer (pageable or pinned) or a DEVICE pointer on
 * the handle's device; the library tells them apart with cudaPointerGetAttributes and copies with
 * cudaMemcpy*Async on the handle's stream.  All arrays are dense row-major FP32 (FP64 where stated).
 * Ownership: inputs are borrowed for the duration of the call only (copied into the workspace);
 * outputs go to caller-allocated buffers; the handle owns nothing the caller passed in.
 * Threading: a handle is single-threaded; handles on different devices are independent.
 * Errors: every function returns an NFHMM_* status; nothing aborts or throws across the ABI; the
 * detail of the last failure is in nfhmm_last_error().  Device-side conditions (zero support,
 * non-finite values) are sticky flags read once per nfhmm_vb_iterate / nfhmm_sync.
 */
#ifndef NFHMM_H
#define NFHMM_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define NFHMM_OK 0
#define NFHMM_EINVAL (-1)        /* bad dimension, NULL where required, negative/non-finite input,
                                    dictionary column / transition row / prior not normalised (1e-4) */
#define NFHMM_ESTATE (-2)        /* call order violated: create -> [workspace] -> model -> observations
                                    -> iterate -> posteriors / separate */
#define NFHMM_ECUDA (-3)         /* CUDA runtime error; text in nfhmm_last_error */
#define NFHMM_ENOMEM (-4)        /* workspace too small / allocation failed */
#define NFHMM_EZEROSUPPORT (-5)  /* some V_lt > 0 with V_hat_lt = 0 */
#define NFHMM_ENUMERIC (-6)      /* non-finite alpha, phi or log Z */

typedef struct nfhmm nfhmm_t;     /* opaque, library-owned */

#define NFHMM_MATH_TC 0          /* 3xTF32 split on tcgen05: a_lo b_hi + a_hi b_lo + a_hi b_hi, FP32 accumulate */
#define NFHMM_MATH_SIMT 1        /* FP32 FFMA register tiles */

typedef struct {
    int64_t n_mix;      /* independent mixtures (same model) on this handle; default 1           */
    double gamma;       /* Dirichlet concentration gamma >= 0 ("we took gamma = 1"); default 1 */
    int32_t device;     /* CUDA ordinal; default 0                                              */
    int32_t max_iters;  /* capacity of the per-mixture free-energy trace; default 1024            */
    int32_t free_energy;/* 1 = assemble L every sweep (default), 0 = skip the FP64 bound terms      */
    int32_t math;       /* contraction engine for (a)/(b): NFHMM_MATH_TC (default) = tcgen05 3xTF32
                           tensor cores; NFHMM_MATH_SIMT = FP32 FFMA tiles                        */
    void *stream;       /* cudaStream_t to launch on (e.g. torch.cuda.current_stream().cuda_stream);
                           NULL = the legacy default stream                                      */
} nfhmm_options;

/* Fill *opt with the defaults above. */
void nfhmm_default_options(nfhmm_options *opt);

/* Create a handle for n_mix mixtures of F x T counts with S sources of N states x K elements.
 * opt may be NULL (defaults).  Validates dims (all >= 1, Kt and padded sizes fit in int32 rows).
 * *out receives the handle; on error *out = NULL. */
int nfhmm_create(int64_t F, int64_t T, int32_t S, int32_t N, int32_t K, const nfhmm_options *opt,
                 nfhmm_t **out);

/* Device bytes the handle needs (all state, 256-B aligned sub-buffers). */
int nfhmm_workspace_size(const nfhmm_t *h, size_t *bytes);

/* Hand the handle a caller-owned device buffer of >= nfhmm_workspace_size bytes (e.g. a torch
 * uint8 tensor).  dptr = NULL, bytes = 0 asks the library to cudaMalloc (and free in destroy).
 * The hot path never allocates.  Must precede set_model. */
int nfhmm_set_workspace(nfhmm_t *h, void *dptr, size_t bytes);

/* Source models: dict [S][N][K][F] = beta_l(k) at dict[k*F + l], each column >= 0
 * summing to 1 (+-1e-4); trans [S][N][N] row-stochastic, trans[s][i][j] = P(D_t = j | D_{t-1} = i)
 * (= rho^(s) transposed, DESIGN R4); prior [S][N] = pi^(s), sums to 1 (+-1e-4).
 * Shared by all mixtures of the handle. */
int nfhmm_set_model(nfhmm_t *h, const float *dict, const float *trans, const float *prior);

/* Observed spectrogram counts V [n_mix][T][F] (V_lt at V[(m*T + t)*F + l]), >= 0 and
 * finite.  Implies nfhmm_reset. */
int nfhmm_set_observations(nfhmm_t *h, const float *V);

/* Initial state (DESIGN R5): alpha = 1 + gamma/N, d = 1/N, then the z-step of that state.  Clears
 * the free-energy trace and the iteration counter. */
int nfhmm_reset(nfhmm_t *h);

/* Run n_iters sweeps (each: Eq. 6 alpha-step from the current z, Eq. 8, forward-backward per source,
 * then the Eq. 7 z-step of the new alpha, which also gives L of the sweep), then synchronise the
 * stream and check the device error flags.  Sweeps accumulate across calls (resume). */
int nfhmm_vb_iterate(nfhmm_t *h, int32_t n_iters);

/* Same, without the final synchronisation / flag check (enqueue only).  Follow with nfhmm_sync. */
int nfhmm_vb_iterate_async(nfhmm_t *h, int32_t n_iters);

/* Synchronise the handle's stream and return the sticky device error status. */
int nfhmm_sync(nfhmm_t *h);

/* Copy out the current posteriors (any output may be NULL):
 *   d_hat       [n_mix][S][T][N]  q(D_t^(s) = n)
 *   alpha_hat   [n_mix][T][Kt]    Dirichlet parameters of q(theta_t) (Eq. 6)
 *   V_hat       [n_mix][T][F]     sum_k beta_l(k) exp(E log theta_tk) for the current alpha (Eq. 7
 *                                 normaliser, DESIGN R7)
 *   free_energy [n_mix][max_iters] FP64 bound L_i, i = 1..iters_done (row stride max_iters)
 *   iters_done  number of sweeps since the last reset
 * Synchronises. */
int nfhmm_posteriors(nfhmm_t *h, float *d_hat, float *alpha_hat, float *V_hat, double *free_energy,
                     int32_t *iters_done);

/* Section 4 separation from the current alpha: V_star [n_mix][S][T][F] (required),
 * V_src [n_mix][S][T][F] (nullable, the unmasked V_hat^(s)).  Synchronises. */
int nfhmm_separate(nfhmm_t *h, float *V_star, float *V_src);

/* Same, enqueue only (no synchronisation, no flag check; follow with nfhmm_sync).  Host outputs must
 * be pinned for the copies to stay asynchronous, and must not be read before nfhmm_sync returns.
 * With two handles on two streams a caller pipelines batches: one handle's host<->device copies run
 * while the other computes. */
int nfhmm_separate_async(nfhmm_t *h, float *V_star, float *V_src);

/* Free the handle (and the workspace if the library allocated it). NULL is a no-op. */
int nfhmm_destroy(nfhmm_t *h);

/* Static text for a status code. */
const char *nfhmm_strerror(int status);

/* Detail of the last failure on h (empty string if none). */
const char *nfhmm_last_error(const nfhmm_t *h);

/* Number of kernels this handle has launched since creation (evidence for bench gpu_launches). */
int nfhmm_kernel_launches(const nfhmm_t *h, int64_t *count);

/* Tile configuration chosen for the handle: padded F (BN of the reconstruction GEMM multiple) and
 * padded Kt (BN of the back-projection GEMM multiple).  Informational. */
int nfhmm_layout(const nfhmm_t *h, int64_t *F_pad, int64_t *Kt_pad, int32_t *bn_recon,
                 int32_t *bn_backproj);

/* Bounds checker (in place of compute-sanitizer, which this pool does not run).  When the
 * environment variable NFHMM_GUARD=<bytes> (0 .. 2^30) is set at nfhmm_create, the workspace carries a
 * guard zone before its first piece and after every piece: from the piece's exact end (its byte count,
 * not its 256-byte rounding) to the next piece, at least <bytes> long.  nfhmm_set_workspace fills the
 * zones with the byte 0xA5; nfhmm_workspace_size includes them.  nfhmm_guard_check synchronises the
 * handle's streams and copies every zone to the host: *checked_bytes = the zone bytes inspected (0 when
 * NFHMM_GUARD was unset), *bad_bytes = those no longer 0xA5, i.e. written by a kernel or copy outside
 * the extent of a workspace piece.  Returns NFHMM_ECUDA if *bad_bytes > 0 (nfhmm_last_error names the
 * first piece whose zone was hit, in carve order; -1 = before the first piece), NFHMM_ESTATE before a
 * workspace exists, NFHMM_EINVAL for NULL arguments.  Debug/test instrument: reads of a zone are not
 * detected here, but they see 0xA5 instead of 0, which the parity tests (bitwise against an unguarded
 * handle) expose. */
int nfhmm_guard_check(nfhmm_t *h, int64_t *checked_bytes, int64_t *bad_bytes);

/* How the two contractions of the sweep form their products (informational; DESIGN "3xFP16 products"):
 *   NFHMM_PRODUCTS_FFMA   FP32 FFMA tiles (SIMT engine);
 *   NFHMM_PRODUCTS_3XTF32 tcgen05 kind::tf32, x = hi + lo with hi = rn_tf32(x), three MMAs per product;
 *   NFHMM_PRODUCTS_3XFP16 tcgen05 kind::f16, the operands scaled by exact powers of two and split into
 *                         FP16 hi + lo (the same 11-bit significands as TF32), three MMAs per product.
 * Either pointer may be NULL.  Returns NFHMM_EINVAL for h == NULL. */
#define NFHMM_PRODUCTS_FFMA 0
#define NFHMM_PRODUCTS_3XTF32 1
#define NFHMM_PRODUCTS_3XFP16 2
int nfhmm_products(const nfhmm_t *h, int32_t *recon, int32_t *backproj);

/* Per-kernel-class device timing: when enabled, every launch on the handle's stream is bracketed by
 * CUDA events (no host synchronisation).  Classes: */
#define NFHMM_K_RECON 0      /* (a) reconstruction GEMM + ratio epilogue (z-step, Eq. 7)          */
#define NFHMM_K_BACKPROJ 1   /* (b) back-projection GEMM (Eq. 6 data term)                          */
#define NFHMM_K_DIRICHLET 2  /* (c)+(d) Eq. 6 update, digamma/exp, Eq. 8                             */
#define NFHMM_K_FB 3         /* (e) forward-backward                                                 */
#define NFHMM_K_ELBO 4       /* (g) bound reduction                                                  */
#define NFHMM_K_SEPARATE 5   /* (f) Section 4 reconstruction GEMMs + ratio mask                      */
#define NFHMM_K_OTHER 6      /* initial state, observation statistics, dictionary transpose          */
#define NFHMM_NUM_KERNEL_CLASSES 7
/* on != 0 starts recording (and clears previous records); on = 0 stops.  While recording, sweeps run
 * eagerly (no CUDA graphs) and without the forward-backward / reconstruction overlap, so every class is
 * timed on its own. */
int nfhmm_profile_enable(nfhmm_t *h, int on);
/* Synchronise and return, per class, the summed device milliseconds and launch counts recorded since
 * the last enable.  Both arrays have NFHMM_NUM_KERNEL_CLASSES entries; either may be NULL. */
int nfhmm_profile_read(nfhmm_t *h, double *ms, int64_t *launches);

/* Instrumentation: launch ONE kernel class (NFHMM_K_RECON, _BACKPROJ, _DIRICHLET or _FB) `reps` times
 * back to back on the handle's current state and return the mean device time per launch (CUDA events
 * on the handle's stream).  The repeated step leaves the iteration state inconsistent, so the call
 * ends with nfhmm_reset (iters_done = 0, free-energy trace restarted).  Synchronises.
 * Errors: NFHMM_ESTATE before model + observations; NFHMM_EINVAL for another class, reps < 1 or a NULL
 * ms_per_launch. */
int nfhmm_bench_kernel(nfhmm_t *h, int cls, int32_t reps, double *ms_per_launch);

/* ---------------------------------------------------------------------------------------------------
 * Spectrogram front end and resynthesis back end.  Stateless calls on `device`
 * and `stream` (cudaStream_t or NULL); arrays may be host or device pointers (host ones are staged);
 * both synchronise the stream before returning.  Window: periodic Hann w[n] = 1/2 - 1/2 cos(2 pi n / win),
 * DFT length = win (a power of two, 2 .. 4096), hop <= win (DESIGN R23); the paper's analysis is
 * win = 1024, hop = 256 at 16 kHz ("a window size of 64ms and a hop size of 16ms").
 *
 * nfhmm_stft ("A spectrogram is the magnitude of the short-time Fourier transform"):
 *   x [n_sig][n_samples] FP32 waveforms (n_samples >= win, n_sig <= 65535);
 *   T = 1 + (n_samples - win) / hop frames, F = win / 2 + 1 bins;
 *   X [n_sig][T][F] complex64 as interleaved (re, im) FP32 pairs:  X_t[k] = sum_n w[n] x[t hop + n] e^{-2 pi i k n / win}
 *   V [n_sig][T][F] FP32 quanta  V = gain |X|  (the observations of nfhmm_set_observations);
 *   either output may be NULL (not both); gain > 0.
 * nfhmm_istft ("go back to the time domain ... using the phase of the original mixture"):
 *   X [n_mix][T][F] complex64 mixture STFT (from nfhmm_stft), M [n_mix][S][T][F] per-source magnitudes in
 *   quanta (e.g. V* of nfhmm_separate; divided by gain), y [n_mix][S][n_samples] out:
 *   Y = (M / gain) X / |X| (0 where X = 0), y_t = real inverse DFT / win, and the weighted overlap-add
 *   y[n] = sum_t w[n - t hop] y_t[n - t hop] / sum_t w[n - t hop]^2 (0 where no frame covers n).
 *   With M = V of nfhmm_stft, y = x wherever the windows cover x.
 * Errors: NFHMM_EINVAL (sizes, NULL, gain <= 0, win not a power of two), NFHMM_ECUDA. */
int nfhmm_stft(const float *x, int64_t n_sig, int64_t n_samples, int32_t win, int32_t hop, float gain, float *X, float *V,
               int32_t device, void *stream);
int nfhmm_istft(const float *X, const float *M, int64_t n_mix, int32_t S, int64_t T, int32_t win, int32_t hop,
                float gain, float *y, int64_t n_samples, int32_t device, void *stream);

/* ---------------------------------------------------------------------------------------------------
 * N-HMM maximum-likelihood EM training: learns each source's dictionaries,
 * transition matrix and initial distribution from an isolated-source spectrogram, the step before the
 * separation path.  The paper gives only "maximum-likelihood (ML) values of all these parameters may be
 * found by the EM algorithm" for the model of P:76-83; the iteration follows SPEC's em_step
 * (S:179-181): E-step lhat_{t,d}(l) = sum_z theta_t(d)_z beta_l(d,z), log-likelihood of frame t in state d
 * sum_l V_lt log lhat, forward-backward -> gamma, xi; M-step theta_t(d)_z ∝ sum_l V_lt P(z|l,t,d),
 * beta_l(d,z) ∝ sum_t gamma_t(d) V_lt P(z|l,t,d), rho ∝ sum_t xi_t, pi = gamma_0.  n_src independent sources
 * are trained in the same launches.
 * Layouts (FP32, row-major; any argument may be a host or a device pointer, as above):
 *   V       [n_src][T][F]      counts >= 0, finite
 *   dict    [n_src][N][K][F]   beta_l(d, z) = dict[s][d][z][l], each element sums to 1 over l
 *   trans   [n_src][N][N]      row-stochastic, trans[s][i][j] = P(D_t = j | D_{t-1} = i) (DESIGN R4)
 *   prior   [n_src][N]
 *   weights [n_src][T][N][K]   theta_t(d), each (t, d) row sums to 1 (NULL at set_params: uniform 1/K)
 *   loglik  [n_src][max_iters] FP64 log evidence (multinomial coefficient omitted) of the parameters
 *                              iteration i started from; non-decreasing in i
 * Limits: 1 <= N <= 128, 1 <= K <= 32, K*F <= 51200.  The handle allocates its own device memory.
 * Errors: NFHMM_EINVAL (dimensions, NULL, negative / non-finite data, n_iters beyond max_iters),
 * NFHMM_ESTATE (em before set_data + set_params), NFHMM_EZEROSUPPORT (a frame no state can explain),
 * NFHMM_ENUMERIC, NFHMM_ECUDA, NFHMM_ENOMEM; detail in nhmm_train_last_error(). */
typedef struct nhmm_train nhmm_train_t;   /* opaque, library-owned */

int nhmm_train_create(int64_t F, int64_t T, int32_t N, int32_t K, int64_t n_src, int32_t max_iters, int32_t device,
                      void *stream /* cudaStream_t or NULL */, nhmm_train_t **out);
/* Copy and validate the training spectrograms.  Synchronises. */
int nhmm_train_set_data(nhmm_train_t *h, const float *V);
/* Initial parameters (the paper does not state an initialisation; S:168 draws Dirichlet dictionaries,
 * a near-uniform chain and uniform pi).  Resets the iteration count.  Synchronises. */
int nhmm_train_set_params(nhmm_train_t *h, const float *dict, const float *trans, const float *prior,
                          const float *weights);
/* n_iters EM iterations; synchronises and returns the sticky device status. */
int nhmm_train_em(nhmm_train_t *h, int32_t n_iters);
/* Copy out the current parameters and the log-evidence trace (any output may be NULL).  Synchronises. */
int nhmm_train_get(nhmm_train_t *h, float *dict, float *trans, float *prior, float *weights, double *loglik,
                   int32_t *iters_done);
/* Kernel launches enqueued by this handle (instrumentation). */
int nhmm_train_kernel_launches(const nhmm_train_t *h, int64_t *n);
int nhmm_train_destroy(nhmm_train_t *h);
const char *nhmm_train_last_error(const nhmm_train_t *h);

#ifdef __cplusplus
}
#endif

#endif /* NFHMM_H */
