// nfhmm_internal.cuh -- shared declarations of libnfhmm's device kernels and host runtime.
// Product path: no code here is shared with oracle/ (task rule: the two share nothing).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/nfhmm.h"

namespace nfk {

// Device error flags (sticky, OR-ed by kernels, read once per sync).
enum : unsigned { FLAG_ZERO_SUPPORT = 1u, FLAG_NONFINITE = 2u, FLAG_BAD_INPUT = 4u };

// Reconstruction-GEMM modes (kernel (a) and the Section 4 reconstruction of kernel (f)).
enum ReconMode : int {
    RECON_RATIO = 0,     // R = V / V_hat, sum V log V_hat partials, optional V_hat store   (Eq. 7)
    RECON_STORE = 1,     // store V_hat only (posteriors)
    RECON_SEPARATE = 2,  // V_src^(s) = (v_t / alpha_0) * sum_{k in s} beta alpha
};

struct ReconArgs {
    int M;                    // rows (frames) of the GEMM
    int k_begin, k_end;       // contraction range over global elements k
    const float *A;           // [M][lda] theta (RATIO/STORE) or alpha (SEPARATE)
    int lda;
    const float *B;           // betaT [Kpad][ldb]
    int ldb;
    int F;                    // true number of bins
    const float *V;           // [M][ldv] counts (padded with zeros to ldv)
    int ldv;
    float *R;                 // [M][ldv] ratio out (RATIO)
    float *Vhat;              // optional [..][F] V_hat out (RATIO/STORE), row-major ld = F
    double *data_part;        // [M][n_tiles] sum_l V log V_hat per (row, column tile) (RATIO), integer-valued
                              // FP64 in units of 2^-20 nats (exact, tiling-independent sums)
    int n_tiles;
    const float *row_scale;   // SEPARATE: per-row v_t / alpha_0
    float *out_src;           // SEPARATE: V_src base for this source
    int T, S, s;              // SEPARATE: address ((m*S + s)*T + t)*F + l
    unsigned *flags;
    const float *Bsplit;      // tensor-core path: pre-split, pre-tiled beta (tc_presplit_host / tc_presplit16_host)
    int nkb_total;
    const float *colscale;    // non-NULL: FP16-split products (Bsplit from tc_presplit16_host, its column scales);
                              // RATIO / STORE with A = theta~ only; RATIO then writes R' = c_l R (c_l = 2^30 colscale_l)
    unsigned *rowmax;         // H16 RATIO: per-row largest R' (float bits, atomicMax; zeroed by the caller)
    int max_ctas;             // tensor-core path: cap on the persistent grid (0 = one CTA per SM)
};

struct BackprojArgs {
    int M;
    int Kpad;                 // contraction length (padded bins, multiple of 8)
    const float *A;           // R [M][lda]
    int lda;
    const float *B;           // beta [Kpad][ldb]
    int ldb;
    const float *theta;       // [M][ldb]
    float *n_out;             // [M][ldb]  n = theta .* (R beta)   (data term of Eq. 6)
    const float *Bsplit;      // tensor-core path: pre-split, pre-tiled betaT
    int nkb_total;
    int max_ctas;             // tensor-core path: cap on the persistent grid (0 = one CTA per SM)
    const float *colscale;    // non-NULL: 3xFP16 products (Bsplit from tc_presplit16_host of beta^T / c_l); A = R'
    const unsigned *rowmax;   // with colscale: per-row largest R' (from the H16 reconstruction)
};

// Launchers (return cudaError_t of the launch).
cudaError_t launch_recon(int bn, const ReconArgs &a, cudaStream_t st);
cudaError_t launch_backproj(int bn, const BackprojArgs &a, cudaStream_t st);

// tcgen05 3xTF32 variants (gemm_tc.cu).  recon: a.B = beta [F_pad][Kt_pad] K-major (ldb = Kt_pad);
// backproj: a.B = betaT [Kt_pad][F_pad] K-major, a.Kpad = F_pad, a.ldb = row length of theta / n.
// tile width (a multiple of mult, itself a multiple of 16) for n output columns and `rows` output rows
// (rows = 0: ignore the row count) on `sms` SMs
int tc_pick_bn(int64_t n, int mult = 16, int64_t rows = 0, int sms = 148);
// The static operand B[n][k] (n < n_rows, k < k_len; src[n*ld + k], or src[k*ld + n] if transposed) split
// into tf32 hi/lo and re-tiled into the shared-memory image of each pipeline stage (host side, once).
size_t tc_presplit_floats(int64_t n_rows, int64_t k_len, int bn);
void tc_presplit_host(const float *src, int64_t ld_src, bool transposed, int64_t n_rows, int64_t k_len, int bn,
                      float *dst, int64_t k_pad = 0, const float *kscale = nullptr);
// FP16 image for the 3xFP16 reconstruction (rows scaled by powers of two; colscale[nt_n * bn] undoes them)
size_t tc_presplit16_floats(int64_t n_rows, int64_t k_len, int bn);
// kscale (optional): element (n, k) is multiplied by kscale[k] first (the back-projection's 1 / c_l)
void tc_presplit16_host(const float *src, int64_t ld_src, bool transposed, int64_t n_rows, int64_t k_len, int bn,
                        float *dst, float *colscale, int64_t k_pad = 0, const float *kscale = nullptr);
cudaError_t launch_recon_tc(int bn, const ReconArgs &a, cudaStream_t st);
cudaError_t launch_backproj_tc(int bn, int n_valid, const BackprojArgs &a, cudaStream_t st);
// Split-K reconstruction for few row tiles (single mixtures): tc_split_count(k) units of one TMEM accumulation chunk per
// (row tile, column tile); raw sums in part [splits][M][n_tiles * bn], then a fixed-order reduction with the
// RATIO / BACKPROJ epilogue (results bitwise equal to the unsplit kernel; the RATIO data term goes to
// data_part[row][ceil(ldv / 16)] -- 16-column sub-tiles -- in the same fixed point)
int tc_split_count(int64_t k_len);
int tc_pick_bn_split(int64_t n, int64_t rows, int splits, int sms = 148);
cudaError_t launch_recon_tc_split(int bn, const ReconArgs &a, float *part, cudaStream_t st);

// Back-projection with the Dirichlet element step fused into its epilogue (bn % K == 0, K <= 32):
// theta is updated in place; Eq. 8 block sums and g~ partials leave block-major ([block][ldf]).
struct FusedDirichletArgs {
    int K, Kt, SN, ldf;       // ldf: frame pitch of the block-major arrays (a multiple of 4)
    const float *dvT;         // [SN][ldf]   gamma d + 1 (dv_kernel)
    const double *fconst;     // [frames][4] (DirichletArgs)
    double *spsT, *sps2T;     // [SN][ldf]   psi block sums (first / second parts)
    double *hpartT;           // [n_tiles][ldf] g~ partial sums per column tile (NULL: no bound)
    float *alpha_out;         // [frames][ldb] alpha, or NULL (not the last sweep)
};
cudaError_t launch_backproj_dirichlet_tc(int bn, int n_valid, const BackprojArgs &a, const FusedDirichletArgs &d,
                                         cudaStream_t st);

struct DirichletArgs {
    int frames, T, S, N, K, Kt, ld;   // ld = padded row length of n/alpha/theta
    float gamma;
    const float *n_in;        // [frames][ld]  data term of Eq. 6 (sum_l V z)
    float *alpha;             // [frames][ld]  out: alpha (may alias n_in)
    float *theta;             // [frames][ld]  out: exp(psi(alpha) - psi(alpha_0))
    const float *u_fwd;       // [M][S][T][N]  previous sweep's FB messages: q(D) marginals are
    const float *b_bwd;       // [M][S][T][N]  d = u .* b / sum_n(u .* b)
    const double *fconst;     // [frames][4]   alpha_0, psi(alpha_0), -alpha_0 - lnG(alpha_0) + (alpha_0 - Kt) psi(alpha_0),
                              //               e^{-psi(alpha_0)}
    int write_alpha;          // 1: store alpha (last sweep of a call); 0: only theta / e (alpha is not read in the loop)
    float *ec;                // [M][S][T][N]  out: emission exp(gamma*(phi - max_n phi)) in (0, 1]
    double *eoff;             // [M][S][T]     out: gamma * max_n phi (FP64)
    double *hdir;             // [frames]      out: Dirichlet entropy terms of the bound (or NULL)
    int ldf;                  // fused path: frame pitch of the block-major arrays
    int variant;              // 0: ring kernel (dirichlet_ring.cu) where supported, else the per-warp pipelined
                              // kernel; 1: frame-tile kernel (NFHMM_DIRICHLET=tile); 2: per-warp kernel (=pipe)
    unsigned *flags;
};
cudaError_t launch_dirichlet(const DirichletArgs &a, cudaStream_t st);
// Round-2 default (dirichlet_ring.cu): persistent frame tiles with a two-stage bulk-copy ring
bool dirichlet_ring_supported(const DirichletArgs &a);
cudaError_t launch_dirichlet_ring(const DirichletArgs &a, cudaStream_t st);
// Fused path: pseudo-counts before the back-projection GEMM, Eq. 8 / bound terms after it (dirichlet.cu)
cudaError_t launch_dv(const DirichletArgs &a, float *dvT, cudaStream_t st);
cudaError_t launch_eq8(const DirichletArgs &a, const double *spsT, const double *sps2T, const double *hpartT,
                       int n_tiles, int bn, cudaStream_t st);

struct FBArgs {
    int M, S, T, N;
    const float *ec;          // [M][S][T][N]  emissions exp(gamma*(phi - max_n phi))
    const double *eoff;       // [M][S][T]
    const float *trans;       // [S][N][N]
    const float *prior;       // [S][N]
    float *fwd;               // [M][S][T][N] out: scaled forward messages u_t
    float *bwd;               // [M][S][T][N] out: scaled backward messages b_t (d_t = u_t .* b_t / sum)
    double *logZ;             // [M][S] out
    unsigned *flags;
    int wide;                 // multi-warp kernel per chain and direction: 1 for N > 64 (default), 2 also for
                              // 32 < N <= 64 (few chains), 0 never
    int multi;                // 2: 16 chains of one source per warp on the tensor cores (fb_mma_kernel),
                              // 1: several chains per warp with FFMA2 (fb_multi_kernel), 0: one chain per warp
    // parallel-in-time path (fbp_*): nchunk chunks of chunk_len steps; exact chunk-start messages
    int nchunk, chunk_len;    // nchunk <= 1: one sequential pass over [0, T)
    float *fstart;            // [M*S][nchunk][NMAX]  u_{t0} of each chunk (scratch)
    float *bstart;            // [M*S][nchunk][NMAX]  b_{t1-1} of each chunk (scratch)
    float *P, *PT;            // [M*S][nchunk][NMAX][NMAX] chunk transfer matrices and transposes (scratch)
    int *PE;                  // [M*S][nchunk][NMAX] per-row power-of-two exponents of P
};
// Chunking of the parallel-in-time FB for a handle (0 = sequential): used when few chains would leave
// the GPU idle during the 2T dependent steps.
int fb_pick_chunks(int64_t chains, int64_t T, int N, int *chunk_len);
// multi-chain kernel (fb_multi_kernel) for this shape: N = 32 Q + R with R | 32 among the compiled ones
bool fb_multi_supported(int N, int64_t M, int nchunk);
// tensor-core kernel (fb_mma_kernel, 16 chains per warp, mma.sync 3xTF32) for this shape: N = 8 NT
bool fb_mma_supported(int N, int64_t M, int nchunk);
cudaError_t launch_fb(const FBArgs &a, cudaStream_t st);

struct ElboArgs {
    int M, T, n_tiles, S, max_iters;
    int *iter_ctr;            // device sweep counter (row of fe to write; advanced by the kernel)
    unsigned *done_ctr;       // device: blocks finished (last-block pattern)
    double c_prior_T;         // T * (lnGamma(Kt + gamma S K) - S K lnGamma(1 + gamma))
    const double *data_part;  // [M*T][n_tiles]
    const double *hdir;       // [M*T]
    const double *logZ;       // [M][S]
    double *fe;               // [M][max_iters]
    double *part;             // [M][ELBO_MAX_BLOCKS] per-block partial sums
    unsigned *mix_ctr;        // [M] blocks of each mixture finished (zero between launches)
};
constexpr int ELBO_MAX_BLOCKS = 16;   // blocks per mixture (frames split so a single mixture fills several SMs)
cudaError_t launch_elbo(const ElboArgs &a, cudaStream_t st);

// Initial state (DESIGN R5): alpha = 1 + gamma/N, theta = exp(psi(a) - psi(Kt a)), d = 1/N.
cudaError_t launch_init_state(int frames, int ld, int Kt, double alpha0, float *alpha, float *theta, float *u_fwd,
                              float *b_bwd, long long d_count, cudaStream_t st);
// d[r][:] = u[r][:] .* b[r][:] / sum(u[r][:] .* b[r][:]) over rows of N (q(D) marginals from the FB messages)
cudaError_t launch_marginals(const float *u, const float *b, float *d, long long rows, int N, cudaStream_t st);
// betaT [rows][ldT] -> beta [ldT][ldb] transpose (rows = Kt, cols = F)
cudaError_t launch_transpose(const float *src, int rows, int cols, int ld_src, float *dst, int ld_dst,
                             cudaStream_t st);
// Observation checks + per-frame row sums v_t (FP32 exact for integer counts; FP64 accumulate).
cudaError_t launch_obs_stats(const float *V, int frames, int F, int ld, float *vt, unsigned *flags,
                             cudaStream_t st);
// Per-frame constants of the Dirichlet step (DESIGN R19: alpha_0 = v_t + Kt + gamma S K is the same in
// every sweep): fc[4f] = alpha_0, fc[4f+1] = psi(alpha_0), fc[4f+2] = -alpha_0 - lnG(alpha_0) + (alpha_0 - Kt)
// psi(alpha_0), fc[4f+3] = e^{-psi(alpha_0)} (FP64).
cudaError_t launch_frame_consts(const float *vt, int frames, int Kt, double gamma, int S, int K, double *fc,
                                cudaStream_t st);
// Per-row scale v_t / alpha_0 for separation.
cudaError_t launch_sep_scale(const float *alpha, int frames, int Kt, int ld, const float *vt, float *scale,
                             cudaStream_t st);
// V*^(s) = V V_src^(s) / sum_s' V_src^(s'), V_src layout [M][S][T][F]; writes V_star.
cudaError_t launch_wiener(const float *V, int ldv, const float *vsrc, float *vstar, int M, int S, int T,
                          int F, cudaStream_t st);

// Per-device launch state (the kernel attributes and SM counts are properties of a device, so a process
// with handles on several devices must not share one cache): raise `func`'s dynamic shared-memory limit
// to `bytes` on the current device (once per (kernel, device)); SM count and occupancy of the current
// device (cached per (kernel, device, block size, smem)).
cudaError_t ensure_dyn_smem(const void *func, size_t bytes);
int device_sms();
int occupancy_ctas(const void *func, int threads, size_t smem);

}  // namespace nfk
