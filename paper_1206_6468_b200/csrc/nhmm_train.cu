// nhmm_train.cu -- maximum-likelihood EM training of single-source N-HMMs on the GPU (SURVEY §8(f)
// NEXT-3: "learn beta, rho, pi from isolated sources ... reuses K-a/K-b/K-e plus pairwise posteriors and
// an M-step").  The paper states only that "maximum-likelihood (ML) values of all these parameters may
// be found by the EM algorithm" (model P:76-83); the steps follow SPEC's em_step:
//   E-step  lhat_{t,d}(l) = sum_z theta_t(d)_z beta_l(d,z);  loglik_{t,d} = sum_l V_lt log lhat_{t,d}(l);
//           scaled forward-backward over each source's chain (the VB path's fb kernels, S = n_src)
//           -> gamma_t(d), xi_t(i,j), log evidence;
//   M-step  theta_t(d)_z ∝ theta_t(d)_z C_{t,d,z},  C_{t,d,z} = sum_l beta_l(d,z) V_lt / lhat_{t,d}(l);
//           beta_l(d,z)  ∝ beta_l(d,z) sum_t gamma_t(d) theta_t(d)_z V_lt / lhat_{t,d}(l);
//           rho(i -> j)  ∝ sum_{t>=1} xi_t(i,j),  xi_t(i,j) = u_{t-1}(i) A_ij e_t(j) b_t(j) / Z_t;  pi = gamma_0;
//           beta and rho floored at 1e-12 and renormalised (SPEC's decision S:214), pi likewise (DESIGN R21).
// The posterior weights span hundreds of orders of magnitude (at 1e4-1e5 counts per frame the per-state
// log-likelihoods of a frame differ by thousands of nats): a state the posterior barely visits has
// gamma_t(d) ~ 1e-289, and its ML dictionary update is a ratio of such weights.  Everything that carries
// posterior weight therefore runs in FP64 -- the emissions e, the chain recursion (train_fb_kernel), gamma,
// xi and the beta sums -- so the GPU reaches the same plain ML update as the FP64 oracle (round 1 ran the
// FP32 VB recursion here and had to skip the updates of such states).
// Kernels, per EM iteration (n_src independent sources batched in every launch):
//   estep_kernel<KM>     CTA per (source, state d, tile of frames): beta(d) [K][F] staged in shared memory,
//                        a warp per frame, lanes over l; loglik in FP64 (per-bin terms v log lhat are
//                        ~1e3 and the frame totals ~1e5: FP32 sums would move e = exp(loglik - max) by
//                        ~1e-3), C_{t,d,:} by warp reductions;
//   emission_kernel      e_t(d) = exp(loglik - max_d loglik) (FP64), eoff_t = max;
//   train_fb_kernel      FP64 scaled forward-backward per source (forward and backward warps concurrently),
//                        log evidence;
//   posterior_kernel     gamma_t = u_t .* b_t / sum and the pairwise normaliser Z_t = u_{t-1} A (e_t .* b_t);
//   xi_kernel            sum_{t>=1} xi_t(i,j), thread per (i, j), FP64 accumulation over t;
//   beta_kernel<KM>      thread per (source, d, l): beta_l(d,:) in registers, FP64 accumulation over t;
//   beta_norm_kernel / mstep_kernel  normalisations, floors, theta, rho, pi.
// The messages are normalised per step (forward by its sum, whose logs give the evidence; backward by its
// sum); every consumer normalises per frame, so the scales cancel.
#include <cuda_runtime.h>
#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <new>
#include <string>

#include "nfhmm_internal.cuh"
#include "../../include/nfhmm.h"

namespace nfk {
namespace {

constexpr int ES_FT = 16;     // frames per estep CTA (8 warps x 2)
constexpr int BK_THREADS = 128;

template <int KM>
__global__ void __launch_bounds__(256) estep_kernel(int F, int T, int N, int K, const float *V, const float *beta,
                                                    const float *theta, double *LL, float *C) {
    extern __shared__ __align__(16) float bs[];   // beta(m, d) [K][F]
    const int m = blockIdx.z, d = blockIdx.y, t0 = blockIdx.x * ES_FT;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const float *bg = beta + ((size_t)m * N + d) * K * F;
    for (int i = threadIdx.x; i < K * F; i += blockDim.x) bs[i] = bg[i];
    __syncthreads();
    for (int t = t0 + warp; t < min(T, t0 + ES_FT); t += 8) {
        const float *th = theta + (((size_t)m * T + t) * N + d) * K;
        double tz[KM];
        float cz[KM];
#pragma unroll
        for (int z = 0; z < KM; ++z) {
            tz[z] = z < K ? (double)th[z] : 0.0;
            cz[z] = 0.f;
        }
        const float *vr = V + ((size_t)m * T + t) * F;
        double ll = 0.0;
        bool zero = false;
        // branch-free body, unrolled: the bins' independent FP64 chains (lhat, log) interleave
#pragma unroll 2
        for (int l = lane; l < F; l += 32) {
            const float v = vr[l];
            // lhat in FP64: an FP32 sum (~3e-7 relative) times counts of 1e2-1e3 per bin would move
            // loglik by ~1e-3 and the emission ratios of the non-dominant states by as much
            double lh = 0.0;
#pragma unroll
            for (int z = 0; z < KM; ++z)
                if (z < K) lh = fma(tz[z], (double)bs[z * F + l], lh);
            const bool use = v > 0.f && lh > 0.0;
            zero |= v > 0.f && !(lh > 0.0);
            const double lg = log(use ? lh : 1.0);
            ll = fma((double)(use ? v : 0.f), lg, ll);
            const float r = use ? __fdiv_rn(v, (float)lh) : 0.f;   // a weight: FP32 suffices
#pragma unroll
            for (int z = 0; z < KM; ++z)
                if (z < K) cz[z] = fmaf(bs[z * F + l], r, cz[z]);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) ll += __shfl_xor_sync(0xffffffffu, ll, o);
        zero = __any_sync(0xffffffffu, zero);
#pragma unroll
        for (int z = 0; z < KM; ++z)
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) cz[z] += __shfl_xor_sync(0xffffffffu, cz[z], o);
        if (lane == 0) LL[((size_t)m * T + t) * N + d] = zero ? -INFINITY : ll;
        float *cd = C + (((size_t)m * T + t) * N + d) * K;
        if (lane < K) {
            float c = cz[0];
#pragma unroll
            for (int z = 1; z < KM; ++z)
                if (z == lane) c = cz[z];
            cd[lane] = c;
        }
    }
}

// one warp per (source, frame): e = exp(loglik - max_d), eoff = max_d (FP64)
__global__ void emission_kernel(int T, int N, int MT, const double *LL, double *ec, double *eoff, unsigned *flags) {
    const int w = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
    if (w >= MT) return;
    const double *l = LL + (size_t)w * N;
    double mx = -INFINITY;
    for (int d = lane; d < N; d += 32) mx = fmax(mx, l[d]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if (!(mx > -INFINITY)) {
        if (lane == 0) atomicOr(flags, FLAG_ZERO_SUPPORT);
        mx = 0.0;
    }
    for (int d = lane; d < N; d += 32) ec[(size_t)w * N + d] = exp(l[d] - mx);
    if (lane == 0) eoff[w] = mx;
}

// FP64 scaled forward-backward, one warp per (source, direction), lanes over states, A in shared memory:
//   u_0 = pi .* e_0 / c_0,  u_t = (u_{t-1} A) .* e_t / c_t  (c_t = the sum; log Z = sum_t ln c_t + eoff_t);
//   b_{T-1} = 1,  b_t = A (e_{t+1} .* b_{t+1}) / (its sum).
__global__ void __launch_bounds__(64) train_fb_kernel(int T, int N, const double *ec, const double *eoff,
                                                      const float *A, const float *prior, double *fw, double *bw,
                                                      double *logZ, unsigned *flags) {
    extern __shared__ __align__(16) double tsm[];
    double *As = tsm;                 // [N][N]
    const int m = blockIdx.x, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    double *xb = tsm + (size_t)N * N + warp * 2 * N;   // [2][N] broadcast buffers of this warp
    const float *Ag = A + (size_t)m * N * N;
    for (int i = threadIdx.x; i < N * N; i += blockDim.x) As[i] = (double)Ag[i];
    __syncthreads();
    const double *e = ec + (size_t)m * T * N;
    unsigned bad = 0;
    auto wsum = [&](double v) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        return v;
    };
    if (warp == 0) {   // forward
        double *f = fw + (size_t)m * T * N;
        double lz = 0.0, part = 0.0;
        for (int j = lane; j < N; j += 32) {
            const double v = (double)prior[(size_t)m * N + j] * e[j];
            xb[j] = v;
            part += v;
        }
        double c = wsum(part);
        if (!(c > 0.0)) bad |= FLAG_NONFINITE;
        double ic = 1.0 / c;
        __syncwarp();
        for (int j = lane; j < N; j += 32) {
            xb[j] *= ic;
            f[j] = xb[j];
        }
        lz += log(c) + eoff[(size_t)m * T];
        __syncwarp();
        for (int t = 1; t < T; ++t) {
            const double *prev = xb + ((t - 1) & 1) * N;
            double *cur = xb + (t & 1) * N;
            part = 0.0;
            for (int j = lane; j < N; j += 32) {
                double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;   // four chains: latency
                int i = 0;
                for (; i + 3 < N; i += 4) {
                    a0 = fma(prev[i], As[i * N + j], a0);
                    a1 = fma(prev[i + 1], As[(i + 1) * N + j], a1);
                    a2 = fma(prev[i + 2], As[(i + 2) * N + j], a2);
                    a3 = fma(prev[i + 3], As[(i + 3) * N + j], a3);
                }
                for (; i < N; ++i) a0 = fma(prev[i], As[i * N + j], a0);
                const double v = ((a0 + a1) + (a2 + a3)) * e[(size_t)t * N + j];
                cur[j] = v;
                part += v;
            }
            c = wsum(part);
            if (!(c > 0.0)) bad |= FLAG_NONFINITE;
            ic = 1.0 / c;
            __syncwarp();
            for (int j = lane; j < N; j += 32) {
                cur[j] *= ic;
                f[(size_t)t * N + j] = cur[j];
            }
            lz += log(c) + eoff[(size_t)m * T + t];
            __syncwarp();
        }
        if (lane == 0) {
            logZ[m] = lz;
            if (!isfinite(lz)) bad |= FLAG_NONFINITE;
        }
    } else {           // backward
        double *b = bw + (size_t)m * T * N;
        for (int j = lane; j < N; j += 32) {
            b[(size_t)(T - 1) * N + j] = 1.0;
            xb[((T - 1) & 1) * N + j] = e[(size_t)(T - 1) * N + j];   // x_{T-1} = e_{T-1} .* b_{T-1}
        }
        __syncwarp();
        for (int t = T - 2; t >= 0; --t) {
            const double *x = xb + ((t + 1) & 1) * N;
            double *cur = xb + (t & 1) * N;
            double part = 0.0;
            double bv[4];
            int q = 0;
            for (int i = lane; i < N; i += 32, ++q) {
                double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
                int j = 0;
                for (; j + 3 < N; j += 4) {
                    a0 = fma(As[i * N + j], x[j], a0);
                    a1 = fma(As[i * N + j + 1], x[j + 1], a1);
                    a2 = fma(As[i * N + j + 2], x[j + 2], a2);
                    a3 = fma(As[i * N + j + 3], x[j + 3], a3);
                }
                for (; j < N; ++j) a0 = fma(As[i * N + j], x[j], a0);
                bv[q] = (a0 + a1) + (a2 + a3);
                part += bv[q];
            }
            const double sum = wsum(part);
            if (!(sum > 0.0)) bad |= FLAG_NONFINITE;
            const double is = 1.0 / sum;
            __syncwarp();
            q = 0;
            for (int i = lane; i < N; i += 32, ++q) {
                const double v = bv[q] * is;
                b[(size_t)t * N + i] = v;
                cur[i] = v * e[(size_t)t * N + i];
            }
            __syncwarp();
        }
    }
    if (bad) atomicOr(flags, bad);
}

// one warp per (source, frame): gamma_t = u .* b / sum; for t >= 1, 1 / Z_t with
// Z_t = sum_i u_{t-1}(i) sum_j A_ij e_t(j) b_t(j) (the pairwise normaliser; reciprocal once per frame)
__global__ void posterior_kernel(int T, int N, int MT, const double *u, const double *b, const double *ec,
                                 const float *A, double *gamma, double *Zt) {
    const int w = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
    if (w >= MT) return;
    const int m = w / T, t = w - m * T;
    const size_t row = (size_t)w * N;
    double s = 0.0;
    for (int d = lane; d < N; d += 32) s += u[row + d] * b[row + d];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    const double is = 1.0 / s;
    for (int d = lane; d < N; d += 32) gamma[row + d] = u[row + d] * b[row + d] * is;
    if (t == 0) {
        if (lane == 0) Zt[w] = 0.0;
        return;
    }
    const float *Am = A + (size_t)m * N * N;
    double z = 0.0;
    for (int i = lane; i < N; i += 32) {
        double y = 0.0;
        for (int j = 0; j < N; ++j) y = fma((double)Am[i * N + j], ec[row + j] * b[row + j], y);
        z += u[row - N + i] * y;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) z += __shfl_xor_sync(0xffffffffu, z, o);
    if (lane == 0) Zt[w] = 1.0 / z;
}

// thread per (source, i, j) and chunk of frames: partial xi sums A_ij sum_{t in chunk, t>=1}
// u_{t-1}(i) e_t(j) b_t(j) / Z_t (FP64); mstep_kernel adds the chunks in a fixed order
__global__ void xi_kernel(int T, int N, int M, int tchunk, const double *u, const double *b, const double *ec,
                          const double *invZ, const float *A, double *xi_part) {
    const int idx = blockIdx.x * blockDim.x + threadIdx.x, c = blockIdx.y;
    if (idx >= M * N * N) return;
    const int m = idx / (N * N), ij = idx - m * N * N, i = ij / N, j = ij - i * N;
    const size_t base = (size_t)m * T * N;
    double acc = 0.0;
    for (int t = max(1, c * tchunk); t < min(T, (c + 1) * tchunk); ++t)
        acc += u[base + (size_t)(t - 1) * N + i] * (ec[base + (size_t)t * N + j] * b[base + (size_t)t * N + j]) *
               invZ[(size_t)m * T + t];
    xi_part[(size_t)c * M * N * N + idx] = acc * (double)A[(size_t)m * N * N + ij];
}

// thread per (source, d, l) and chunk of frames: partial nb_l(d, z) = beta_l(d,z) sum_{t in chunk}
// gamma_t(d) theta_t(d)_z V_lt / lhat_{t,d}(l) in FP64 (gamma may be ~1e-289); beta_norm_kernel adds the chunks
template <int KM>
__global__ void __launch_bounds__(BK_THREADS) beta_kernel(int F, int T, int N, int K, int tchunk, const float *V,
                                                          const float *beta, const float *theta, const double *gamma,
                                                          double *nb_part) {
    const int M = gridDim.z / ((T + tchunk - 1) / tchunk);
    const int c = blockIdx.z / M, m = blockIdx.z - c * M, d = blockIdx.y, l = blockIdx.x * BK_THREADS + threadIdx.x;
    const bool lv = l < F;
    const float *bg = beta + ((size_t)m * N + d) * K * F;
    float bz[KM];
    double acc[KM];
#pragma unroll
    for (int z = 0; z < KM; ++z) {
        bz[z] = (lv && z < K) ? bg[z * F + l] : 0.f;
        acc[z] = 0.0;
    }
    const int t1 = min(T, (c + 1) * tchunk);
    // branch-free body (a zero weight where V = 0 or lhat = 0) so the loads of the next frames issue
    // ahead of the arithmetic (the loop is bound by their latency)
#pragma unroll 4
    for (int t = c * tchunk; t < t1; ++t) {
        const float v = lv ? V[((size_t)m * T + t) * F + l] : 0.f;
        const float *th = theta + (((size_t)m * T + t) * N + d) * K;
        const double gm = gamma[((size_t)m * T + t) * N + d];
        float tz[KM];
        float lh = 0.f;   // V / lhat needs FP32 only (the log-likelihood's lhat is FP64, estep_kernel)
#pragma unroll
        for (int z = 0; z < KM; ++z) {
            tz[z] = z < K ? th[z] : 0.f;
            lh = fmaf(tz[z], bz[z], lh);
        }
        const double g = (v > 0.f && lh > 0.f) ? gm * (double)__fdiv_rn(v, lh) : 0.0;
#pragma unroll
        for (int z = 0; z < KM; ++z)
            if (z < K) acc[z] = fma(g, (double)tz[z], acc[z]);
    }
    if (lv) {
        double *dst = nb_part + (size_t)c * gridDim.y * M * K * F;   // [chunk][M][N][K][F]
#pragma unroll
        for (int z = 0; z < KM; ++z)
            if (z < K) dst[(((size_t)m * N + d) * K + z) * F + l] = acc[z] * (double)bz[z];
    }
}

// warp per (source, d, z): nb = sum over frame chunks of the partials (fixed order), beta <- nb / sum_l nb
// (kept when the element got no weight at all: 0/0), then the 1e-12 floor and renormalisation
__global__ void beta_norm_kernel(int F, int T, int N, int K, int rows, int nchunk, const double *nb_part,
                                 float *beta) {
    const int w = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
    if (w >= rows) return;
    const size_t stride = (size_t)rows * F;
    double s = 0.0;
    for (int l = lane; l < F; l += 32) {
        double v = 0.0;
        for (int c = 0; c < nchunk; ++c) v += nb_part[c * stride + (size_t)w * F + l];
        s += v;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    float *bt = beta + (size_t)w * F;
    double s2 = 0.0;   // sum of the floored values
    for (int l = lane; l < F; l += 32) {
        double v;
        if (s > 0.0) {
            v = 0.0;
            for (int c = 0; c < nchunk; ++c) v += nb_part[c * stride + (size_t)w * F + l];
            v /= s;
        } else {
            v = (double)bt[l];
        }
        s2 += fmax(v, 1e-12);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s2 += __shfl_xor_sync(0xffffffffu, s2, o);
    for (int l = lane; l < F; l += 32) {
        double v;
        if (s > 0.0) {
            v = 0.0;
            for (int c = 0; c < nchunk; ++c) v += nb_part[c * stride + (size_t)w * F + l];
            v /= s;
        } else {
            v = (double)bt[l];
        }
        bt[l] = (float)(fmax(v, 1e-12) / s2);
    }
}

// theta_t(d) <- theta .* C / sum (thread per (source, t, d)); rho rows from xi, pi = gamma_0 (threads of
// the first blocks)
__global__ void mstep_kernel(int T, int N, int K, int M, int nchunk, float *theta, const float *C, const double *xi_part,
                             float *A, float *prior, const double *gamma) {
    const int idx = blockIdx.x * blockDim.x + threadIdx.x;
    if (idx < M * T * N) {
        float *th = theta + (size_t)idx * K;
        const float *c = C + (size_t)idx * K;
        double s = 0.0;
        for (int z = 0; z < K; ++z) s += (double)th[z] * (double)c[z];
        if (s > 0.0)
            for (int z = 0; z < K; ++z) th[z] = (float)((double)th[z] * (double)c[z] / s);
    }
    if (idx < M * N) {   // rho row i of source m: ML row (kept on 0/0), 1e-12 floor, renormalised
        const int m = idx / N, i = idx - m * N;
        const size_t row = (size_t)m * N * N + (size_t)i * N, cs = (size_t)M * N * N;
        float *a = A + row;
        double s = 0.0;
        for (int j = 0; j < N; ++j)
            for (int c = 0; c < nchunk; ++c) s += xi_part[c * cs + row + j];
        double s2 = 0.0;
        for (int j = 0; j < N; ++j) {
            double x = (double)a[j];
            if (s > 0.0) {
                x = 0.0;
                for (int c = 0; c < nchunk; ++c) x += xi_part[c * cs + row + j];
                x /= s;
            }
            s2 += fmax(x, 1e-12);
        }
        for (int j = 0; j < N; ++j) {
            double x = (double)a[j];
            if (s > 0.0) {
                x = 0.0;
                for (int c = 0; c < nchunk; ++c) x += xi_part[c * cs + row + j];
                x /= s;
            }
            a[j] = (float)(fmax(x, 1e-12) / s2);
        }
    }
    if (idx < M) {   // pi = gamma_0, floored at 1e-12 and renormalised like rho (DESIGN R21)
        const double *g = gamma + (size_t)idx * T * N;
        double s = 0.0;
        for (int d = 0; d < N; ++d) s += fmax(g[d], 1e-12);
        for (int d = 0; d < N; ++d) prior[(size_t)idx * N + d] = (float)(fmax(g[d], 1e-12) / s);
    }
}

__global__ void trace_kernel(int M, int iter, int max_iters, const double *logZ, double *trace) {
    const int m = blockIdx.x * blockDim.x + threadIdx.x;
    if (m < M) trace[(size_t)m * max_iters + iter] = logZ[m];
}

__global__ void check_data_kernel(size_t n, const float *V, unsigned *flags) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        if (!(V[i] >= 0.f) || !(V[i] < INFINITY)) atomicOr(flags, FLAG_BAD_INPUT);
}

template <int KM>
cudaError_t launch_estep(int F, int T, int N, int K, int M, const float *V, const float *beta, const float *theta,
                         double *LL, float *C, cudaStream_t st) {
    const size_t smem = (size_t)K * F * 4;
    if (smem > 220 * 1024) return cudaErrorInvalidValue;
    {
        cudaError_t e = ensure_dyn_smem((const void *)estep_kernel<KM>, smem);
        if (e != cudaSuccess) return e;
    }
    estep_kernel<KM><<<dim3((T + ES_FT - 1) / ES_FT, N, M), 256, smem, st>>>(F, T, N, K, V, beta, theta, LL, C);
    return cudaGetLastError();
}

template <int KM>
cudaError_t launch_beta(int F, int T, int N, int K, int M, int tchunk, const float *V, const float *beta,
                        const float *theta, const double *gamma, double *nb, cudaStream_t st) {
    const int nc = (T + tchunk - 1) / tchunk;
    beta_kernel<KM><<<dim3((F + BK_THREADS - 1) / BK_THREADS, N, M * nc), BK_THREADS, 0, st>>>(F, T, N, K, tchunk, V, beta,
                                                                                              theta, gamma, nb);
    return cudaGetLastError();
}

}  // namespace
}  // namespace nfk

using namespace nfk;

struct nhmm_train {
    int64_t F = 0, T = 0, M = 0;
    int N = 0, K = 0, max_iters = 0, device = 0, iters = 0;
    cudaStream_t st = nullptr;
    void *mem = nullptr;
    float *V = nullptr, *beta = nullptr, *theta = nullptr, *A = nullptr, *prior = nullptr, *C = nullptr;
    double *nb = nullptr, *ec = nullptr, *fwd = nullptr, *bwd = nullptr, *gamma = nullptr, *xi = nullptr;
    double *Zt = nullptr, *LL = nullptr, *eoff = nullptr, *logZ = nullptr, *trace = nullptr;
    unsigned *flags = nullptr;
    bool have_data = false, have_params = false;
    int64_t launches = 0;
    std::string err;
};

namespace {

int tfail(nhmm_train_t *h, int code, const char *fmt, ...) {
    if (h) {
        char buf[512];
        va_list ap;
        va_start(ap, fmt);
        vsnprintf(buf, sizeof buf, fmt, ap);
        va_end(ap);
        h->err = buf;
    }
    return code;
}

#define TCU(h, call)                                                                                 \
    do {                                                                                             \
        cudaError_t e_ = (call);                                                                     \
        if (e_ != cudaSuccess) return tfail(h, NFHMM_ECUDA, "%s: %s", #call, cudaGetErrorString(e_)); \
    } while (0)

int kmax_of(int K) { return K <= 4 ? 4 : K <= 8 ? 8 : K <= 10 ? 10 : K <= 16 ? 16 : K <= 20 ? 20 : 32; }
constexpr int TCHUNK = 256;   // frames per partial sum of the beta / xi reductions

int t_flags(nhmm_train_t *h) {
    unsigned f = 0;
    TCU(h, cudaMemcpyAsync(&f, h->flags, sizeof f, cudaMemcpyDeviceToHost, h->st));
    TCU(h, cudaStreamSynchronize(h->st));
    if (f & FLAG_BAD_INPUT) return tfail(h, NFHMM_EINVAL, "training data contain negative or non-finite values");
    if (f & FLAG_ZERO_SUPPORT) return tfail(h, NFHMM_EZEROSUPPORT, "a frame no state can explain (V > 0 where every lhat = 0)");
    if (f & FLAG_NONFINITE) return tfail(h, NFHMM_ENUMERIC, "non-finite log evidence");
    return NFHMM_OK;
}

}  // namespace

extern "C" {

int nhmm_train_create(int64_t F, int64_t T, int32_t N, int32_t K, int64_t n_src, int32_t max_iters, int32_t device,
                      void *stream, nhmm_train_t **out) {
    if (!out) return NFHMM_EINVAL;
    *out = nullptr;
    if (F < 1 || T < 1 || N < 1 || N > 128 || K < 1 || K > 32 || n_src < 1 || max_iters < 1 || (int64_t)K * F > 51200 ||
        n_src * T > (int64_t)1 << 28)
        return NFHMM_EINVAL;
    nhmm_train_t *h = new (std::nothrow) nhmm_train;
    if (!h) return NFHMM_ENOMEM;
    h->F = F;
    h->T = T;
    h->M = n_src;
    h->N = N;
    h->K = K;
    h->max_iters = max_iters;
    h->device = device;
    h->st = (cudaStream_t)stream;
    if (cudaSetDevice(device) != cudaSuccess) {
        delete h;
        return NFHMM_ECUDA;
    }
    const size_t MT = (size_t)n_src * T, MN = (size_t)n_src * N, nchunk = (size_t)((T + TCHUNK - 1) / TCHUNK);
    size_t off = 0;
    auto take = [&](size_t bytes) {
        const size_t o = off;
        off += (bytes + 255) & ~size_t(255);
        return o;
    };
    const size_t oV = take(MT * F * 4), oB = take(MN * K * F * 4), oNB = take(nchunk * MN * K * F * 8), oTh = take(MT * N * K * 4),
                 oA = take(MN * N * 4), oP = take(MN * 4), oC = take(MT * N * K * 4), oE = take(MT * N * 8),
                 oF = take(MT * N * 8), oBw = take(MT * N * 8), oG = take(MT * N * 8), oZ = take(MT * 8),
                 oX = take(nchunk * MN * N * 8), oLL = take(MT * N * 8), oEo = take(MT * 8), oLZ = take(n_src * 8),
                 oTr = take((size_t)n_src * max_iters * 8), oFl = take(256);

    if (cudaMalloc(&h->mem, off) != cudaSuccess) {
        delete h;
        return NFHMM_ENOMEM;
    }
    char *b = (char *)h->mem;
    h->V = (float *)(b + oV);
    h->beta = (float *)(b + oB);
    h->nb = (double *)(b + oNB);
    h->theta = (float *)(b + oTh);
    h->A = (float *)(b + oA);
    h->prior = (float *)(b + oP);
    h->C = (float *)(b + oC);
    h->ec = (double *)(b + oE);
    h->fwd = (double *)(b + oF);
    h->bwd = (double *)(b + oBw);
    h->gamma = (double *)(b + oG);
    h->Zt = (double *)(b + oZ);
    h->xi = (double *)(b + oX);
    h->LL = (double *)(b + oLL);
    h->eoff = (double *)(b + oEo);
    h->logZ = (double *)(b + oLZ);
    h->trace = (double *)(b + oTr);
    h->flags = (unsigned *)(b + oFl);

    if (cudaMemsetAsync(h->flags, 0, 256, h->st) != cudaSuccess) {
        cudaFree(h->mem);
        delete h;
        return NFHMM_ECUDA;
    }
    *out = h;
    return NFHMM_OK;
}

int nhmm_train_set_data(nhmm_train_t *h, const float *V) {
    if (!h) return NFHMM_EINVAL;
    h->err.clear();
    if (!V) return tfail(h, NFHMM_EINVAL, "NULL data");
    TCU(h, cudaSetDevice(h->device));
    const size_t n = (size_t)h->M * h->T * h->F;
    TCU(h, cudaMemcpyAsync(h->V, V, n * 4, cudaMemcpyDefault, h->st));
    TCU(h, cudaMemsetAsync(h->flags, 0, sizeof(unsigned), h->st));
    check_data_kernel<<<256, 256, 0, h->st>>>(n, h->V, h->flags);
    TCU(h, cudaGetLastError());
    h->launches++;
    int r = t_flags(h);
    if (r) return r;
    h->have_data = true;
    return NFHMM_OK;
}

int nhmm_train_set_params(nhmm_train_t *h, const float *dict, const float *trans, const float *prior, const float *weights) {
    if (!h) return NFHMM_EINVAL;
    h->err.clear();
    if (!dict || !trans || !prior) return tfail(h, NFHMM_EINVAL, "dict, trans and prior are required");
    TCU(h, cudaSetDevice(h->device));
    const size_t MN = (size_t)h->M * h->N, MTN = (size_t)h->M * h->T * h->N;
    TCU(h, cudaMemcpyAsync(h->beta, dict, MN * h->K * h->F * 4, cudaMemcpyDefault, h->st));
    TCU(h, cudaMemcpyAsync(h->A, trans, MN * h->N * 4, cudaMemcpyDefault, h->st));
    TCU(h, cudaMemcpyAsync(h->prior, prior, MN * 4, cudaMemcpyDefault, h->st));
    if (weights) {
        TCU(h, cudaMemcpyAsync(h->theta, weights, MTN * h->K * 4, cudaMemcpyDefault, h->st));
    } else {   // uniform weights 1/K
        float *tmp = new (std::nothrow) float[MTN * h->K];
        if (!tmp) return tfail(h, NFHMM_ENOMEM, "host buffer");
        for (size_t i = 0; i < MTN * h->K; ++i) tmp[i] = 1.f / (float)h->K;
        cudaError_t e = cudaMemcpy(h->theta, tmp, MTN * h->K * 4, cudaMemcpyHostToDevice);
        delete[] tmp;
        TCU(h, e);
    }
    TCU(h, cudaStreamSynchronize(h->st));
    h->have_params = true;
    h->iters = 0;
    return NFHMM_OK;
}

int nhmm_train_em(nhmm_train_t *h, int32_t n_iters) {
    if (!h) return NFHMM_EINVAL;
    h->err.clear();
    if (!h->have_data || !h->have_params) return tfail(h, NFHMM_ESTATE, "set_data and set_params must precede em");
    if (n_iters < 0 || h->iters + n_iters > h->max_iters) return tfail(h, NFHMM_EINVAL, "n_iters beyond max_iters");
    TCU(h, cudaSetDevice(h->device));
    const int F = (int)h->F, T = (int)h->T, N = h->N, K = h->K, M = (int)h->M, MT = M * T;
    const int km = kmax_of(K), nch = (T + TCHUNK - 1) / TCHUNK;
    for (int it = 0; it < n_iters; ++it) {
        cudaError_t e;
        switch (km) {
            case 4: e = launch_estep<4>(F, T, N, K, M, h->V, h->beta, h->theta, h->LL, h->C, h->st); break;
            case 8: e = launch_estep<8>(F, T, N, K, M, h->V, h->beta, h->theta, h->LL, h->C, h->st); break;
            case 10: e = launch_estep<10>(F, T, N, K, M, h->V, h->beta, h->theta, h->LL, h->C, h->st); break;
            case 16: e = launch_estep<16>(F, T, N, K, M, h->V, h->beta, h->theta, h->LL, h->C, h->st); break;
            case 20: e = launch_estep<20>(F, T, N, K, M, h->V, h->beta, h->theta, h->LL, h->C, h->st); break;
            default: e = launch_estep<32>(F, T, N, K, M, h->V, h->beta, h->theta, h->LL, h->C, h->st); break;
        }
        TCU(h, e);
        emission_kernel<<<(MT + 7) / 8, 256, 0, h->st>>>(T, N, MT, h->LL, h->ec, h->eoff, h->flags);
        TCU(h, cudaGetLastError());
        {   // FP64 chain recursion per source (forward and backward warps), A in shared memory
            const size_t smem = ((size_t)N * N + 4 * (size_t)N) * 8;
            TCU(h, ensure_dyn_smem((const void *)train_fb_kernel, smem));
            train_fb_kernel<<<M, 64, smem, h->st>>>(T, N, h->ec, h->eoff, h->A, h->prior, h->fwd, h->bwd, h->logZ, h->flags);
            TCU(h, cudaGetLastError());
        }
        trace_kernel<<<(M + 127) / 128, 128, 0, h->st>>>(M, h->iters, h->max_iters, h->logZ, h->trace);
        posterior_kernel<<<(MT + 7) / 8, 256, 0, h->st>>>(T, N, MT, h->fwd, h->bwd, h->ec, h->A, h->gamma, h->Zt);
        xi_kernel<<<dim3((M * N * N + 255) / 256, nch), 256, 0, h->st>>>(T, N, M, TCHUNK, h->fwd, h->bwd, h->ec, h->Zt, h->A,
                                                                          h->xi);
        switch (km) {
            case 4: e = launch_beta<4>(F, T, N, K, M, TCHUNK, h->V, h->beta, h->theta, h->gamma, h->nb, h->st); break;
            case 8: e = launch_beta<8>(F, T, N, K, M, TCHUNK, h->V, h->beta, h->theta, h->gamma, h->nb, h->st); break;
            case 10: e = launch_beta<10>(F, T, N, K, M, TCHUNK, h->V, h->beta, h->theta, h->gamma, h->nb, h->st); break;
            case 16: e = launch_beta<16>(F, T, N, K, M, TCHUNK, h->V, h->beta, h->theta, h->gamma, h->nb, h->st); break;
            case 20: e = launch_beta<20>(F, T, N, K, M, TCHUNK, h->V, h->beta, h->theta, h->gamma, h->nb, h->st); break;
            default: e = launch_beta<32>(F, T, N, K, M, TCHUNK, h->V, h->beta, h->theta, h->gamma, h->nb, h->st); break;
        }
        TCU(h, e);
        beta_norm_kernel<<<(M * N * K + 7) / 8, 256, 0, h->st>>>(F, T, N, K, M * N * K, nch, h->nb, h->beta);
        mstep_kernel<<<(MT * N + 255) / 256, 256, 0, h->st>>>(T, N, K, M, nch, h->theta, h->C, h->xi, h->A, h->prior,
                                                              h->gamma);
        TCU(h, cudaGetLastError());
        h->launches += 9;
        h->iters++;
    }
    return t_flags(h);
}

int nhmm_train_get(nhmm_train_t *h, float *dict, float *trans, float *prior, float *weights, double *loglik,
                   int32_t *iters_done) {
    if (!h) return NFHMM_EINVAL;
    h->err.clear();
    TCU(h, cudaSetDevice(h->device));
    const size_t MN = (size_t)h->M * h->N, MTN = (size_t)h->M * h->T * h->N;
    if (dict) TCU(h, cudaMemcpyAsync(dict, h->beta, MN * h->K * h->F * 4, cudaMemcpyDefault, h->st));
    if (trans) TCU(h, cudaMemcpyAsync(trans, h->A, MN * h->N * 4, cudaMemcpyDefault, h->st));
    if (prior) TCU(h, cudaMemcpyAsync(prior, h->prior, MN * 4, cudaMemcpyDefault, h->st));
    if (weights) TCU(h, cudaMemcpyAsync(weights, h->theta, MTN * h->K * 4, cudaMemcpyDefault, h->st));
    if (loglik) TCU(h, cudaMemcpyAsync(loglik, h->trace, (size_t)h->M * h->max_iters * 8, cudaMemcpyDefault, h->st));
    TCU(h, cudaStreamSynchronize(h->st));
    if (iters_done) *iters_done = h->iters;
    return NFHMM_OK;
}

int nhmm_train_kernel_launches(const nhmm_train_t *h, int64_t *n) {
    if (!h || !n) return NFHMM_EINVAL;
    *n = h->launches;
    return NFHMM_OK;
}

int nhmm_train_destroy(nhmm_train_t *h) {
    if (!h) return NFHMM_OK;
    cudaSetDevice(h->device);
    if (h->mem) cudaFree(h->mem);
    delete h;
    return NFHMM_OK;
}

const char *nhmm_train_last_error(const nhmm_train_t *h) { return h ? h->err.c_str() : ""; }

}  // extern "C"
