// dirichlet.cu -- kernels (c) and (d) of the VB sweep, fused: one CTA per frame.
//
//   (c) Eq. 6:  alpha_k = n_k + gamma * d^{(s(k))}_{t, n(k)} + 1, alpha_0 = sum_k alpha_k (FP64),
//       Eq. 7 weights: theta_k = exp(psi(alpha_k) - psi(alpha_0));
//   (d) Eq. 8:  phi_n^{(s)} = sum_{j<K} psi(alpha_{(sN+n)K+j}) - K psi(alpha_0), emitted to the
//       forward-backward as gamma * phi (DESIGN R1), centred per (s, t): ec = gamma (phi - max_n phi),
//       eoff = gamma max_n phi in FP64 (the FB is shift-invariant per frame);
//   bound term (DESIGN R8): H_t = sum_k [lnG(alpha_k) - (alpha_k - 1) psi(alpha_k)]
//                                 - lnG(alpha_0) + (alpha_0 - Kt) psi(alpha_0)   (FP64 accumulation).
// HBM-bound: reads n (Kt floats) + d (S N), writes alpha, theta (2 Kt) + phi (S N) per frame,
// 128-bit vectorised and coalesced; the per-block sums of Eq. 8 read psi back from shared memory.
#include <cuda_runtime.h>
#include <math.h>

#include "nfhmm_internal.cuh"

namespace nfk {

namespace {

// psi(x) for x >= 1 (alpha >= 1 by Eq. 6).  Recurrence to x >= 6, then the asymptotic series to
// x^-10 (truncation < 1e-11 at x = 6); IEEE FP32, no fast-math (DESIGN R14).
__device__ __forceinline__ float digammaf_pos(float x) {
    float r = 0.f;
    while (x < 6.f) {
        r -= 1.f / x;
        x += 1.f;
    }
    const float f = 1.f / (x * x);
    const float t = f * (-1.f / 12.f + f * (1.f / 120.f + f * (-1.f / 252.f + f * (1.f / 240.f + f * (-1.f / 132.f)))));
    return r + logf(x) - 0.5f / x + t;
}

__device__ double digamma_d(double x) {
    double r = 0.0;
    while (x < 10.0) {
        r -= 1.0 / x;
        x += 1.0;
    }
    const double f = 1.0 / (x * x);
    const double t = f * (-1.0 / 12 + f * (1.0 / 120 + f * (-1.0 / 252 + f * (1.0 / 240 + f * (-1.0 / 132 +
                     f * (691.0 / 32760 + f * (-1.0 / 12)))))));
    return r + log(x) - 0.5 / x + t;
}

// g(a) = lnGamma(a) - (a - 1) psi(a): FP32 for a < 64 (no catastrophic cancellation there), FP64
// Stirling form for large a, where lnGamma and (a-1)psi are both ~a ln a and cancel to ~ -a.
__device__ __forceinline__ double gterm(float a, float psi_a) {
    if (a < 64.f) return (double)(lgammaf(a) - (a - 1.f) * psi_a);
    const double x = a, ix = 1.0 / x, ix2 = ix * ix;
    // lnG(x) - (x-1) psi(x) = 0.5 ln x - x + 0.5 ln(2 pi) + 0.5 - 1/(3x) - 1/(12x^2) - 1/(90x^3) + 1/(120 x^4) ...
    // (derived from the Stirling series of lnGamma and the asymptotic series of psi; terms to x^-5)
    const double series = -ix / 3.0 - ix2 / 12.0 - ix2 * ix / 90.0 + ix2 * ix2 / 120.0 + ix2 * ix2 * ix / 1260.0;
    return 0.5 * log(x) - x + 0.91893853320467274178 + 0.5 + series;
}

__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Block-wide FP64 sum with a fixed reduction tree (deterministic).  All threads get the result.
__device__ double block_sum_d(double v, double *scratch) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    v = warp_sum_d(v);
    __syncthreads();
    if (lane == 0) scratch[w] = v;
    __syncthreads();
    double s = 0.0;
    for (int i = 0; i < nw; ++i) s += scratch[i];
    return s;
}

__global__ void __launch_bounds__(128) dirichlet_kernel(DirichletArgs p) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    // layout: row [ld] floats (alpha, then psi) | dsm [S*N] floats | sps [S*N] doubles | mx [S] doubles | scratch [4]
    float *row = reinterpret_cast<float *>(smem_raw);
    const int SN = p.S * p.N;
    float *dsm = row + p.ld;
    double *sps = reinterpret_cast<double *>(reinterpret_cast<uintptr_t>(dsm + SN + 1) & ~uintptr_t(7));
    double *mx = sps + SN;
    double *scratch = mx + p.S;
    __shared__ double s_psi0;

    const int f = blockIdx.x;
    const int m = f / p.T, t = f - m * p.T;
    const int tid = threadIdx.x;
    const int nv = p.ld >> 2;

    for (int b = tid; b < SN; b += blockDim.x) {
        const int s = b / p.N, n = b - s * p.N;
        dsm[b] = p.d_hat[((size_t)(m * p.S + s) * p.T + t) * p.N + n];
    }
    __syncthreads();

    // Eq. 6: alpha_k = n_k + gamma d_{s(k), n(k)} + 1, kept in shared memory; alpha_0 in FP64.
    const float4 *nin = reinterpret_cast<const float4 *>(p.n_in + (size_t)f * p.ld);
    double a0p = 0.0;
    for (int q = tid; q < nv; q += blockDim.x) {
        const float4 v = nin[q];
        const float vv[4] = {v.x, v.y, v.z, v.w};
        float a[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int k = 4 * q + j;
            a[j] = k < p.Kt ? vv[j] + p.gamma * dsm[k / p.K] + 1.f : 0.f;
            a0p += (double)a[j];
        }
        *reinterpret_cast<float4 *>(row + 4 * q) = make_float4(a[0], a[1], a[2], a[3]);
    }
    const double a0 = block_sum_d(a0p, scratch);
    if (tid == 0) s_psi0 = digamma_d(a0);
    __syncthreads();
    const double psi0 = s_psi0;
    const float psi0f = (float)psi0;

    // Eq. 7 weights theta = exp(psi(alpha) - psi(alpha_0)); psi kept for Eq. 8; bound terms.
    float4 *aout = reinterpret_cast<float4 *>(p.alpha + (size_t)f * p.ld);
    float4 *tout = reinterpret_cast<float4 *>(p.theta + (size_t)f * p.ld);
    double hp = 0.0;
    unsigned bad = 0;
    for (int q = tid; q < nv; q += blockDim.x) {
        const float4 a4 = *reinterpret_cast<const float4 *>(row + 4 * q);
        const float a[4] = {a4.x, a4.y, a4.z, a4.w};
        float ps[4], th[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int k = 4 * q + j;
            if (k < p.Kt) {
                ps[j] = digammaf_pos(a[j]);
                th[j] = expf(ps[j] - psi0f);
                if (p.hdir) hp += gterm(a[j], ps[j]);
                if (!isfinite(a[j]) || !isfinite(th[j])) bad |= FLAG_NONFINITE;
            } else {
                ps[j] = 0.f;
                th[j] = 0.f;
            }
        }
        aout[q] = a4;
        tout[q] = make_float4(th[0], th[1], th[2], th[3]);
        *reinterpret_cast<float4 *>(row + 4 * q) = make_float4(ps[0], ps[1], ps[2], ps[3]);
    }
    __syncthreads();

    // Eq. 8 block sums (FP64) of psi over the K elements of each (s, n) block.
    for (int b = tid; b < SN; b += blockDim.x) {
        double acc = 0.0;
        const float *pp = row + b * p.K;
        for (int j = 0; j < p.K; ++j) acc += (double)pp[j];
        sps[b] = acc;
    }
    __syncthreads();
    if (tid < p.S) {
        double mm = -INFINITY;
        for (int n = 0; n < p.N; ++n) mm = fmax(mm, sps[tid * p.N + n]);
        mx[tid] = mm;
        const size_t o = (size_t)(m * p.S + tid) * p.T + t;
        const double off = (double)p.gamma * (mm - (double)p.K * psi0);
        p.eoff[o] = off;
        if (!isfinite(off)) bad |= FLAG_NONFINITE;
    }
    __syncthreads();
    for (int b = tid; b < SN; b += blockDim.x) {
        const int s = b / p.N, n = b - s * p.N;
        p.ec[((size_t)(m * p.S + s) * p.T + t) * p.N + n] = (float)((double)p.gamma * (sps[b] - mx[s]));
    }
    if (p.hdir) {
        const double h = block_sum_d(hp, scratch);
        if (tid == 0) p.hdir[f] = h - lgamma(a0) + (a0 - (double)p.Kt) * psi0;
    }
    if (bad) atomicOr(p.flags, bad);
}

}  // namespace

cudaError_t launch_dirichlet(const DirichletArgs &a, cudaStream_t st) {
    const int SN = a.S * a.N;
    size_t smem = (size_t)a.ld * 4 + (size_t)SN * 4 + 16 + (size_t)SN * 8 + (size_t)a.S * 8 + 4 * 8;
    smem = (smem + 15) & ~size_t(15);
    static bool attr_set = false;
    if (smem > 48 * 1024 && !attr_set) {
        cudaFuncSetAttribute(dirichlet_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
        attr_set = true;
    }
    dirichlet_kernel<<<a.frames, 128, smem, st>>>(a);
    return cudaGetLastError();
}

}  // namespace nfk
