// dirichlet.cu -- kernels (c) and (d) of the VB sweep, fused: one warp per frame, no block barriers.
//
//   (c) Eq. 6:  alpha_k = n_k + gamma * d^{(s(k))}_{t, n(k)} + 1,  alpha_0 = sum_k alpha_k (FP64),
//       Eq. 7 weights: theta_k = exp(psi(alpha_k) - psi(alpha_0));
//   (d) Eq. 8:  phi_n^{(s)} = sum_{j<K} psi(alpha_{(sN+n)K+j}) - K psi(alpha_0), handed to the
//       forward-backward as gamma * phi (DESIGN R1), centred per (s, t): the emission
//       e = exp(gamma (phi - max_n phi)) in (0, 1] (FP32) and eoff = gamma max_n phi in FP64 (the FB is
//       shift-invariant per frame);
//   bound term (DESIGN R8): H_t = sum_k [lnG(alpha_k) - (alpha_k - 1) psi(alpha_k)]
//                                 - lnG(alpha_0) + (alpha_0 - Kt) psi(alpha_0)      (FP64 accumulation).
// HBM-bound: per frame it reads n (Kt floats) + d (S N) and writes alpha, theta (2 Kt) + phi (S N).
// Pass 1 streams the row with 128-bit loads for alpha_0; pass 2 re-reads it (L1/L2-resident) in chunks
// of 32 (s, n) blocks staged through shared memory, so that each lane owns whole blocks (the Eq. 8
// segment sums need no cross-lane reduction) while global loads and stores stay coalesced float4.
#include <cuda_runtime.h>
#include <math.h>

#include "nfhmm_internal.cuh"
#include "psi_lngamma_poly.cuh"

namespace nfk {

namespace {

constexpr int WPB = 8;   // frames (warps) per CTA

// psi(x) and lnGamma(x) for x >= 1 (alpha >= 1 by Eq. 6), FP32 without fast-math (DESIGN R14).
// x in [1, 6): degree-10 polynomials per unit interval (psi_lngamma_poly.cuh, float32 error <= 1.3e-7 /
// 3.3e-7 absolute), read from a shared-memory copy of the tables (lanes in different intervals hit
// different banks); x >= 6: the asymptotic series
// psi(x) = ln x - 1/(2x) - 1/(12x^2) + 1/(120x^4) - 1/(252x^6) + 1/(240x^8)          (trunc. < 2e-9)
// lnG(x) = (x - 1/2) ln x - x + ln(2 pi)/2 + 1/(12x) - 1/(360x^3) + 1/(1260x^5)       (trunc. < 2e-8)
struct PsiLg {
    float psi, lng, ly, r;   // ly = ln x, r = 1/x on the asymptotic branch (reused by gterm)
};
__device__ __forceinline__ PsiLg psi_lngamma(float x, bool want_lng, const float *tab) {
    PsiLg o;
    if (x < 6.f) {
        const int n = (int)x;                               // 1..5
        const float v = 2.f * (x - (float)n) - 1.f;
        const float *cp = tab + (n - 1) * 11, *cl = tab + 55 + (n - 1) * 11;
        float ps = cp[10], lg = cl[10];
#pragma unroll
        for (int i = 9; i >= 0; --i) {
            ps = fmaf(ps, v, cp[i]);
            lg = fmaf(lg, v, cl[i]);
        }
        o.psi = ps;
        o.lng = lg;
        o.ly = o.r = 0.f;
        return o;
    }
    const float r = 1.f / x;
    const float f = r * r;
    const float ly = logf(x);
    o.psi = ly - 0.5f * r + f * (-1.f / 12.f + f * (1.f / 120.f + f * (-1.f / 252.f + f * (1.f / 240.f))));
    o.lng = 0.f;
    o.ly = ly;
    o.r = r;
    if (want_lng) o.lng = (x - 0.5f) * ly - x + 0.91893853320467274f + r * (1.f / 12.f + f * (-1.f / 360.f + f * (1.f / 1260.f)));
    return o;
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

// g(a) = lnGamma(a) - (a - 1) psi(a).  FP32 below 64 (no catastrophic cancellation there); above, the
// FP64 Stirling form (lnGamma and (a-1) psi are both ~ a ln a and cancel to ~ -a):
// g(x) = ln(x)/2 - x + ln(2 pi)/2 + 1/2 - 1/(3x) - 1/(12x^2) - 1/(90x^3) + 1/(120x^4) + 1/(1260x^5) + ...
__device__ __forceinline__ double gterm(float a, const PsiLg &pl) {
    if (a < 64.f) return (double)(pl.lng - (a - 1.f) * pl.psi);
    // large a: the series terms in FP32 (|.| < 6e-3), the O(a) part assembled in FP64 from the FP32 ln a
    const float ix = pl.r, ix2 = ix * ix;
    const float series = ix * (-1.f / 3.f + ix * (-1.f / 12.f + ix * (-1.f / 90.f + ix * (1.f / 120.f + ix * (1.f / 1260.f)))));
    (void)ix2;
    return 0.5 * (double)pl.ly - (double)a + (0.91893853320467274178 + 0.5) + (double)series;
}

__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ double warp_max_d(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

__global__ void __launch_bounds__(WPB * 32) dirichlet_kernel(DirichletArgs p) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int SN = p.S * p.N, K = p.K, CK = 32 * K;   // CK = elements per chunk of 32 blocks
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // per warp: sps [SN] doubles | dsm [SN] floats | ca [CK] floats | ct [CK] floats (16-B aligned pieces)
    const size_t sps_b = ((size_t)SN * 8 + 15) & ~size_t(15), dsm_b = ((size_t)SN * 4 + 15) & ~size_t(15);
    const size_t per_warp = sps_b + dsm_b + 2 * (((size_t)CK * 4 + 15) & ~size_t(15));   // multiple of 16
    unsigned char *base = smem_raw + warp * per_warp;
    double *sps = reinterpret_cast<double *>(base);
    float *dsm = reinterpret_cast<float *>(base + sps_b);
    float *ca = reinterpret_cast<float *>(base + sps_b + dsm_b);
    float *ct = ca + ((CK + 3) & ~3);

    __shared__ float tab[110];   // psi / lnGamma polynomial tables (see psi_lngamma)
    for (int i = threadIdx.x; i < 110; i += blockDim.x) tab[i] = i < 55 ? (&kPsiPoly[0][0])[i] : (&kLgPoly[0][0])[i - 55];
    __syncthreads();
    const int f = blockIdx.x * WPB + warp;
    if (f >= p.frames) return;
    const int m = f / p.T, t = f - m * p.T;
    const float gamma = p.gamma;

    // d of the previous sweep for this frame (one coalesced row of N per source)
    double dsum = 0.0;
    for (int s = 0; s < p.S; ++s) {
        const float *src = p.d_hat + ((size_t)(m * p.S + s) * p.T + t) * p.N;
        for (int n = lane; n < p.N; n += 32) {
            const float v = src[n];
            dsm[s * p.N + n] = v;
            dsum += (double)v;
        }
    }
    // pass 1: alpha_0 = sum_k n_k + Kt + gamma K sum_{s,n} d   (FP64)
    const float4 *nin = reinterpret_cast<const float4 *>(p.n_in + (size_t)f * p.ld);
    const int nv = p.ld >> 2;
    double nsum = 0.0;
    for (int q = lane; q < nv; q += 32) {
        const float4 v = nin[q];
        nsum += ((double)v.x + (double)v.y) + ((double)v.z + (double)v.w);
    }
    const double a0 = warp_sum_d(nsum) + (double)p.Kt + (double)gamma * (double)K * warp_sum_d(dsum);
    const double psi0 = digamma_d(a0);
    const float psi0f = (float)psi0;
    __syncwarp();

    // pass 2: chunks of 32 blocks; lane b owns block (c*32 + b)
    float4 *aout = reinterpret_cast<float4 *>(p.alpha + (size_t)f * p.ld);
    float4 *tout = reinterpret_cast<float4 *>(p.theta + (size_t)f * p.ld);
    const bool want_h = p.hdir != nullptr;
    double hp = 0.0;
    unsigned bad = 0;
    for (int c0 = 0; c0 < p.Kt; c0 += CK) {
        const int cend = min(c0 + CK, p.Kt);
        const int q0 = c0 >> 2, q1 = (cend + 3) >> 2;      // float4 range covering the chunk
        for (int q = q0 + lane; q < q1; q += 32) reinterpret_cast<float4 *>(ca)[q - q0] = nin[q];
        __syncwarp();
        const int b = (c0 / K) + lane;                        // global block index
        if (b < SN) {
            const float dv = gamma * dsm[b] + 1.f;
            float *pa = ca + lane * K, *pt = ct + lane * K;
            double sp = 0.0;
            for (int j = 0; j < K; ++j) {
                const float a = pa[j] + dv;
                const PsiLg pl = psi_lngamma(a, want_h, tab);
                const float th = expf(pl.psi - psi0f);
                pa[j] = a;
                pt[j] = th;
                sp += (double)pl.psi;
                if (want_h) hp += gterm(a, pl);
                if (!isfinite(a) || !isfinite(th)) bad |= FLAG_NONFINITE;
            }
            sps[b] = sp;
        }
        __syncwarp();
        for (int q = q0 + lane; q < q1; q += 32) {
            float4 av = reinterpret_cast<const float4 *>(ca)[q - q0];
            float4 tv = reinterpret_cast<const float4 *>(ct)[q - q0];
            const int k = 4 * q;
            if (k + 0 >= p.Kt) av.x = tv.x = 0.f;
            if (k + 1 >= p.Kt) av.y = tv.y = 0.f;
            if (k + 2 >= p.Kt) av.z = tv.z = 0.f;
            if (k + 3 >= p.Kt) av.w = tv.w = 0.f;
            aout[q] = av;
            tout[q] = tv;
        }
        __syncwarp();
    }

    // Eq. 8: centre per source and emit
    for (int s = 0; s < p.S; ++s) {
        double mx = -INFINITY;
        for (int n = lane; n < p.N; n += 32) mx = fmax(mx, sps[s * p.N + n]);
        mx = warp_max_d(mx);
        float *dst = p.ec + ((size_t)(m * p.S + s) * p.T + t) * p.N;
        for (int n = lane; n < p.N; n += 32) dst[n] = expf((float)((double)gamma * (sps[s * p.N + n] - mx)));
        if (lane == 0) {
            const double off = (double)gamma * (mx - (double)K * psi0);
            p.eoff[(size_t)(m * p.S + s) * p.T + t] = off;
            if (!isfinite(off)) bad |= FLAG_NONFINITE;
        }
    }
    if (want_h) {
        const double h = warp_sum_d(hp);
        if (lane == 0) p.hdir[f] = h - lgamma(a0) + (a0 - (double)p.Kt) * psi0;
    }
    if (bad) atomicOr(p.flags, bad);
}

}  // namespace

cudaError_t launch_dirichlet(const DirichletArgs &a, cudaStream_t st) {
    const int SN = a.S * a.N, CK = 32 * a.K;
    const size_t per_warp = (((size_t)SN * 8 + 15) & ~size_t(15)) + (((size_t)SN * 4 + 15) & ~size_t(15)) +
                            2 * (((size_t)CK * 4 + 15) & ~size_t(15));
    const size_t smem = per_warp * WPB;
    static size_t attr = 0;
    if (smem > 48 * 1024 && attr < smem) {
        cudaError_t e = cudaFuncSetAttribute(dirichlet_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        attr = smem;
    }
    dirichlet_kernel<<<(a.frames + WPB - 1) / WPB, WPB * 32, smem, st>>>(a);
    return cudaGetLastError();
}

}  // namespace nfk
