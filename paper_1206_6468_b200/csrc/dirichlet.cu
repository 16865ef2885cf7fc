// dirichlet.cu -- kernels (c) and (d) of the VB sweep, fused: one warp per frame, one pass, no block
// barriers.
//
//   (c) Eq. 6:  alpha_k = n_k + gamma * d^{(s(k))}_{t, n(k)} + 1,
//       alpha_0 = sum_k alpha_k = v_t + Kt + gamma S K   (Eq. 6 summed over k: sum_k z_{t,l,k} = 1 gives
//       sum_k n_k = v_t, and each q(D^(s)) marginal sums to 1 -- DESIGN R19), the same in every sweep: it
//       and its FP64 scalars (psi(alpha_0), the frame's bound constant) are computed once per
//       set_observations (frame_consts_kernel),
//       Eq. 7 weights: theta_k = exp(psi(alpha_k) - psi(alpha_0));
//   (d) Eq. 8:  phi_n^{(s)} = sum_{j<K} psi(alpha_{(sN+n)K+j}) - K psi(alpha_0), handed to the
//       forward-backward as gamma * phi (DESIGN R1), centred per (s, t): the emission
//       e = exp(gamma (phi - max_n phi)) in (0, 1] (FP32) and eoff = gamma max_n phi in FP64 (the FB is
//       shift-invariant per frame);
//   bound term (DESIGN R8): H_t = sum_k [lnG(alpha_k) - (alpha_k - 1) psi(alpha_k)]
//                                 - lnG(alpha_0) + (alpha_0 - Kt) psi(alpha_0).
// psi and lnGamma of every element come from one SFU log2, one SFU reciprocal and short polynomials in
// u = 1/x (digamma_u_poly.cuh, generated): psi(x) = ln x - u/2 - u^2 G(2u-1); theta = x e^{-psi_0}
// exp(-u/2 - u^2 G) (one SFU exp2 of a small argument); lnG(x) - (x-1) psi(x) + x =
// ln(x)/2 + ln(2 pi)/2 + 1/2 + u (H(2u-1) - 1/2) + (u - u^2) G(2u-1), which is O(ln x) -- the O(x ln x)
// parts cancel analytically, and the -x is added back once per frame as -alpha_0 in FP64.
// Each chunk of 32 (s, n) blocks is processed flat (lane = float4 of consecutive elements, coalesced
// loads and stores straight from / to HBM, independent elements for ILP), psi parked in shared memory;
// then lane b sums the K psi values of block b in FP64 for Eq. 8.
// HBM-bound: per frame it reads n (Kt floats) + u, b (2 S N) and writes theta (Kt) + e (S N) (+ alpha on the
// last sweep of a call: alpha is not read inside the sweep loop).
#include <cuda_runtime.h>
#include <math.h>

#include "digamma_u_poly.cuh"
#include "nfhmm_internal.cuh"

namespace nfk {

namespace {

constexpr int WPB = 8;   // frames (warps) per CTA

struct PsiU {
    float psi, lx, u, G, r;
};
// ln x for x >= 1 (normal): exponent * ln 2 + lg2(mantissa) * ln 2 on the SFU (|error| <= ~1.1e-7 for the
// mantissa part, plus the final rounding)
__device__ __forceinline__ float ln_sfu(float x) {
    const uint32_t b = __float_as_uint(x);
    const float m = __uint_as_float((b & 0x007FFFFFu) | 0x3F800000u);   // [1, 2)
    float l2m;
    asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(l2m) : "f"(m));
    return fmaf((float)((int)(b >> 23) - 127), 0.693147180559945309f, l2m * 0.693147180559945309f);
}
// psi(x) = ln x - r, r = u/2 + u^2 G(2u - 1), x >= 1 (alpha >= 1 by Eq. 6), FP32 (DESIGN R14)
__device__ __forceinline__ PsiU psi_u(float x) {
    PsiU o;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(o.u) : "f"(x));
    o.lx = ln_sfu(x);
    o.G = dig_G(fmaf(2.f, o.u, -1.f));
    o.r = fmaf(o.u * o.u, o.G, 0.5f * o.u);
    o.psi = o.lx - o.r;
    return o;
}
// theta = exp(psi(x) - psi_0) = x e^{-psi_0} exp(-r): the exponent is small (r <= 0.58), so the SFU exp2 is
// accurate to ~2^-22 relative (e0 = e^{-psi_0} is a per-frame FP64-derived constant)
__device__ __forceinline__ float theta_of(float x, const PsiU &o, float e0) {
    float er;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(er) : "f"(-1.44269504088896341f * o.r));
    return (x * e0) * er;
}
// g~(x) = lnG(x) - (x - 1) psi(x) + x, from the pieces of psi_u (no cancellation)
__device__ __forceinline__ float gtilde(const PsiU &o) {
    const float H = lng_H(fmaf(2.f, o.u, -1.f));
    return fmaf(0.5f, o.lx, 1.41893853320467274f) + fmaf(o.u, H - 0.5f, (o.u - o.u * o.u) * o.G);
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
    // per warp: sps [SN] doubles | dvs [SN] floats | psis [CK] floats (16-B aligned pieces)
    const size_t sps_b = ((size_t)SN * 8 + 15) & ~size_t(15), dvs_b = ((size_t)SN * 4 + 15) & ~size_t(15);
    const size_t per_warp = sps_b + dvs_b + (((size_t)CK * 4 + 15) & ~size_t(15));   // multiple of 16
    unsigned char *base = smem_raw + warp * per_warp;
    double *sps = reinterpret_cast<double *>(base);
    float *dvs = reinterpret_cast<float *>(base + sps_b);
    float *psis = reinterpret_cast<float *>(base + sps_b + dvs_b);

    const int f = blockIdx.x * WPB + warp;
    if (f >= p.frames) return;
    const int m = f / p.T, t = f - m * p.T;
    const float gamma = p.gamma;

    // per-block prior pseudo-counts gamma d + 1 of Eq. 6: d of the previous sweep = the FB messages'
    // product u .* b divided by its sum over n (one row of N per source)
    unsigned bad = 0;
    for (int s = 0; s < p.S; ++s) {
        const size_t row = ((size_t)(m * p.S + s) * p.T + t) * p.N;
        float qs = 0.f;
        for (int n = lane; n < p.N; n += 32) {
            const float v = p.u_fwd[row + n] * p.b_bwd[row + n];
            dvs[s * p.N + n] = v;
            qs += v;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) qs += __shfl_xor_sync(0xffffffffu, qs, o);
        if (!(qs > 0.f) || !(qs < INFINITY)) bad |= FLAG_NONFINITE;
        const float gq = gamma / qs;
        __syncwarp();
        for (int n = lane; n < p.N; n += 32) dvs[s * p.N + n] = fmaf(gq, dvs[s * p.N + n], 1.f);
    }
    const double psi0 = p.fconst[4 * (size_t)f + 1];
    const float e0 = (float)p.fconst[4 * (size_t)f + 3];   // e^{-psi(alpha_0)}
    const float invK = 1.f / (float)K;
    __syncwarp();

    const float4 *nin = reinterpret_cast<const float4 *>(p.n_in + (size_t)f * p.ld);
    float4 *aout = reinterpret_cast<float4 *>(p.alpha + (size_t)f * p.ld);
    float4 *tout = reinterpret_cast<float4 *>(p.theta + (size_t)f * p.ld);
    const bool want_h = p.hdir != nullptr, want_a = p.write_alpha != 0;
    float hg = 0.f;   // sum of g~ over this lane's elements
    for (int c0 = 0; c0 < p.Kt; c0 += CK) {
        const int cn = min(CK, p.Kt - c0), b0 = c0 / K;
        // flat, coalesced pass over the chunk: alpha, psi, theta, g~ per element (independent -> ILP);
        // psi parked in shared memory for the Eq. 8 block sums
        for (int q = lane; 4 * q < cn; q += 32) {
            const float4 v = nin[(c0 >> 2) + q];
            const float nv[4] = {v.x, v.y, v.z, v.w};
            float av[4], tv[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int i = 4 * q + e;
                av[e] = tv[e] = 0.f;
                if (i < cn) {
                    const int bl = (int)(((float)i + 0.5f) * invK);      // block of element i (i < 32 K)
                    const float a = nv[e] + dvs[b0 + bl];
                    const PsiU o = psi_u(a);
                    av[e] = a;
                    tv[e] = theta_of(a, o, e0);
                    psis[i] = o.psi;
                    if (want_h) hg += gtilde(o);   // (non-finite alpha propagates to eoff: checked there)
                }
            }
            if (want_a) aout[(c0 >> 2) + q] = make_float4(av[0], av[1], av[2], av[3]);
            tout[(c0 >> 2) + q] = make_float4(tv[0], tv[1], tv[2], tv[3]);
        }
        __syncwarp();
        // Eq. 8 segment sums: lane b owns block b0 + b (FP64)
        if (lane * K < cn) {
            double sp = 0.0;
            for (int j = 0; j < K; ++j) sp += (double)psis[lane * K + j];
            sps[b0 + lane] = sp;
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
        const double h = warp_sum_d((double)hg);
        if (lane == 0) p.hdir[f] = h + p.fconst[4 * (size_t)f + 2];
    }
    if (bad) atomicOr(p.flags, bad);
}

}  // namespace

cudaError_t launch_dirichlet(const DirichletArgs &a, cudaStream_t st) {
    const int SN = a.S * a.N, CK = 32 * a.K;
    const size_t per_warp = (((size_t)SN * 8 + 15) & ~size_t(15)) + (((size_t)SN * 4 + 15) & ~size_t(15)) +
                            (((size_t)CK * 4 + 15) & ~size_t(15));
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
