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
// Lane b owns (s, n) block b (rounds of 32 blocks): the Eq. 6 pseudo-count is one register, the Eq. 8
// block sum is lane-local (FP64), and elements go two at a time through a packed FFMA2 pipeline.
// HBM-bound: per frame it reads n (Kt floats) + u, b (2 S N) and writes theta (Kt) + e (S N) (+ alpha on the
// last sweep of a call: alpha is not read inside the sweep loop).
#include <cuda_runtime.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "dirichlet_math.cuh"
#include "nfhmm_internal.cuh"

namespace nfk {

namespace {

constexpr int WPB = 8;   // frames (warps) per CTA

__global__ void __launch_bounds__(WPB * 32) dirichlet_kernel(DirichletArgs p) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int SN = p.S * p.N, K = p.K;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // per warp: sps [SN] doubles (Eq. 8 block sums) | dvs [SN] floats (prior pseudo-counts) | rb [32 K]
    // floats (one round of 32 blocks of the n row, staged with coalesced loads), 16-B aligned
    const size_t sps_b = ((size_t)SN * 8 + 15) & ~size_t(15), dvs_b = ((size_t)SN * 4 + 15) & ~size_t(15);
    const size_t rb_b = ((size_t)32 * K * 4 + 15) & ~size_t(15);
    unsigned char *base = smem_raw + warp * (sps_b + dvs_b + rb_b);
    double *sps = reinterpret_cast<double *>(base);
    float *dvs = reinterpret_cast<float *>(base + sps_b);
    float *rb = reinterpret_cast<float *>(base + sps_b + dvs_b);

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
    const uint64_t e0_2 = f2c((float)p.fconst[4 * (size_t)f + 3]);   // e^{-psi(alpha_0)}
    __syncwarp();

    // rounds of 32 blocks: the round's n span (32 K contiguous floats) is staged with coalesced float4
    // loads, lane b owns block b of the round (pseudo-count in one register, lane-local Eq. 8 sum), theta
    // replaces n in the staging buffer and leaves with coalesced stores
    const float *nrow = p.n_in + (size_t)f * p.ld;
    float *arow = p.alpha + (size_t)f * p.ld;
    float *trow = p.theta + (size_t)f * p.ld;
    const bool want_h = p.hdir != nullptr, want_a = p.write_alpha != 0;
    uint64_t hg2 = 0ull;   // packed running sum of g~ over this lane's elements
    for (int r0 = 0; r0 < SN; r0 += 32) {
        const int nb = min(32, SN - r0), cnt = nb * K, k0r = r0 * K;   // k0r * 4 is a multiple of 16
        const int c4 = cnt >> 2;
        {
            const float4 *src = reinterpret_cast<const float4 *>(nrow + k0r);
            float4 *dst = reinterpret_cast<float4 *>(rb);
            for (int q = lane; q < c4; q += 32) dst[q] = src[q];
            for (int q = 4 * c4 + lane; q < cnt; q += 32) rb[q] = nrow[k0r + q];
        }
        __syncwarp();
        if (lane < nb) {
            const int b = r0 + lane;
            const float dv = dvs[b];
            const uint64_t dv2 = f2c(dv);
            float *pn = rb + lane * K;
            const int k0 = b * K;
            double sp = 0.0;
            for (int j = 0; j < K; j += 2) {
                const bool two = j + 1 < K;
                const float n0 = pn[j], n1 = two ? pn[j + 1] : 0.f;
                const uint64_t a2 = f2add(f2pack(n0, n1), dv2);
                float a0, a1;
                f2unpack(a2, a0, a1);
                if (!two) a1 = 1.f;
                uint64_t ps2, th2, g2;
                elem_pair(a0, a1, e0_2, want_h, ps2, th2, g2);
                float p0, p1, t0, t1, g0, g1;
                f2unpack(ps2, p0, p1);
                f2unpack(th2, t0, t1);
                f2unpack(g2, g0, g1);
                sp += (double)p0 + (two ? (double)p1 : 0.0);
                hg2 = f2add(hg2, f2pack(g0, two ? g1 : 0.f));
                pn[j] = t0;
                if (two) pn[j + 1] = t1;
                if (want_a) {
                    arow[k0 + j] = a0;
                    if (two) arow[k0 + j + 1] = a1;
                }
            }
            sps[b] = sp;
        }
        __syncwarp();
        {
            const float4 *src = reinterpret_cast<const float4 *>(rb);
            float4 *dst = reinterpret_cast<float4 *>(trow + k0r);
            for (int q = lane; q < c4; q += 32) dst[q] = src[q];
            for (int q = 4 * c4 + lane; q < cnt; q += 32) trow[k0r + q] = rb[q];
        }
        __syncwarp();
    }
    float hg;
    {
        float h0, h1;
        f2unpack(hg2, h0, h1);
        hg = h0 + h1;
    }
    __syncwarp();

    // Eq. 8: centre per source and emit.  Any offset works (the FB is shift-invariant per frame)
    // as long as e and eoff use the same one: the max is taken in FP32, the differences in FP64.
    for (int s = 0; s < p.S; ++s) {
        float mxf = -INFINITY;
        for (int n = lane; n < p.N; n += 32) mxf = fmaxf(mxf, (float)sps[s * p.N + n]);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) mxf = fmaxf(mxf, __shfl_xor_sync(0xffffffffu, mxf, o));
        const double mx = (double)mxf;
        float *dst = p.ec + ((size_t)(m * p.S + s) * p.T + t) * p.N;
        for (int n = lane; n < p.N; n += 32) dst[n] = expf((float)((double)gamma * (sps[s * p.N + n] - mx)));
        if (lane == 0) {
            const double off = (double)gamma * (mx - (double)K * psi0);
            p.eoff[(size_t)(m * p.S + s) * p.T + t] = off;
            if (!isfinite(off)) bad |= FLAG_NONFINITE;
        }
    }
    if (want_h) {   // (FP32 warp sum: |sum g~| ~ 3e3 per frame, error ~1e-4 against a tolerance of ~6 per frame)
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) hg += __shfl_xor_sync(0xffffffffu, hg, o);
        if (lane == 0) p.hdir[f] = (double)hg + p.fconst[4 * (size_t)f + 2];
    }
    if (bad) atomicOr(p.flags, bad);
}

__device__ __forceinline__ void cp_async_n(void *smem_dst, const void *gsrc, int bytes16) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"((unsigned)__cvta_generic_to_shared(smem_dst)),
                 "l"(gsrc));
    (void)bytes16;
}
__device__ __forceinline__ void cp_async_4(void *smem_dst, const void *gsrc) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"((unsigned)__cvta_generic_to_shared(smem_dst)),
                 "l"(gsrc));
}
__device__ __forceinline__ void cp_async_8(void *smem_dst, const void *gsrc) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"((unsigned)__cvta_generic_to_shared(smem_dst)),
                 "l"(gsrc));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_wait1() { asm volatile("cp.async.wait_group 1;\n" ::: "memory"); }

// Per-warp shared-memory layout of the pipelined kernel (bytes, 16-B aligned pieces): Eq. 8 block sums,
// pseudo-counts, and two frame buffers [n row (Kt rounded to 4) | u (S N) | b (S N) | 4 frame constants].
struct PipeLayout {
    size_t sps, dvs, buf0, nb, ub, bb, cb, buf_bytes, total;
    __host__ __device__ PipeLayout(int S, int N, int Kt, int nbuf = 2) {
        const int SN = S * N;
        size_t o = 0;
        sps = o; o += ((size_t)SN * 8 + 15) & ~size_t(15);
        dvs = o; o += ((size_t)SN * 4 + 15) & ~size_t(15);
        buf0 = o;
        nb = 0;
        ub = ((size_t)((Kt + 3) & ~3)) * 4;
        bb = ub + (((size_t)SN * 4 + 15) & ~size_t(15));
        cb = bb + (((size_t)SN * 4 + 15) & ~size_t(15));
        buf_bytes = cb + 32;
        total = buf0 + nbuf * buf_bytes;
    }
};

// Software-pipelined variant (per-warp smem small enough): persistent warps walk a strided set of frames
// and cp.async the NEXT frame's n row, FB messages and constants into the other buffer while computing
// the current one, so the kernel is bound by issue / HBM instead of one outstanding load per warp.
// theta is written back in place and leaves with coalesced float4 stores.  Same arithmetic as
// dirichlet_kernel (results are bitwise identical).
// NBUF = 1: one frame buffer per warp (no prefetch; more warps per SM hide the latency instead)
template <bool EVEN, int NBUF>   // K even: element pairs never straddle a block end (no pairing selects)
__global__ void __launch_bounds__(WPB * 32) dirichlet_pipe_kernel(DirichletArgs p) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int SN = p.S * p.N, K = p.K, Kt = p.Kt;
    const PipeLayout L(p.S, p.N, Kt, NBUF);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    unsigned char *base = smem_raw + warp * L.total;
    double *sps = reinterpret_cast<double *>(base + L.sps);
    float *dvs = reinterpret_cast<float *>(base + L.dvs);
    const int nwarps = gridDim.x * WPB;
    const float gamma = p.gamma;
    const bool want_h = p.hdir != nullptr, want_a = p.write_alpha != 0;
    const int Kt4 = (Kt + 3) >> 2;
    unsigned bad = 0;

    auto issue = [&](int f, int slot) {
        unsigned char *bf = base + L.buf0 + slot * L.buf_bytes;
        const float *nrow = p.n_in + (size_t)f * p.ld;
        for (int q = lane; q < Kt4; q += 32) cp_async_n(bf + L.nb + 16 * q, nrow + 4 * q, 16);
        const int m = f / p.T, t = f - m * p.T;
        if ((p.N & 3) == 0) {   // rows of N floats are 16-byte aligned: 16-byte copies
            const int N4 = p.N >> 2;
            for (int i = lane; i < p.S * N4; i += 32) {
                const int s = i / N4, n4 = i - s * N4;
                const size_t row = ((size_t)(m * p.S + s) * p.T + t) * p.N + 4 * n4;
                cp_async_n(bf + L.ub + 16 * i, p.u_fwd + row, 16);
                cp_async_n(bf + L.bb + 16 * i, p.b_bwd + row, 16);
            }
        } else {
            for (int i = lane; i < SN; i += 32) {
                const int s = i / p.N, n = i - s * p.N;
                const size_t row = ((size_t)(m * p.S + s) * p.T + t) * p.N + n;
                cp_async_4(bf + L.ub + 4 * i, p.u_fwd + row);
                cp_async_4(bf + L.bb + 4 * i, p.b_bwd + row);
            }
        }
        if (lane < 4) cp_async_8(bf + L.cb + 8 * lane, p.fconst + 4 * (size_t)f + lane);
        cp_commit();
    };

    int f = blockIdx.x * WPB + warp;
    if (NBUF == 2 && f < p.frames) issue(f, 0);
    for (int it = 0; f < p.frames; ++it) {
        const int fn = f + nwarps;
        if (NBUF == 2) {
            if (fn < p.frames) issue(fn, (it + 1) & 1);
            else cp_commit();
            cp_wait1();
        } else {
            issue(f, 0);
            asm volatile("cp.async.wait_group 0;\n" ::: "memory");
        }
        __syncwarp();
        unsigned char *bf = base + L.buf0 + (NBUF == 2 ? (it & 1) : 0) * L.buf_bytes;
        float *nbuf = reinterpret_cast<float *>(bf + L.nb);
        const float *ub = reinterpret_cast<const float *>(bf + L.ub);
        const float *bb = reinterpret_cast<const float *>(bf + L.bb);
        const double *fc = reinterpret_cast<const double *>(bf + L.cb);
        const int m = f / p.T, t = f - m * p.T;

        // pseudo-counts gamma d + 1 (d = u .* b / sum_n per source)
        for (int s = 0; s < p.S; ++s) {
            float qs = 0.f;
            for (int n = lane; n < p.N; n += 32) {
                const float v = ub[s * p.N + n] * bb[s * p.N + n];
                dvs[s * p.N + n] = v;
                qs += v;
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) qs += __shfl_xor_sync(0xffffffffu, qs, o);
            if (!(qs > 0.f) || !(qs < INFINITY)) bad |= FLAG_NONFINITE;
            const float gq = gamma * __frcp_rn(qs);
            __syncwarp();
            for (int n = lane; n < p.N; n += 32) dvs[s * p.N + n] = fmaf(gq, dvs[s * p.N + n], 1.f);
        }
        const double psi0 = fc[1];
        const uint64_t e0_2 = f2c((float)fc[3]);
        __syncwarp();

        // block-owner element pass over the staged row; theta replaces n in place
        float *arow = p.alpha + (size_t)f * p.ld;
        uint64_t hg2 = 0ull;
        for (int b = lane; b - lane < SN; b += 32) {
            if (b < SN) {
                const uint64_t dv2 = f2c(dvs[b]);
                float *pn = nbuf + b * K;
                double sp = 0.0;
                if (EVEN) {
                    for (int j = 0; j < K; j += 2) {
                        const float2 nv = *reinterpret_cast<const float2 *>(pn + j);
                        const uint64_t a2 = f2add(f2pack(nv.x, nv.y), dv2);
                        float a0, a1;
                        f2unpack(a2, a0, a1);
                        uint64_t ps2, th2, g2;
                        elem_pair(a0, a1, e0_2, want_h, ps2, th2, g2);
                        float p0, p1, t0, t1;
                        f2unpack(ps2, p0, p1);
                        f2unpack(th2, t0, t1);
                        sp += (double)p0 + (double)p1;
                        hg2 = f2add(hg2, g2);
                        *reinterpret_cast<float2 *>(pn + j) = make_float2(t0, t1);
                        if (want_a) *reinterpret_cast<float2 *>(arow + b * K + j) = make_float2(a0, a1);
                    }
                } else {
                    for (int j = 0; j < K; j += 2) {
                        const bool two = j + 1 < K;
                        const uint64_t a2 = f2add(f2pack(pn[j], two ? pn[j + 1] : 0.f), dv2);
                        float a0, a1;
                        f2unpack(a2, a0, a1);
                        uint64_t ps2, th2, g2;
                        elem_pair(a0, a1, e0_2, want_h, ps2, th2, g2);
                        float p0, p1, t0, t1, g0, g1;
                        f2unpack(ps2, p0, p1);
                        f2unpack(th2, t0, t1);
                        f2unpack(g2, g0, g1);
                        sp += (double)p0 + (two ? (double)p1 : 0.0);
                        hg2 = f2add(hg2, f2pack(g0, two ? g1 : 0.f));
                        pn[j] = t0;
                        if (two) pn[j + 1] = t1;
                        if (want_a) {
                            arow[b * K + j] = a0;
                            if (two) arow[b * K + j + 1] = a1;
                        }
                    }
                }
                sps[b] = sp;
            }
        }
        __syncwarp();
        float4 *trow = reinterpret_cast<float4 *>(p.theta + (size_t)f * p.ld);
        const int Ktf = Kt >> 2;   // whole float4s; a partial last one keeps the row padding zero
        for (int q = lane; q < Ktf; q += 32) trow[q] = reinterpret_cast<const float4 *>(nbuf)[q];
        if (Ktf < Kt4 && lane == 0) {
            float4 tv = reinterpret_cast<const float4 *>(nbuf)[Ktf];
            const int k = 4 * Ktf;
            if (k + 1 >= Kt) tv.y = 0.f;
            if (k + 2 >= Kt) tv.z = 0.f;
            if (k + 3 >= Kt) tv.w = 0.f;
            trow[Ktf] = tv;
        }
        float hg;
        {
            float h0, h1;
            f2unpack(hg2, h0, h1);
            hg = h0 + h1;
        }
        // Eq. 8: centre per source and emit (see dirichlet_kernel)
        for (int s = 0; s < p.S; ++s) {
            float mxf = -INFINITY;
            for (int n = lane; n < p.N; n += 32) mxf = fmaxf(mxf, (float)sps[s * p.N + n]);
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) mxf = fmaxf(mxf, __shfl_xor_sync(0xffffffffu, mxf, o));
            const double mx = (double)mxf;
            float *dst = p.ec + ((size_t)(m * p.S + s) * p.T + t) * p.N;
            // e = exp(gamma (phi - max)) <= 1: the difference in FP64, then one SFU exp2 (relative error of
            // e ~ 6e-8 |gamma (phi - max)|, i.e. < 1e-6 wherever e is not negligible)
            for (int n = lane; n < p.N; n += 32)
                dst[n] = ex2_sfu((float)((double)gamma * (sps[s * p.N + n] - mx)) * 1.44269504088896341f);
            if (lane == 0) {
                const double off = (double)gamma * (mx - (double)K * psi0);
                p.eoff[(size_t)(m * p.S + s) * p.T + t] = off;
                if (!isfinite(off)) bad |= FLAG_NONFINITE;
            }
        }
        if (want_h) {
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) hg += __shfl_xor_sync(0xffffffffu, hg, o);
            if (lane == 0) p.hdir[f] = (double)hg + fc[2];
        }
        __syncwarp();   // this buffer is refilled two frames from now
        f = fn;
    }
    if (bad) atomicOr(p.flags, bad);
}

// Frame-tile variant (N, Kt multiples of 4; configs 0-3): a CTA owns a tile of FT consecutive frames.
// The tile's n rows, FB message rows (consecutive t of one mixture are contiguous) and constants arrive
// by a few cp.async.bulk copies issued by one thread and tracked by one mbarrier; per-frame small-vector
// work is vectorised across the CTA instead of being repeated per warp: the Eq. 6 per-source sums and
// the Eq. 8 per-source maxima run one thread per (frame, source), the emissions one thread per (frame,
// block); the element pass runs one lane per (frame, block) over a warp's frames, so its lanes stay
// busy when S N is not a multiple of 32.  Same element arithmetic as the kernels above; the FP32 sums
// of u .* b over n are associated sequentially.
__device__ __forceinline__ uint32_t smem_addr(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void bar_init(uint64_t *b, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_addr(b)), "r"(count));
}
__device__ __forceinline__ void bar_expect_tx(uint64_t *b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_addr(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bar_wait(uint64_t *b, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@!P1 bra WAIT_%=;\n"
        "}\n" ::"r"(smem_addr(b)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_load(void *dst, const void *src, uint32_t bytes, uint64_t *b) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                     smem_addr(dst)),
                 "l"(src), "r"(bytes), "r"(smem_addr(b))
                 : "memory");
}

__device__ __forceinline__ int div_small(int x, int d, float inv) {   // x / d for 0 <= x < 2^24
    int q = __float2int_rz(__int2float_rn(x) * inv);
    const int r = x - q * d;
    if (r < 0) --q;
    else if (r >= d) ++q;
    return q;
}

constexpr int TILE_MAXFW = 4;   // frames per warp (FT <= 4 * warps)

struct TileLayout {   // bytes from the start of dynamic shared memory
    size_t bar, nb, ub, bb, fc, sps, gq, ecb, total;
    __host__ __device__ TileLayout(int S, int N, int Kt, int FT) {
        const size_t SN = (size_t)S * N;
        bar = 0;
        nb = 16;
        ub = nb + (size_t)FT * Kt * 4;
        bb = ub + SN * FT * 4;
        fc = bb + SN * FT * 4;
        sps = fc + (size_t)FT * 32;
        gq = sps + SN * FT * 8;
        ecb = gq + (size_t)FT * S * 4;
        ecb = (ecb + 7) & ~size_t(7);
        total = ecb + (size_t)FT * 8;
    }
    __host__ __device__ static size_t per_frame(int S, int N, int Kt) {
        return (size_t)Kt * 4 + (size_t)S * N * 16 + 32 + (size_t)S * 4 + 8;
    }
};

template <bool EVEN, int NW>   // NW warps per CTA
__global__ void __launch_bounds__(NW * 32) dirichlet_tile_kernel(DirichletArgs p, int FT) {
    constexpr int TILE_THREADS = NW * 32;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int S = p.S, N = p.N, SN = S * N, K = p.K, Kt = p.Kt, T = p.T;
    const TileLayout L(S, N, Kt, FT);
    uint64_t *bar = reinterpret_cast<uint64_t *>(smem_raw + L.bar);
    float *nb = reinterpret_cast<float *>(smem_raw + L.nb);       // [FT][Kt]   n, then theta in place
    float *ub = reinterpret_cast<float *>(smem_raw + L.ub);       // [S][FT][N] u
    float *bb = reinterpret_cast<float *>(smem_raw + L.bb);       // [S][FT][N] b
    double *fc = reinterpret_cast<double *>(smem_raw + L.fc);     // [FT][4]    frame constants
    double *sps = reinterpret_cast<double *>(smem_raw + L.sps);   // [FT][SN]   Eq. 8 block sums
    float *gq = reinterpret_cast<float *>(smem_raw + L.gq);       // [FT][S]    gamma / sum_n u b
    long long *ecb = reinterpret_cast<long long *>(smem_raw + L.ecb);   // [FT] m S T + t: (m, s=0, t) row
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const float gamma = p.gamma;
    const bool want_h = p.hdir != nullptr, want_a = p.write_alpha != 0;
    const float invN = 1.f / (float)N, invSN = 1.f / (float)SN, invS = 1.f / (float)S;
    const int ntiles = (p.frames + FT - 1) / FT;
    unsigned bad = 0;
    if (tid == 0) {
        bar_init(bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
    uint32_t phase = 0;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, phase ^= 1) {
        const int f0 = tile * FT, nf = min(FT, p.frames - f0);
        if (tid == 0) {
            asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");   // the previous tile's reads first
            bar_expect_tx(bar, (uint32_t)nf * ((uint32_t)Kt * 4 + 8u * (uint32_t)SN + 32u));
            if (p.ld == Kt) {
                bulk_load(nb, p.n_in + (size_t)f0 * Kt, (uint32_t)nf * Kt * 4, bar);
            } else {
                for (int f = 0; f < nf; ++f) bulk_load(nb + (size_t)f * Kt, p.n_in + (size_t)(f0 + f) * p.ld, Kt * 4, bar);
            }
            for (int f = f0; f < f0 + nf;) {   // runs of consecutive t inside one mixture
                const int m = f / T, t = f - m * T, len = min(f0 + nf - f, T - t);
                for (int s2 = 0; s2 < S; ++s2) {
                    const size_t row = ((size_t)(m * S + s2) * T + t) * N;
                    const size_t dst = ((size_t)s2 * FT + (f - f0)) * N;
                    bulk_load(ub + dst, p.u_fwd + row, (uint32_t)len * N * 4, bar);
                    bulk_load(bb + dst, p.b_bwd + row, (uint32_t)len * N * 4, bar);
                }
                f += len;
            }
            bulk_load(fc, p.fconst + 4 * (size_t)f0, (uint32_t)nf * 32, bar);
        }
        if (tid < nf) {
            const int f = f0 + tid, m = f / T, t = f - m * T;
            ecb[tid] = (long long)m * S * T + t;
        }
        bar_wait(bar, phase);

        // Eq. 6 prior pseudo-counts: gq = gamma / sum_n u .* b, one warp per (frame, source)
        for (int k = warp; k < nf * S; k += NW) {
            const int f = div_small(k, S, invS), s2 = k - f * S;
            const float *u = ub + ((size_t)s2 * FT + f) * N, *b = bb + ((size_t)s2 * FT + f) * N;
            float q = 0.f;
            for (int n = lane; n < N; n += 32) q = fmaf(u[n], b[n], q);
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) q += __shfl_xor_sync(0xffffffffu, q, o);
            if (!(q > 0.f) || !(q < INFINITY)) bad |= FLAG_NONFINITE;
            if (lane == 0) gq[k] = gamma * __frcp_rn(q);
        }
        __syncthreads();

        // element pass: warp w owns frames w, w + NW, ...; lane = (frame, block) item
        {
            const int nfw = warp < nf ? (nf - warp + NW - 1) / NW : 0;
            float hsum[TILE_MAXFW] = {0.f, 0.f, 0.f, 0.f};
            const int items = nfw * SN;
            for (int i0 = 0; i0 < items; i0 += 32) {
                const int i = i0 + lane;
                if (i < items) {
                    const int jj = div_small(i, SN, invSN), b = i - jj * SN;
                    const int f = warp + NW * jj;
                    const int s2 = div_small(b, N, invN), n = b - s2 * N;
                    const size_t ui = ((size_t)s2 * FT + f) * N + n;
                    const uint64_t dv2 = f2c(fmaf(gq[f * S + s2], ub[ui] * bb[ui], 1.f));
                    const uint64_t e0_2 = f2c((float)fc[4 * f + 3]);
                    float *pn = nb + (size_t)f * Kt + b * K;
                    float *arow = p.alpha + (size_t)(f0 + f) * p.ld + b * K;
                    double sp = 0.0;
                    uint64_t hg2 = 0ull;
                    if (EVEN) {
                        for (int j = 0; j < K; j += 2) {
                            const float2 nv = *reinterpret_cast<const float2 *>(pn + j);
                            const uint64_t a2 = f2add(f2pack(nv.x, nv.y), dv2);
                            float a0, a1;
                            f2unpack(a2, a0, a1);
                            uint64_t ps2, th2, g2;
                            elem_pair(a0, a1, e0_2, want_h, ps2, th2, g2);
                            float p0, p1, t0, t1;
                            f2unpack(ps2, p0, p1);
                            f2unpack(th2, t0, t1);
                            sp += (double)p0 + (double)p1;
                            hg2 = f2add(hg2, g2);
                            *reinterpret_cast<float2 *>(pn + j) = make_float2(t0, t1);
                            if (want_a) *reinterpret_cast<float2 *>(arow + j) = make_float2(a0, a1);
                        }
                    } else {
                        for (int j = 0; j < K; j += 2) {
                            const bool two = j + 1 < K;
                            const uint64_t a2 = f2add(f2pack(pn[j], two ? pn[j + 1] : 0.f), dv2);
                            float a0, a1;
                            f2unpack(a2, a0, a1);
                            uint64_t ps2, th2, g2;
                            elem_pair(a0, a1, e0_2, want_h, ps2, th2, g2);
                            float p0, p1, t0, t1, g0, g1;
                            f2unpack(ps2, p0, p1);
                            f2unpack(th2, t0, t1);
                            f2unpack(g2, g0, g1);
                            sp += (double)p0 + (two ? (double)p1 : 0.0);
                            hg2 = f2add(hg2, f2pack(g0, two ? g1 : 0.f));
                            pn[j] = t0;
                            if (two) pn[j + 1] = t1;
                            if (want_a) {
                                arow[j] = a0;
                                if (two) arow[j + 1] = a1;
                            }
                        }
                    }
                    sps[(size_t)f * SN + b] = sp;
                    float h0, h1;
                    f2unpack(hg2, h0, h1);
#pragma unroll
                    for (int k = 0; k < TILE_MAXFW; ++k)
                        if (k == jj) hsum[k] += h0 + h1;
                }
            }
            if (want_h) {   // per-frame bound term (FP32 warp sum, as in the kernels above)
#pragma unroll
                for (int k = 0; k < TILE_MAXFW; ++k) {
                    if (k >= nfw) break;
                    float h = hsum[k];
#pragma unroll
                    for (int o = 16; o > 0; o >>= 1) h += __shfl_xor_sync(0xffffffffu, h, o);
                    const int f = warp + NW * k;
                    if (lane == 0) p.hdir[f0 + f] = (double)h + fc[4 * f + 2];
                }
            }
        }
        __syncthreads();

        // theta leaves (coalesced float4 rows; contiguous when ld == Kt)
        {
            const int q4 = Kt >> 2;
            if (p.ld == Kt) {
                float4 *dst = reinterpret_cast<float4 *>(p.theta + (size_t)f0 * Kt);
                const float4 *src = reinterpret_cast<const float4 *>(nb);
                for (int q = tid; q < nf * q4; q += TILE_THREADS) dst[q] = src[q];
            } else {
                for (int q = tid; q < nf * q4; q += TILE_THREADS) {
                    const int f = q / q4, c = q - f * q4;
                    reinterpret_cast<float4 *>(p.theta + (size_t)(f0 + f) * p.ld)[c] =
                        reinterpret_cast<const float4 *>(nb + (size_t)f * Kt)[c];
                }
            }
        }
        // Eq. 8 per (frame, source): max in FP32 (over the FP64 sums), offset eoff = gamma (max - K psi_0);
        // the max goes to gq (no longer needed)
        for (int k = warp; k < nf * S; k += NW) {   // one warp per (frame, source)
            const int f = div_small(k, S, invS), s2 = k - f * S;
            const double *v = sps + (size_t)f * SN + s2 * N;
            float mxf = -INFINITY;
            for (int n = lane; n < N; n += 32) mxf = fmaxf(mxf, (float)v[n]);
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) mxf = fmaxf(mxf, __shfl_xor_sync(0xffffffffu, mxf, o));
            if (lane == 0) {
                gq[k] = mxf;
                const double off = (double)gamma * ((double)mxf - (double)K * fc[4 * f + 1]);
                p.eoff[(size_t)ecb[f] + (size_t)s2 * T] = off;
                if (!isfinite(off)) bad |= FLAG_NONFINITE;
            }
        }
        __syncthreads();
        // emissions, one thread per (frame, block): e = exp(gamma (phi - max)) in (0, 1]
        for (int j = tid; j < nf * SN; j += TILE_THREADS) {
            const int f = div_small(j, SN, invSN), b = j - f * SN;
            const int s2 = div_small(b, N, invN), n = b - s2 * N;
            const double mx = (double)gq[f * S + s2];
            p.ec[((size_t)ecb[f] + (size_t)s2 * T) * N + n] =
                ex2_sfu((float)((double)gamma * (sps[j] - mx)) * 1.44269504088896341f);
        }
        __syncthreads();   // the next tile's copies overwrite the buffers
    }
    if (bad) atomicOr(p.flags, bad);
}

// ---------------------------------------------------------------------------------------------------
// Fused path (the element work of (c)+(d) runs in the back-projection GEMM's epilogue, gemm_tc.cu):
//   dv_kernel   (before the GEMM)  dvT[b][f] = gamma d_{s,t,n} + 1 for block b = s N + n,
//               d = u .* b / sum_n (u .* b);
//   eq8_kernel  (after the GEMM)   Eq. 8 block sums of psi (spsT, plus sps2T for the blocks whose K elements
//               straddle two epilogue warps' 32-column chunks) -> centred emissions e and offsets eoff, and
//               the frame's bound term H_t from the per-column-tile g~ partial sums hpartT.
// The per-block arrays are block-major ([block][frame]): in the GEMM epilogue thread = frame row, so
// a warp's reads of dvT and writes of spsT / hpartT are 128-byte coalesced rows.  Both kernels move them
// through a [SN][33] shared tile, 32 frames per CTA.
constexpr int FR = 32;   // frames per CTA of the fused-path kernels

__global__ void __launch_bounds__(WPB * 32) dv_kernel(DirichletArgs p, float *dvT) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    float *tl = reinterpret_cast<float *>(smem_raw);   // [SN][FR + 1]
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int SN = p.S * p.N, f0 = blockIdx.x * FR;
    unsigned bad = 0;
    for (int fl = warp; fl < FR; fl += WPB) {
        const int f = f0 + fl;
        if (f >= p.frames) break;
        const int m = f / p.T, t = f - m * p.T;
        for (int s = 0; s < p.S; ++s) {
            const size_t row = ((size_t)(m * p.S + s) * p.T + t) * p.N;
            float q[4], qs = 0.f;   // N <= 128
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int n = lane + 32 * i;
                q[i] = n < p.N ? p.u_fwd[row + n] * p.b_bwd[row + n] : 0.f;
                qs += q[i];
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) qs += __shfl_xor_sync(0xffffffffu, qs, o);
            if (!(qs > 0.f) || !(qs < INFINITY)) bad |= FLAG_NONFINITE;
            const float gq = p.gamma * __frcp_rn(qs);
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int n = lane + 32 * i;
                if (n < p.N) tl[(s * p.N + n) * (FR + 1) + fl] = fmaf(gq, q[i], 1.f);
            }
        }
    }
    __syncthreads();
    if (f0 + lane < p.frames)
        for (int b = warp; b < SN; b += WPB) dvT[(size_t)b * p.ldf + f0 + lane] = tl[b * (FR + 1) + lane];
    if (bad) atomicOr(p.flags, bad);
}

__global__ void __launch_bounds__(WPB * 32) eq8_kernel(DirichletArgs p, const double *spsT, const double *sps2T,
                                                       const double *hpartT, int n_tiles, int bn) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    double *tl = reinterpret_cast<double *>(smem_raw);   // [SN][FR + 1]
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int SN = p.S * p.N, K = p.K, f0 = blockIdx.x * FR;
    const bool fok = f0 + lane < p.frames;
    for (int b = warp; b < SN; b += WPB) {
        double v = 0.0;
        if (fok) {
            const size_t i = (size_t)b * p.ldf + f0 + lane;
            v = spsT[i];
            const int ls = (b * K) % bn;   // block start inside its column tile
            if ((ls >> 5) != ((ls + K - 1) >> 5)) v += sps2T[i];
        }
        tl[b * (FR + 1) + lane] = v;
    }
    if (p.hdir && warp == 0 && fok) {
        const int f = f0 + lane;
        double h = 0.0;
        for (int c = 0; c < n_tiles; ++c) h += hpartT[(size_t)c * p.ldf + f];
        p.hdir[f] = h + p.fconst[4 * (size_t)f + 2];
    }
    __syncthreads();
    unsigned bad = 0;
    for (int fl = warp; fl < FR; fl += WPB) {
        const int f = f0 + fl;
        if (f >= p.frames) break;
        const int m = f / p.T, t = f - m * p.T;
        const double psi0 = p.fconst[4 * (size_t)f + 1];
        for (int s = 0; s < p.S; ++s) {
            double v[4];
            float mxf = -INFINITY;
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int n = lane + 32 * i;
                v[i] = n < p.N ? tl[(s * p.N + n) * (FR + 1) + fl] : 0.0;
                if (n < p.N) mxf = fmaxf(mxf, (float)v[i]);
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) mxf = fmaxf(mxf, __shfl_xor_sync(0xffffffffu, mxf, o));
            const double mx = (double)mxf;
            float *dst = p.ec + ((size_t)(m * p.S + s) * p.T + t) * p.N;
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int n = lane + 32 * i;
                if (n < p.N) dst[n] = ex2_sfu((float)((double)p.gamma * (v[i] - mx)) * 1.44269504088896341f);
            }
            if (lane == 0) {
                const double off = (double)p.gamma * (mx - (double)K * psi0);
                p.eoff[(size_t)(m * p.S + s) * p.T + t] = off;
                if (!isfinite(off)) bad |= FLAG_NONFINITE;
            }
        }
    }
    if (bad) atomicOr(p.flags, bad);
}

}  // namespace

size_t fused_tile_bytes(int SN, int elem) { return (size_t)SN * (FR + 1) * elem; }

cudaError_t launch_dv(const DirichletArgs &a, float *dvT, cudaStream_t st) {
    const size_t smem = fused_tile_bytes(a.S * a.N, 4);
    if (a.N > 128 || smem > 200 * 1024) return cudaErrorInvalidValue;
    {
        cudaError_t e = ensure_dyn_smem((const void *)dv_kernel, smem);
        if (e != cudaSuccess) return e;
    }
    dv_kernel<<<(a.frames + FR - 1) / FR, WPB * 32, smem, st>>>(a, dvT);
    return cudaGetLastError();
}

cudaError_t launch_eq8(const DirichletArgs &a, const double *spsT, const double *sps2T, const double *hpartT,
                       int n_tiles, int bn, cudaStream_t st) {
    const size_t smem = fused_tile_bytes(a.S * a.N, 8);
    if (a.N > 128 || smem > 200 * 1024) return cudaErrorInvalidValue;
    {
        cudaError_t e = ensure_dyn_smem((const void *)eq8_kernel, smem);
        if (e != cudaSuccess) return e;
    }
    eq8_kernel<<<(a.frames + FR - 1) / FR, WPB * 32, smem, st>>>(a, spsT, sps2T, hpartT, n_tiles, bn);
    return cudaGetLastError();
}

cudaError_t launch_dirichlet(const DirichletArgs &a, cudaStream_t st) {
    if (a.variant == 0 && dirichlet_ring_supported(a)) return launch_dirichlet_ring(a, st);
    const int SN = a.S * a.N;
    const PipeLayout L(a.S, a.N, a.Kt);
    if (a.variant == 1 && a.N % 4 == 0 && a.Kt % 4 == 0 && a.ld % 4 == 0) {
        // frame tile: 2 frames per warp (so a warp's (frame, block) items fill its lanes), as many warps as
        // fit the shared-memory budget, 4 or 8 (NFHMM_DIR_TILE=warps,KB overrides for experiments)
        static int nw = 4, budget = 37;
        static bool env_read = false;
        if (!env_read) {
            env_read = true;
            const char *e = getenv("NFHMM_DIR_TILE");
            if (e) sscanf(e, "%d,%d", &nw, &budget);
            if (nw != 8) nw = 4;
        }
        int FT = (int)(((size_t)budget * 1024 - 16) / TileLayout::per_frame(a.S, a.N, a.Kt));
        if (FT > TILE_MAXFW * nw) FT = TILE_MAXFW * nw;
        FT &= ~(nw - 1);
        if (FT >= nw) {
            const size_t smem = TileLayout(a.S, a.N, a.Kt, FT).total;
            const bool even = (a.K & 1) == 0;
            const int ki = (even ? 1 : 0) + (nw == 8 ? 2 : 0);
            auto kern = nw == 8 ? (even ? dirichlet_tile_kernel<true, 8> : dirichlet_tile_kernel<false, 8>)
                                : (even ? dirichlet_tile_kernel<true, 4> : dirichlet_tile_kernel<false, 4>);
            (void)ki;
            cudaError_t e = ensure_dyn_smem((const void *)kern, smem);
            if (e != cudaSuccess) return e;
            const long long need = (a.frames + FT - 1) / FT;
            const long long cap = (long long)device_sms() * occupancy_ctas((const void *)kern, nw * 32, smem);
            const int grid = (int)(need < cap ? need : cap);
            kern<<<grid, nw * 32, smem, st>>>(a, FT);
            return cudaGetLastError();
        }
    }
    if (L.total <= 12 * 1024) {   // pipelined variant (configs 0-3); config 4's 32 KB rows use the other
        // one frame buffer per warp (4 CTAs = 32 warps per SM hide the load latency) measured 4.5 % faster
        // than two buffers (3 CTAs, next frame prefetched); NFHMM_DIR_NBUF=2 selects the latter
        // (the round-staged kernel below measured 1.50 vs 1.13 ms at config 3)
        static int nbuf = 0;
        if (!nbuf) {
            const char *e = getenv("NFHMM_DIR_NBUF");
            nbuf = (e && atoi(e) == 2) ? 2 : 1;
        }
        const size_t smem = PipeLayout(a.S, a.N, a.Kt, nbuf).total * WPB;
        const bool even = (a.K & 1) == 0;
        auto kern = nbuf == 1 ? (even ? dirichlet_pipe_kernel<true, 1> : dirichlet_pipe_kernel<false, 1>)
                              : (even ? dirichlet_pipe_kernel<true, 2> : dirichlet_pipe_kernel<false, 2>);
        cudaError_t e = ensure_dyn_smem((const void *)kern, smem);
        if (e != cudaSuccess) return e;
        const long long need = (a.frames + WPB - 1) / WPB;
        const long long cap = (long long)device_sms() * occupancy_ctas((const void *)kern, WPB * 32, smem);
        const int grid = (int)(need < cap ? need : cap);
        kern<<<grid, WPB * 32, smem, st>>>(a);
        return cudaGetLastError();
    }
    const size_t per_warp = (((size_t)SN * 8 + 15) & ~size_t(15)) + (((size_t)SN * 4 + 15) & ~size_t(15)) +
                            (((size_t)32 * a.K * 4 + 15) & ~size_t(15));
    const size_t smem = per_warp * WPB;
    {
        cudaError_t e = ensure_dyn_smem((const void *)dirichlet_kernel, smem);
        if (e != cudaSuccess) return e;
    }
    dirichlet_kernel<<<(a.frames + WPB - 1) / WPB, WPB * 32, smem, st>>>(a);
    return cudaGetLastError();
}

}  // namespace nfk
