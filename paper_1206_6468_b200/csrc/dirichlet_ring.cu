// dirichlet_ring.cu -- kernels (c)+(d) of the VB sweep (Eq. 6-8), round 2 default: persistent CTAs over
// tiles of FT consecutive frames, a two-stage ring of bulk copies (TMA engine) in and out.
//
// Same mathematics as dirichlet.cu (see there; DESIGN §6 "Dirichlet"):
//   Eq. 6  alpha_k = n_k + gamma d^{(s(k))}_{t,n(k)} + 1,  d = u .* b / sum_n (u .* b)  (R20);
//   Eq. 7  theta_k = exp(psi(alpha_k) - psi(alpha_0)),  alpha_0 = v_t + Kt + gamma S K (R19);
//   Eq. 8  phi_n^{(s)} = sum_{j<K} psi(alpha_{(sN+n)K+j}) - K psi(alpha_0), emitted centred:
//                  e = exp(gamma (phi - max_n phi)) (FP32), eoff = gamma (max_n phi - K psi_0) (FP64);
//   bound term (R8) H_t = sum_k g~(alpha_k) + fc[2],  g~(x) = lnG(x) - (x-1) psi(x) + x.
// What is different from the round-1 kernels is the schedule, not the arithmetic:
//   * work items are (frame, block) pairs: a tile of FT frames has FT*S*N items and FT is chosen so
//     every thread gets the same number of items (config 3: 16 frames x 80 blocks over 256 threads = 5
//     each; round 1 gave lanes 3 or 2 blocks of one frame) -- the per-frame small-vector steps (the Eq. 6
//     normalisers, the Eq. 8 maxima, the emissions, the bound sum) are likewise spread over the CTA;
//   * the tile's n rows, FB message rows and frame constants arrive by cp.async.bulk on an mbarrier while
//     the previous tile computes (two stages), and theta leaves by cp.async.bulk from the same stage
//     buffer (in place), so HBM traffic overlaps the element arithmetic;
//   * the Eq. 8 block sum of psi is accumulated as (integer exponent sum) ln 2 + FP32 sum of the bounded
//     remainders ln(mantissa) - r in (-0.6, 0.7) (psi(x) = E ln 2 + ln m - r, x = m 2^E), instead of one
//     FP64 conversion + add per element; the exponent part is exact, so the block sum is at least as
//     accurate as round 1's (whose per-element ln x = E ln 2 + ln m was rounded in FP32 before the FP64 add).
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include "dirichlet_math.cuh"
#include "nfhmm_internal.cuh"

namespace nfk {

namespace {

__device__ __forceinline__ uint32_t saddr(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t *b, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(saddr(b)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(saddr(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *b, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "RW_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@!P1 bra RW_%=;\n"
        "}\n" ::"r"(saddr(b)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *b) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                     saddr(dst)),
                 "l"(src), "r"(bytes), "r"(saddr(b))
                 : "memory");
}
__device__ __forceinline__ void bulk_s2g(void *dst, const void *src, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n" ::"l"(dst), "r"(saddr(src)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory"); }
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }

// x / d for 0 <= x < 2^22 via a float reciprocal (d <= 2^11), exact after one correction step
__device__ __forceinline__ int divq(int x, int d, float inv) {
    int q = __float2int_rz(__int2float_rn(x) * inv);
    const int r = x - q * d;
    if (r < 0) --q;
    else if (r >= d) ++q;
    return q;
}

// Shared-memory layout (bytes).  Per stage: n [FT][Kt] (theta in place) | u [S][FT][N] | b [S][FT][N] |
// fc [FT][4] doubles.  Common: 2 mbarriers | sps [FT][SN] doubles | hs [FT][SN] floats | gq, mx [FT][S].
struct RingLayout {
    size_t n, u, b, fc, stage, bars, sps, hs, gq, mx, total;
    __host__ __device__ RingLayout(int S, int N, int Kt, int FT) {
        const size_t SN = (size_t)S * N;
        n = 0;
        u = n + (((size_t)FT * Kt * 4 + 15) & ~size_t(15));
        b = u + ((SN * FT * 4 + 15) & ~size_t(15));
        fc = b + ((SN * FT * 4 + 15) & ~size_t(15));
        stage = fc + (size_t)FT * 32;
        stage = (stage + 127) & ~size_t(127);
        bars = 2 * stage;
        sps = bars + 16;
        hs = sps + SN * FT * 8;
        gq = hs + ((SN * FT * 4 + 7) & ~size_t(7));
        mx = gq + (size_t)FT * S * 4;
        total = mx + (size_t)FT * S * 4;
    }
};

// Element work of one (frame, block) item: KC = K at compile time (0: runtime K, any parity).
// psi(a) = E ln 2 + ln m - r,  a = m 2^E (m in [1, 2)),  u = 1/a,  r = u/2 + u^2 G(u)  (G as a polynomial in
// u, digamma_u_poly.cuh);  with w = u (-G) - 1/2:  -r = u w,
//   theta = a e^{-psi_0} exp(-r),
//   g~(a) = lnG(a) - (a-1) psi(a) + a = (E ln 2 + ln m)/2 + (ln(2 pi) + 1)/2 + u (H(u) + G - u G)
//         = (E ln 2 + ln m)/2 + (ln(2 pi) + 1)/2 + u (H(u) - (-G) + w + 1/2)   [H(u) - 1/2 + (1 - u) G].
// The item accumulates sum E (integer), sum log2 m, sum (-r) and sum u (H + G + w + 1/2 ...) in packed
// FP32 and assembles the Eq. 8 block sum of psi in FP64 once.  Per element pair: LDS.64, exponent
// (SHF + LEA.HI), mantissa (LOP3 x2), six SFU ops (lg2, rcp, ex2 per element), ~17 packed FP32 ops.
template <int KC>
__device__ __forceinline__ void item_elements(float *pn, int K, float dv, uint64_t e0_2, bool want_h, float *arow,
                                              double &psum, float &gsum) {
    const int KK = KC ? KC : K;
    const uint64_t dv2 = f2c(dv);
    const float gcoef[9] = DIG_GNU_COEF, hcoef[4] = LNG_HU_COEF;
    uint64_t L2 = 0ull, Q2 = 0ull, Gs2 = 0ull;   // sum log2 m, sum (-r), sum of the u-terms of g~
    int ebias = 0;                                // sum of the biased exponents (b >> 23)
#pragma unroll
    for (int j = 0; j < KK; j += 2) {
        const bool two = KC ? true : (j + 1 < KK);
        float n0, n1;
        if (KC) {
            const float2 nv = *reinterpret_cast<const float2 *>(pn + j);
            n0 = nv.x;
            n1 = nv.y;
        } else {
            n0 = pn[j];
            n1 = two ? pn[j + 1] : 0.f;
        }
        const uint64_t a2 = f2add(f2pack(n0, n1), dv2);
        float a0, a1;
        f2unpack(a2, a0, a1);
        if (!two) a1 = 1.f;   // padding element: exponent 127, log2 m = 0, u = 1 -- its terms are masked below
        const uint32_t b0 = __float_as_uint(a0), b1 = __float_as_uint(a1);
        ebias += (int)(b0 >> 23) + (int)(b1 >> 23);
        float l0, l1;   // log2 of the mantissas
        asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(l0) : "f"(__uint_as_float((b0 & 0x007FFFFFu) | 0x3F800000u)));
        asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(l1) : "f"(__uint_as_float((b1 & 0x007FFFFFu) | 0x3F800000u)));
        float u0 = rcp_sfu(a0), u1 = rcp_sfu(a1);
        if (!KC && !two) u1 = 0.f;                 // masks the padding element's -r and g~ terms
        const uint64_t u2 = f2pack(u0, u1);
        uint64_t Gn2 = f2c(gcoef[0]);              // -G(u), Horner in u
#pragma unroll
        for (int i = 1; i < 9; ++i) Gn2 = f2fma(Gn2, u2, f2c(gcoef[i]));
        const uint64_t w2 = f2fma(u2, Gn2, f2c(-0.5f));                           // w = -u G - 1/2
        const uint64_t rn2 = f2mul(u2, w2);                                       // -r
        float th0, th1;
        {   // theta = a e^{-psi_0} exp(-r)
            float r0, r1;
            f2unpack(f2mul(rn2, f2c(1.44269504088896341f)), r0, r1);
            f2unpack(f2mul(f2mul(a2, e0_2), f2pack(ex2_sfu(r0), ex2_sfu(r1))), th0, th1);
        }
        Q2 = f2add(Q2, rn2);
        L2 = f2add(L2, f2pack(l0, l1));            // (padding: log2 1 = 0)
        if (want_h) {   // u (H(u) - 1/2 + (1 - u) G) = u (H + (-G)(u - 1) - 1/2) = u (H - (-G) + w + 1/2 ... )
            uint64_t H2 = f2c(hcoef[0]);
#pragma unroll
            for (int i = 1; i < 4; ++i) H2 = f2fma(H2, u2, f2c(hcoef[i]));
            const uint64_t d2 = f2add(f2sub(H2, Gn2), w2);                       // H - 1/2 + (1 - u) G
            Gs2 = f2fma(u2, d2, Gs2);
        }
        if (KC) {
            *reinterpret_cast<float2 *>(pn + j) = make_float2(th0, th1);
            if (arow) *reinterpret_cast<float2 *>(arow + j) = make_float2(a0, a1);
        } else {
            pn[j] = th0;
            if (two) pn[j + 1] = th1;
            if (arow) {
                arow[j] = a0;
                if (two) arow[j + 1] = a1;
            }
        }
    }
    // exponent part: sum E = sum (b >> 23) - 127 x (elements + padding element, whose E is 0)
    const int npad = KC ? 0 : (KK & 1);
    const float esum = (float)(ebias - 127 * (KK + npad));
    float lx, ly, qx, qy, gx, gy;
    f2unpack(L2, lx, ly);
    f2unpack(Q2, qx, qy);
    f2unpack(Gs2, gx, gy);
    const float lsum = lx + ly;                    // sum log2 m
    // sum psi = ln 2 (sum E + sum log2 m) + sum (-r)
    psum = ((double)esum + (double)lsum) * 0.69314718055994530942 + (double)(qx + qy);
    // sum g~ = (ln 2 / 2)(sum E + sum log2 m) + K (ln(2 pi) + 1)/2 + sum u (...)
    gsum = (gx + gy) + (esum + lsum) * 0.346573590279972655f + (float)KK * 1.41893853320467274f;
}

constexpr int RING_IPT = 8;   // max (frame, block) items per thread and tile
constexpr int RING_G = 8;     // lanes per (frame, source) group in the small-vector phases
#ifndef RING_MAXREG
#define RING_MAXREG 128   // register cap: ptxas otherwise settles at 64 registers and serialises the element
                           // chains (config 3, 6-frame tiles: 0.98 -> 0.88 ms per launch with 112 registers)
#endif

template <int KC, int NT>
__global__ void __maxnreg__(RING_MAXREG) dirichlet_ring_kernel(DirichletArgs p, int FT) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    constexpr int NW = NT / 32;
    const int S = p.S, N = p.N, SN = S * N, K = KC ? KC : p.K, Kt = p.Kt, T = p.T, ld = p.ld;
    const int frames = p.frames;
    const float *__restrict__ n_in = p.n_in;
    const float *__restrict__ u_fwd = p.u_fwd;
    const float *__restrict__ b_bwd = p.b_bwd;
    const double *__restrict__ fconst = p.fconst;
    float *__restrict__ theta = p.theta;
    float *__restrict__ alpha = p.alpha;
    float *__restrict__ ec = p.ec;
    double *__restrict__ eoffp = p.eoff;
    double *__restrict__ hdir = p.hdir;
    const RingLayout L(S, N, Kt, FT);
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem_raw + L.bars);
    double *sps = reinterpret_cast<double *>(smem_raw + L.sps);   // [FT][SN]
    float *hs = reinterpret_cast<float *>(smem_raw + L.hs);       // [FT][SN]
    float *gq = reinterpret_cast<float *>(smem_raw + L.gq);       // [FT][S] gamma / sum_n u b
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int grp = lane / RING_G, g = lane % RING_G;             // (frame, source) group of 8 lanes
    const float gamma = p.gamma;
    const bool want_h = hdir != nullptr, want_a = p.write_alpha != 0;
    const int ntiles = (frames + FT - 1) / FT;
    const bool contiguous = ld == Kt;
    unsigned bad = 0;
    // this thread's first item (frame f, source s, state n) and the per-item stride NT in those digits
    int f_1st, s_1st, n_1st, df, ds, dn;
    {
        const float invSN = 1.f / (float)SN, invN = 1.f / (float)N;
        f_1st = divq(tid, SN, invSN);
        const int b = tid - f_1st * SN;
        s_1st = divq(b, N, invN);
        n_1st = b - s_1st * N;
        df = NT / SN;
        const int db = NT - df * SN;
        ds = db / N;
        dn = db - ds * N;
    }
    // one thread of the last warp (whose tail-phase share is the smallest) stores theta; its warp issues
    // the loads (the store thread first waits until its previous store has read the stage)
    constexpr int IO_WARP = NW - 1;
    const bool io_warp = warp == IO_WARP, io_thread = tid == IO_WARP * 32;
    if (io_thread) {
        mbar_init(&bars[0], 1);
        mbar_init(&bars[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();

    // warp IO_WARP: the tile's inputs into stage st, one bulk copy per lane (n rows | fc rows | u, b rows
    // per (run of consecutive t inside one mixture, source))
    auto issue = [&](int tile, int st) {
        unsigned char *sb = smem_raw + st * L.stage;
        float *nb = reinterpret_cast<float *>(sb + L.n);
        float *ub = reinterpret_cast<float *>(sb + L.u);
        float *bb = reinterpret_cast<float *>(sb + L.b);
        const int f0 = tile * FT, nf = min(FT, frames - f0);
        if (lane == 0) {
            bulk_wait_read0();     // the store of the tile that last used this stage has read it
            fence_async_smem();
            mbar_expect_tx(&bars[st], (uint32_t)nf * ((uint32_t)Kt * 4 + 8u * (uint32_t)SN + 32u));
        }
        __syncwarp();
        const int m0 = f0 / T, nrun = (f0 + nf - 1) / T - m0 + 1;
        const int nn = contiguous ? 1 : nf, ncopy = nn + 1 + nrun * S * 2;
        for (int c = lane; c < ncopy; c += 32) {
            if (c < nn) {
                if (contiguous) bulk_g2s(nb, n_in + (size_t)f0 * Kt, (uint32_t)nf * Kt * 4, &bars[st]);
                else bulk_g2s(nb + (size_t)c * Kt, n_in + (size_t)(f0 + c) * ld, Kt * 4, &bars[st]);
            } else if (c == nn) {
                bulk_g2s(sb + L.fc, fconst + 4 * (size_t)f0, (uint32_t)nf * 32, &bars[st]);
            } else {
                const int q = c - nn - 1, r = q / (2 * S), s = (q >> 1) - r * S, m = m0 + r;
                const int fs = max(f0, m * T), fe = min(f0 + nf, (m + 1) * T), t = fs - m * T;
                const size_t row = ((size_t)(m * S + s) * T + t) * N;
                const size_t dst = ((size_t)s * FT + (fs - f0)) * N;
                if (q & 1) bulk_g2s(bb + dst, b_bwd + row, (uint32_t)(fe - fs) * N * 4, &bars[st]);
                else bulk_g2s(ub + dst, u_fwd + row, (uint32_t)(fe - fs) * N * 4, &bars[st]);
            }
        }
    };
    // Eq. 6 normalisers gq[f][s] = gamma / sum_n u b of the tile in stage st: 8 lanes per (frame, source),
    // fixed-order sums; (frame, source) groups taken from the last warp down (the Eq. 8 phase, which
    // runs beside it, takes them from warp 0 up)
    const float invS = 1.f / (float)S;
    auto normalisers = [&](int tile, int st) {
        const unsigned char *sb = smem_raw + st * L.stage;
        const float *ub = reinterpret_cast<const float *>(sb + L.u);
        const float *bb = reinterpret_cast<const float *>(sb + L.b);
        const int npairs = min(FT, frames - tile * FT) * S;
        for (int pb = (NW - 1 - warp) * (32 / RING_G); pb < npairs; pb += NW * (32 / RING_G)) {
            const int pr = pb + grp;
            float q = 0.f;
            if (pr < npairs) {
                const int f = divq(pr, S, invS), s = pr - f * S;
                const float *u = ub + ((size_t)s * FT + f) * N, *b = bb + ((size_t)s * FT + f) * N;
                for (int n = g; n < N; n += RING_G) q = fmaf(u[n], b[n], q);
            }
            q += __shfl_xor_sync(0xffffffffu, q, 4);
            q += __shfl_xor_sync(0xffffffffu, q, 2);
            q += __shfl_xor_sync(0xffffffffu, q, 1);
            if (pr < npairs && g == 0) {
                if (!(q > 0.f) || !(q < INFINITY)) bad |= FLAG_NONFINITE;
                gq[pr] = gamma * __frcp_rn(q);
            }
        }
    };

    // prologue: the first tile's inputs and normalisers
    if ((int)blockIdx.x < ntiles) {
        if (io_warp) issue(blockIdx.x, 0);
        mbar_wait(&bars[0], 0);
        normalisers(blockIdx.x, 0);
    }
    __syncthreads();
    // per tile, two CTA barriers: [issue next | element pass] | [store | Eq. 8 | bound | next normalisers]
    int it = 0;
    // (mixture, t) of the tile's first frame, advanced incrementally (no division per tile)
    int m_t0 = (int)((long long)blockIdx.x * FT / T), t_t0 = (int)((long long)blockIdx.x * FT - (long long)m_t0 * T);
    const long long tstride = (long long)gridDim.x * FT;
    const int dm = (int)(tstride / T), dt = (int)(tstride - (long long)dm * T);
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
        const int st = it & 1;
        const int f0 = tile * FT, nf = min(FT, frames - f0), nitems = nf * SN, npairs = nf * S;
        const int nxt = tile + gridDim.x;
        unsigned char *sb = smem_raw + st * L.stage;
        float *nb = reinterpret_cast<float *>(sb + L.n);
        const float *ub = reinterpret_cast<const float *>(sb + L.u);
        const float *bb = reinterpret_cast<const float *>(sb + L.b);
        const double *fc = reinterpret_cast<const double *>(sb + L.fc);
        // the other stage is free (tile it-1's element pass, Eq. 8 and bound phases read it before the
        // last barrier; its theta store is awaited inside issue): refill it with the next tile
        if (io_warp && nxt < ntiles) issue(nxt, st ^ 1);

        // element pass: one thread per (frame, block) item; theta replaces n in the stage buffer
        {
            int f = f_1st, s = s_1st, n = n_1st;
#pragma unroll 1
            for (int i = tid; i < nitems; i += NT) {
                const int b = s * N + n;
                const int ui = (s * FT + f) * N + n;
                const float dv = fmaf(gq[f * S + s], ub[ui] * bb[ui], 1.f);
                const uint64_t e0_2 = f2c((float)fc[4 * f + 3]);
                float *arow = want_a ? alpha + (size_t)(f0 + f) * ld + b * K : nullptr;
                double ps;
                float gs;
                item_elements<KC>(nb + (size_t)f * Kt + b * K, K, dv, e0_2, want_h, arow, ps, gs);
                sps[i] = ps;
                hs[i] = gs;
                // next item i + NT in (frame, source, state) digits
                n += dn;
                const int cn = n >= N;
                n -= cn ? N : 0;
                s += ds + cn;
                const int cs = s >= S;
                s -= cs ? S : 0;
                f += df + cs;
            }
        }
        fence_async_smem();   // theta (generic writes) before the bulk store (async proxy) reads it
        __syncthreads();
        if (io_thread) {
            if (contiguous) {
                bulk_s2g(theta + (size_t)f0 * Kt, nb, (uint32_t)nf * Kt * 4);
            } else {
                for (int f = 0; f < nf; ++f) bulk_s2g(theta + (size_t)(f0 + f) * ld, nb + (size_t)f * Kt, Kt * 4);
            }
            bulk_commit();
        }
        // Eq. 8 per (frame, source), 8 lanes each: max over n (FP32 of the FP64 sums), offset eoff, and the
        // centred emissions e = exp(gamma (phi - max)) in (0, 1]
        for (int pb = warp * (32 / RING_G); pb < npairs; pb += NW * (32 / RING_G)) {
            const int pr = pb + grp;
            const bool ok = pr < npairs;
            const int f = ok ? divq(pr, S, invS) : 0, s = pr - f * S;
            const double *v = sps + (size_t)f * SN + s * N;
            float mxf = -INFINITY;
            if (ok)
                for (int n = g; n < N; n += RING_G) mxf = fmaxf(mxf, (float)v[n]);
            mxf = fmaxf(mxf, __shfl_xor_sync(0xffffffffu, mxf, 4));
            mxf = fmaxf(mxf, __shfl_xor_sync(0xffffffffu, mxf, 2));
            mxf = fmaxf(mxf, __shfl_xor_sync(0xffffffffu, mxf, 1));
            if (ok) {
                int m = m_t0, t = t_t0 + f;
                while (t >= T) t -= T, ++m;
                const double mx = (double)mxf;
                float *dst = ec + ((size_t)(m * S + s) * T + t) * N;
                for (int n = g; n < N; n += RING_G)
                    dst[n] = ex2_sfu((float)((double)gamma * (v[n] - mx)) * 1.44269504088896341f);
                if (g == 0) {
                    const double off = (double)gamma * (mx - (double)K * fc[4 * f + 1]);
                    eoffp[(size_t)(m * S + s) * T + t] = off;
                    if (!isfinite(off)) bad |= FLAG_NONFINITE;
                }
            }
        }
        if (want_h) {   // bound term per frame, 8 lanes each (fixed order), from the last warp down
            for (int fb = (NW - 1 - warp) * (32 / RING_G); fb < nf; fb += NW * (32 / RING_G)) {
                const int f = fb + grp;
                float h = 0.f;
                if (f < nf)
                    for (int b = g; b < SN; b += RING_G) h += hs[(size_t)f * SN + b];
                h += __shfl_xor_sync(0xffffffffu, h, 4);
                h += __shfl_xor_sync(0xffffffffu, h, 2);
                h += __shfl_xor_sync(0xffffffffu, h, 1);
                if (f < nf && g == 0) hdir[f0 + f] = (double)h + fc[4 * f + 2];
            }
        }
        // the next tile's normalisers (its inputs were issued at the top of this tile)
        if (nxt < ntiles) {
            mbar_wait(&bars[st ^ 1], ((it + 1) >> 1) & 1);
            normalisers(nxt, st ^ 1);
        }
        m_t0 += dm;
        t_t0 += dt;
        while (t_t0 >= T) t_t0 -= T, ++m_t0;
        __syncthreads();   // gq, sps, hs and this stage are free for the next tile
    }
    if (io_thread) bulk_wait0();   // the last theta store has landed before the kernel retires
    if (bad) atomicOr(p.flags, bad);
}

struct RingPick {
    int FT, nt;
};

// Tile shape: FT frames x (threads) with FT*S*N a multiple of the thread count (equal items per thread),
// a stage of at most ~40 KB (two stages + sums: three CTAs per SM) or, for long rows, one frame per stage.
RingPick ring_pick(int S, int N, int Kt) {
    // model (fitted to the round-2 tile sweep at config 3): throughput ~ lane utilisation of the element
    // pass x resident warps (up to 16 per SM; ~112 registers per thread, so registers cap the CTAs too)
    // (measured at config 3, ms per launch: 6 frames x 128 threads 0.88, 8 x 128 0.89, 8 x 160 0.92,
    // 4 x 128 1.06, 6 x 192 1.28)
    const int SN = S * N;
    RingPick best{0, 0};
    double best_score = -1.0;
    if (S > 255 || N > 65535) return best;
    for (int nt = 128; nt <= 160; nt += 32) {   // (192+ threads measured slower at every tile size)
        for (int FT = 1; FT <= 255; ++FT) {
            const RingLayout L(S, N, Kt, FT);
            if (L.total > 200 * 1024) break;
            const int items = FT * SN;
            const int per = (items + nt - 1) / nt;
            if (per > RING_IPT) break;
            const double eff = (double)items / ((double)per * nt);
            int ctas = (int)((227 * 1024) / (L.total + 1024));
            const int ctas_reg = 65536 / (RING_MAXREG * nt);
            if (ctas > ctas_reg) ctas = ctas_reg;
            if (ctas < 1) continue;
            const int warps = ctas * nt / 32;
            // (1 + 0.15 / FT): the per-tile phases, barriers and copy issue amortised over the tile's frames
            const double score = eff * (warps >= 16 ? 1.0 : warps / 16.0) / (1.0 + 0.15 / FT) * (nt == 128 ? 1.0 : 0.97);
            if (score > best_score + 1e-9) {   // ties: the first (fewest threads)
                best_score = score;
                best = {FT, nt};
            }
        }
    }
    return best;
}

template <int KC, int NT>
cudaError_t launch_ring_t(const DirichletArgs &a, int FT, cudaStream_t st) {
    const size_t smem = RingLayout(a.S, a.N, a.Kt, FT).total;
    auto kern = dirichlet_ring_kernel<KC, NT>;
    cudaError_t e = ensure_dyn_smem((const void *)kern, smem);
    if (e != cudaSuccess) return e;
    const long long need = (a.frames + FT - 1) / FT;
    const long long cap = (long long)device_sms() * occupancy_ctas((const void *)kern, NT, smem);
    const int grid = (int)(need < cap ? need : cap);
    kern<<<grid, NT, smem, st>>>(a, FT);
    return cudaGetLastError();
}

template <int KC>
cudaError_t launch_ring_k(const DirichletArgs &a, int FT, int nt, cudaStream_t st) {
    switch (nt) {
        case 128: return launch_ring_t<KC, 128>(a, FT, st);
        case 160: return launch_ring_t<KC, 160>(a, FT, st);
        case 192: return launch_ring_t<KC, 192>(a, FT, st);
        case 224: return launch_ring_t<KC, 224>(a, FT, st);
        default: return launch_ring_t<KC, 256>(a, FT, st);
    }
}

}  // namespace

bool dirichlet_ring_supported(const DirichletArgs &a) {
    // 16-byte bulk copies: rows of n (Kt floats, pitch ld) and of the FB messages (N floats) must be
    // multiples of 4 floats; the tile must fit the shared memory
    if (a.N % 4 || a.Kt % 4 || a.ld % 4) return false;
    return ring_pick(a.S, a.N, a.Kt).FT >= 1;
}

cudaError_t launch_dirichlet_ring(const DirichletArgs &a, cudaStream_t st) {
    RingPick pk = ring_pick(a.S, a.N, a.Kt);
    if (const char *e = getenv("NFHMM_DIR_RING")) {   // "FT,threads": tile-shape experiments
        int ft = 0, nt = 0;
        if (sscanf(e, "%d,%d", &ft, &nt) == 2 && ft >= 1 && ft <= 255 && nt >= 128 && nt <= 256 && nt % 32 == 0 &&
            RingLayout(a.S, a.N, a.Kt, ft).total <= 200 * 1024 && (ft * a.S * a.N + nt - 1) / nt <= RING_IPT)
            pk = {ft, nt};
    }
    if (pk.FT < 1) return cudaErrorInvalidValue;
    if (a.K == 10) return launch_ring_k<10>(a, pk.FT, pk.nt, st);
    if (a.K == 20) return launch_ring_k<20>(a, pk.FT, pk.nt, st);
    return launch_ring_k<0>(a, pk.FT, pk.nt, st);
}

}  // namespace nfk
