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
// Returns the Eq. 8 sum of psi in FP64 and the item's g~ sum (without its exponent part, added here).
template <int KC>
__device__ __forceinline__ void item_elements(float *pn, int K, float dv, uint64_t e0_2, bool want_h, float *arow,
                                              double &psum, float &gsum) {
    const int KK = KC ? KC : K;
    const uint64_t dv2 = f2c(dv);
    uint64_t q2 = 0ull, E2 = 0ull, g2 = 0ull;
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
        if (!two) a1 = 1.f;   // padding element: psi(1) etc. are discarded below
        // psi(a) = E ln 2 + ln m - r,  r = u/2 + u^2 G(2u - 1),  u = 1/a,  a = m 2^E, m in [1, 2)
        const uint32_t b0 = __float_as_uint(a0), b1 = __float_as_uint(a1);
        float l0, l1;
        asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(l0) : "f"(__uint_as_float((b0 & 0x007FFFFFu) | 0x3F800000u)));
        asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(l1) : "f"(__uint_as_float((b1 & 0x007FFFFFu) | 0x3F800000u)));
        const uint64_t e2 = f2pack((float)((int)(b0 >> 23) - 127), two ? (float)((int)(b1 >> 23) - 127) : 0.f);
        const uint64_t lm2 = f2mul(f2pack(l0, l1), f2c(0.693147180559945309f));   // ln m
        const uint64_t u2 = f2pack(rcp_sfu(a0), rcp_sfu(a1));
        const uint64_t t2 = f2fma(u2, f2c(2.f), f2c(-1.f));
        const uint64_t G2 = dig_G2(t2);
        const uint64_t uu2 = f2mul(u2, u2);
        const uint64_t r2 = f2fma(uu2, G2, f2mul(u2, f2c(0.5f)));
        uint64_t qd = f2sub(lm2, r2);                                                // ln m - r
        float th0, th1;
        {
            float r0, r1;
            f2unpack(f2mul(r2, f2c(-1.44269504088896341f)), r0, r1);
            f2unpack(f2mul(f2mul(a2, e0_2), f2pack(ex2_sfu(r0), ex2_sfu(r1))), th0, th1);
        }
        uint64_t gd = 0ull;
        if (want_h) {   // g~ - (E ln 2)/2 = ln(m)/2 + ln(2 pi)/2 + 1/2 + u (H - 1/2) + (u - u^2) G
            const uint64_t H2 = lng_H2(t2);
            const uint64_t g0 = f2fma(f2c(0.5f), lm2, f2c(1.41893853320467274f));
            gd = f2add(g0, f2fma(u2, f2sub(H2, f2c(0.5f)), f2mul(f2sub(u2, uu2), G2)));
        }
        if (!two) {   // drop the padding element's share
            float x0, x1;
            f2unpack(qd, x0, x1);
            qd = f2pack(x0, 0.f);
            f2unpack(gd, x0, x1);
            gd = f2pack(x0, 0.f);
        }
        q2 = f2add(q2, qd);
        E2 = f2add(E2, e2);
        g2 = f2add(g2, gd);
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
    float qx, qy, ex, ey, gx, gy;
    f2unpack(q2, qx, qy);
    f2unpack(E2, ex, ey);
    f2unpack(g2, gx, gy);
    const float esum = ex + ey;   // exact (integers < 2^24)
    psum = (double)esum * 0.69314718055994530942 + (double)(qx + qy);
    gsum = (gx + gy) + esum * 0.346573590279972655f;
}

template <int KC, int NT>
__global__ void __launch_bounds__(NT) dirichlet_ring_kernel(DirichletArgs p, int FT) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int S = p.S, N = p.N, SN = S * N, K = p.K, Kt = p.Kt, T = p.T;
    const RingLayout L(S, N, Kt, FT);
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem_raw + L.bars);
    double *sps = reinterpret_cast<double *>(smem_raw + L.sps);   // [FT][SN]
    float *hs = reinterpret_cast<float *>(smem_raw + L.hs);       // [FT][SN]
    float *gq = reinterpret_cast<float *>(smem_raw + L.gq);       // [FT][S] gamma / sum_n u b
    float *mxs = reinterpret_cast<float *>(smem_raw + L.mx);      // [FT][S] Eq. 8 maxima
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const float gamma = p.gamma;
    const bool want_h = p.hdir != nullptr, want_a = p.write_alpha != 0;
    const float invSN = 1.f / (float)SN, invN = 1.f / (float)N, invS = 1.f / (float)S;
    const int ntiles = (p.frames + FT - 1) / FT;
    const bool contiguous = p.ld == Kt;
    unsigned bad = 0;
    if (tid == 0) {
        mbar_init(&bars[0], 1);
        mbar_init(&bars[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();

    auto issue = [&](int tile, int st) {   // thread 0: the tile's inputs into stage st
        unsigned char *sb = smem_raw + st * L.stage;
        float *nb = reinterpret_cast<float *>(sb + L.n);
        float *ub = reinterpret_cast<float *>(sb + L.u);
        float *bb = reinterpret_cast<float *>(sb + L.b);
        const int f0 = tile * FT, nf = min(FT, p.frames - f0);
        mbar_expect_tx(&bars[st], (uint32_t)nf * ((uint32_t)Kt * 4 + 8u * (uint32_t)SN + 32u));
        if (contiguous) {
            bulk_g2s(nb, p.n_in + (size_t)f0 * Kt, (uint32_t)nf * Kt * 4, &bars[st]);
        } else {
            for (int f = 0; f < nf; ++f) bulk_g2s(nb + (size_t)f * Kt, p.n_in + (size_t)(f0 + f) * p.ld, Kt * 4, &bars[st]);
        }
        for (int f = f0; f < f0 + nf;) {   // runs of consecutive t inside one mixture
            const int m = f / T, t = f - m * T, len = min(f0 + nf - f, T - t);
            for (int s = 0; s < S; ++s) {
                const size_t row = ((size_t)(m * S + s) * T + t) * N;
                const size_t dst = ((size_t)s * FT + (f - f0)) * N;
                bulk_g2s(ub + dst, p.u_fwd + row, (uint32_t)len * N * 4, &bars[st]);
                bulk_g2s(bb + dst, p.b_bwd + row, (uint32_t)len * N * 4, &bars[st]);
            }
            f += len;
        }
        bulk_g2s(sb + L.fc, p.fconst + 4 * (size_t)f0, (uint32_t)nf * 32, &bars[st]);
    };

    int it = 0;
    if (tid == 0 && (int)blockIdx.x < ntiles) issue(blockIdx.x, 0);
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
        const int st = it & 1;
        const uint32_t parity = (it >> 1) & 1;
        const int f0 = tile * FT, nf = min(FT, p.frames - f0);
        unsigned char *sb = smem_raw + st * L.stage;
        float *nb = reinterpret_cast<float *>(sb + L.n);
        const float *ub = reinterpret_cast<const float *>(sb + L.u);
        const float *bb = reinterpret_cast<const float *>(sb + L.b);
        const double *fc = reinterpret_cast<const double *>(sb + L.fc);
        // every thread is done with the other stage (tile it-1: its fc rows, the theta it stored):
        // refill it with the next tile once the bulk store out of it has read its bytes
        __syncthreads();
        if (tid == 0) {
            const int nt = tile + gridDim.x;
            if (nt < ntiles) {
                bulk_wait_read0();
                fence_async_smem();
                issue(nt, st ^ 1);
            }
        }
        mbar_wait(&bars[st], parity);

        // Eq. 6 normalisers: gq[f][s] = gamma / sum_n u b  (one thread per (frame, source))
        for (int k = tid; k < nf * S; k += NT) {
            const int f = divq(k, S, invS), s = k - f * S;
            const float *u = ub + ((size_t)s * FT + f) * N, *b = bb + ((size_t)s * FT + f) * N;
            float q0 = 0.f, q1 = 0.f;
            int n = 0;
            for (; n + 1 < N; n += 2) {
                q0 = fmaf(u[n], b[n], q0);
                q1 = fmaf(u[n + 1], b[n + 1], q1);
            }
            if (n < N) q0 = fmaf(u[n], b[n], q0);
            const float q = q0 + q1;
            if (!(q > 0.f) || !(q < INFINITY)) bad |= FLAG_NONFINITE;
            gq[k] = gamma * __frcp_rn(q);
        }
        __syncthreads();

        // element pass: one thread per (frame, block) item; theta replaces n in the stage buffer
        for (int i = tid; i < nf * SN; i += NT) {
            const int f = divq(i, SN, invSN), b = i - f * SN;
            const int s = divq(b, N, invN), n = b - s * N;
            const size_t ui = ((size_t)s * FT + f) * N + n;
            const float dv = fmaf(gq[f * S + s], ub[ui] * bb[ui], 1.f);
            const uint64_t e0_2 = f2c((float)fc[4 * f + 3]);
            float *arow = want_a ? p.alpha + (size_t)(f0 + f) * p.ld + b * K : nullptr;
            double ps;
            float gs;
            item_elements<KC>(nb + (size_t)f * Kt + b * K, K, dv, e0_2, want_h, arow, ps, gs);
            sps[i] = ps;
            hs[i] = gs;
        }
        fence_async_smem();   // theta (generic writes) before the bulk store (async proxy) reads it
        __syncthreads();
        if (tid == 0) {
            if (contiguous) {
                bulk_s2g(p.theta + (size_t)f0 * Kt, nb, (uint32_t)nf * Kt * 4);
            } else {
                for (int f = 0; f < nf; ++f) bulk_s2g(p.theta + (size_t)(f0 + f) * p.ld, nb + (size_t)f * Kt, Kt * 4);
            }
            bulk_commit();
        }
        // Eq. 8 maxima and offsets, one thread per (frame, source); the bound term, one warp per frame
        for (int k = tid; k < nf * S; k += NT) {
            const int f = divq(k, S, invS), s = k - f * S;
            const double *v = sps + (size_t)f * SN + s * N;
            float m0 = -INFINITY, m1 = -INFINITY;
            int n = 0;
            for (; n + 1 < N; n += 2) {
                m0 = fmaxf(m0, (float)v[n]);
                m1 = fmaxf(m1, (float)v[n + 1]);
            }
            if (n < N) m0 = fmaxf(m0, (float)v[n]);
            const float mxf = fmaxf(m0, m1);
            mxs[k] = mxf;
            const int fg = f0 + f, m = fg / T, t = fg - m * T;
            const double off = (double)gamma * ((double)mxf - (double)K * fc[4 * f + 1]);
            p.eoff[(size_t)(m * S + s) * T + t] = off;
            if (!isfinite(off)) bad |= FLAG_NONFINITE;
        }
        if (want_h) {
            for (int f = warp; f < nf; f += NT / 32) {
                float h = 0.f;
                for (int b = lane; b < SN; b += 32) h += hs[(size_t)f * SN + b];
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) h += __shfl_xor_sync(0xffffffffu, h, o);
                if (lane == 0) p.hdir[f0 + f] = (double)h + fc[4 * f + 2];
            }
        }
        __syncthreads();
        // emissions e = exp(gamma (phi - max)) in (0, 1], one thread per (frame, block)
        for (int i = tid; i < nf * SN; i += NT) {
            const int f = divq(i, SN, invSN), b = i - f * SN;
            const int s = divq(b, N, invN), n = b - s * N;
            const int fg = f0 + f, m = fg / T, t = fg - m * T;
            const double mx = (double)mxs[f * S + s];
            p.ec[((size_t)(m * S + s) * T + t) * N + n] =
                ex2_sfu((float)((double)gamma * (sps[i] - mx)) * 1.44269504088896341f);
        }
    }
    if (tid == 0) bulk_wait0();   // the last theta store has landed before the kernel retires
    if (bad) atomicOr(p.flags, bad);
}

struct RingPick {
    int FT, nt;
};

// Tile shape: FT frames x (threads) with FT*S*N a multiple of the thread count (equal items per thread),
// a stage of at most ~40 KB (two stages + sums: three CTAs per SM) or, for long rows, one frame per stage.
RingPick ring_pick(int S, int N, int Kt) {
    const int SN = S * N;
    RingPick best{0, 0};
    double best_score = -1.0;
    for (int nt = 128; nt <= 256; nt += 32) {
        for (int FT = 1; FT <= 64; ++FT) {
            const RingLayout L(S, N, Kt, FT);
            if (L.total > 110 * 1024) break;
            const int items = FT * SN;
            const int per = (items + nt - 1) / nt;
            const double eff = (double)items / ((double)per * nt);   // lane utilisation of the element pass
            const int ctas = (int)((227 * 1024) / (L.total + 1024));
            const int warps = ctas * nt / 32 > 64 ? 64 : ctas * nt / 32;
            if (ctas < 1) continue;
            // prefer full lanes, then resident warps per SM (latency hiding of the element chains), then
            // bigger tiles (fewer barriers per frame)
            const double score = eff * 100.0 + 0.5 * (warps < 24 ? warps : 24) + (FT >= 4 ? 1.0 : 0.25 * FT) +
                                 (ctas >= 2 ? 2.0 : 0.0);
            if (score > best_score + 1e-9) {
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
    const RingPick pk = ring_pick(a.S, a.N, a.Kt);
    if (pk.FT < 1) return cudaErrorInvalidValue;
    if (a.K == 10) return launch_ring_k<10>(a, pk.FT, pk.nt, st);
    if (a.K == 20) return launch_ring_k<20>(a, pk.FT, pk.nt, st);
    return launch_ring_k<0>(a, pk.FT, pk.nt, st);
}

}  // namespace nfk
