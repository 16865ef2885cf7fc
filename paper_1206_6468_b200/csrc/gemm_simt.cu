// gemm_simt.cu -- FP32 SIMT (FFMA) contraction kernels of the VB sweep.
//
//   (a) recon:    V_hat[f, l] = sum_k theta[f, k] * beta_l(k)                 (Eq. 7 normaliser)
//                 epilogue: R = V / V_hat (0 where V = 0), FP64 partials of sum_l V log V_hat (the
//                 z-part of the bound, DESIGN R8), zero-support flag, optional V_hat store.
//                 Same mainloop with the RECON_SEPARATE epilogue gives Section 4's
//                 V_src^(s)[f, l] = (v_t / alpha_0) * sum_{k in s} alpha[f, k] beta_l(k).
//   (b) backproj: n[f, k] = theta[f, k] * sum_l R[f, l] * beta_l(k)            (Eq. 6 data term)
//
// Both are C[M x BNpad] = A[M x K] * B[K x BNpad] with A row-major (k contiguous) and B row-major
// (n contiguous).  Tiling: 128 x BN x 8 per CTA, BN = 8 * NTC chosen per shape so that F = 513
// pads to 520 (BN 104) and Kt = 800 is exact (BN 160); 16 x NTC threads, 8 x 8 outputs per thread
// split in two 4-wide halves (conflict-free float4 shared loads), register-staged double buffering
// with one __syncthreads per k-tile.  Rows beyond M are clamped on load and skipped on store; K is
// zero-padded to a multiple of 8 and N to a multiple of BN in every operand buffer, so the mainloop
// has no bounds checks except an optional [k_begin, k_end) window used by separation.
// Every output element is produced by one thread with a fixed k order: results are bitwise
// independent of the tile an element lands in (sharding invariance across ranks).
#include <cuda_runtime.h>
#include <math.h>

#include "nfhmm_internal.cuh"

namespace nfk {

namespace {

constexpr int BM = 128;
constexpr int BK = 8;
constexpr int AS = BM + 4;  // padded row of the transposed A tile (conflict-free transposed stores)

template <int NTC>
struct Cfg {
    static constexpr int BN = 8 * NTC;
    static constexpr int NT = 16 * NTC;
    static constexpr int NA = (BM * BK / 4 + NT - 1) / NT;  // float4 A loads per thread
    static constexpr int MINB = NT <= 224 ? 2 : 1;
};

template <int NTC>
struct Smem {
    float As[2][BK][AS];
    float Bs[2][BK][Cfg<NTC>::BN];
};

template <int NTC>
__device__ __forceinline__ void load_tile(const float *__restrict__ A, int lda, const float *__restrict__ B,
                                          int ldb, int M, int m0, int n0, int k0, int kb, int ke,
                                          float4 (&ra)[Cfg<NTC>::NA], float4 &rb) {
    const int tid = threadIdx.x;
    const bool edge = (k0 < kb) || (k0 + BK > ke);
#pragma unroll
    for (int i = 0; i < Cfg<NTC>::NA; ++i) {
        const int q = tid + i * Cfg<NTC>::NT;
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        if (q < BM * BK / 4) {
            const int row = q >> 1, c = (q & 1) * 4;
            const int grow = min(m0 + row, M - 1);
            v = __ldg(reinterpret_cast<const float4 *>(A + (size_t)grow * lda + k0 + c));
            if (edge) {
                const int kk = k0 + c;
                if (kk + 0 < kb || kk + 0 >= ke) v.x = 0.f;
                if (kk + 1 < kb || kk + 1 >= ke) v.y = 0.f;
                if (kk + 2 < kb || kk + 2 >= ke) v.z = 0.f;
                if (kk + 3 < kb || kk + 3 >= ke) v.w = 0.f;
            }
        }
        ra[i] = v;
    }
    {
        const int k = tid / (2 * NTC), c4 = tid % (2 * NTC);
        const int kk = k0 + k;
        rb = make_float4(0.f, 0.f, 0.f, 0.f);
        if (!edge || (kk >= kb && kk < ke))
            rb = __ldg(reinterpret_cast<const float4 *>(B + (size_t)kk * ldb + n0 + 4 * c4));
    }
}

template <int NTC>
__device__ __forceinline__ void store_tile(Smem<NTC> &sm, int buf, const float4 (&ra)[Cfg<NTC>::NA],
                                           const float4 &rb) {
    const int tid = threadIdx.x;
#pragma unroll
    for (int i = 0; i < Cfg<NTC>::NA; ++i) {
        const int q = tid + i * Cfg<NTC>::NT;
        if (q < BM * BK / 4) {
            const int row = q >> 1, c = (q & 1) * 4;
            sm.As[buf][c + 0][row] = ra[i].x;
            sm.As[buf][c + 1][row] = ra[i].y;
            sm.As[buf][c + 2][row] = ra[i].z;
            sm.As[buf][c + 3][row] = ra[i].w;
        }
    }
    const int k = tid / (2 * NTC), c4 = tid % (2 * NTC);
    *reinterpret_cast<float4 *>(&sm.Bs[buf][k][4 * c4]) = rb;
}

// acc[i][j]: row = m0 + (i < 4 ? 4*tr + i : 64 + 4*tr + i - 4), col = n0 + (j < 4 ? 4*tc + j : BN/2 + 4*tc + j - 4)
template <int NTC>
__device__ __forceinline__ void mainloop(float (&acc)[8][8], Smem<NTC> &sm, const float *__restrict__ A, int lda,
                                         const float *__restrict__ B, int ldb, int M, int m0, int n0, int kb,
                                         int ke) {
    constexpr int BN = Cfg<NTC>::BN;
    const int tid = threadIdx.x;
    const int tr = tid / NTC, tc = tid % NTC;
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = 0.f;

    const int kstart = kb & ~(BK - 1);
    const int ntiles = (ke - kstart + BK - 1) / BK;
    float4 ra[Cfg<NTC>::NA];
    float4 rb;
    load_tile<NTC>(A, lda, B, ldb, M, m0, n0, kstart, kb, ke, ra, rb);
    store_tile<NTC>(sm, 0, ra, rb);
    __syncthreads();
    for (int kt = 0; kt < ntiles; ++kt) {
        const int buf = kt & 1;
        if (kt + 1 < ntiles) load_tile<NTC>(A, lda, B, ldb, M, m0, n0, kstart + (kt + 1) * BK, kb, ke, ra, rb);
#pragma unroll
        for (int k = 0; k < BK; ++k) {
            const float4 a0 = *reinterpret_cast<const float4 *>(&sm.As[buf][k][4 * tr]);
            const float4 a1 = *reinterpret_cast<const float4 *>(&sm.As[buf][k][64 + 4 * tr]);
            const float4 b0 = *reinterpret_cast<const float4 *>(&sm.Bs[buf][k][4 * tc]);
            const float4 b1 = *reinterpret_cast<const float4 *>(&sm.Bs[buf][k][BN / 2 + 4 * tc]);
            const float a[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
            const float b[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
            for (int i = 0; i < 8; ++i)
#pragma unroll
                for (int j = 0; j < 8; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
        }
        if (kt + 1 < ntiles) store_tile<NTC>(sm, buf ^ 1, ra, rb);
        __syncthreads();
    }
}

__device__ __forceinline__ int row_of(int i, int tr) { return i < 4 ? 4 * tr + i : 64 + 4 * tr + (i - 4); }

template <int NTC>
__global__ void __launch_bounds__(Cfg<NTC>::NT, Cfg<NTC>::MINB) recon_kernel(ReconArgs p, int mode) {
    constexpr int BN = Cfg<NTC>::BN;
    __shared__ __align__(16) Smem<NTC> sm;
    __shared__ double red[BM][NTC];
    const int tid = threadIdx.x;
    const int tr = tid / NTC, tc = tid % NTC;
    const int ntile = blockIdx.x % p.n_tiles;
    const int mtile = blockIdx.x / p.n_tiles;
    const int m0 = mtile * BM, n0 = ntile * BN;

    float acc[8][8];
    mainloop<NTC>(acc, sm, p.A, p.lda, p.B, p.ldb, p.M, m0, n0, p.k_begin, p.k_end);

    if (mode == RECON_RATIO) {
        unsigned bad = 0;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const int r = m0 + row_of(i, tr);
            double part = 0.0;
            if (r < p.M) {
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int cb = n0 + h * (BN / 2) + 4 * tc;
                    const float4 v = *reinterpret_cast<const float4 *>(p.V + (size_t)r * p.ldv + cb);
                    const float vv[4] = {v.x, v.y, v.z, v.w};
                    float rr[4];
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        const float vh = acc[i][4 * h + j];
                        if (vv[j] > 0.f) {
                            if (vh > 0.f) {
                                rr[j] = vv[j] / vh;
                                part += rint((double)vv[j] * (double)logf(vh) * 1048576.0);   // 2^-20 nats (tc path)
                            } else {
                                rr[j] = 0.f;
                                bad |= FLAG_ZERO_SUPPORT;
                            }
                        } else {
                            rr[j] = 0.f;
                        }
                        if (p.Vhat && cb + j < p.F) p.Vhat[(size_t)r * p.F + cb + j] = vh;
                    }
                    *reinterpret_cast<float4 *>(p.R + (size_t)r * p.ldv + cb) = make_float4(rr[0], rr[1], rr[2], rr[3]);
                }
            }
            red[row_of(i, tr)][tc] = part;
        }
        if (bad) atomicOr(p.flags, bad);
        __syncthreads();
        for (int rl = tid; rl < BM; rl += Cfg<NTC>::NT) {   // NT may be < BM for narrow tiles
            const int r = m0 + rl;
            if (r < p.M) {
                double s = 0.0;
#pragma unroll 4
                for (int c = 0; c < NTC; ++c) s += red[rl][c];
                p.data_part[(size_t)r * p.n_tiles + ntile] = s;
            }
        }
    } else if (mode == RECON_STORE) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const int r = m0 + row_of(i, tr);
            if (r >= p.M) continue;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int cb = n0 + h * (BN / 2) + 4 * tc;
#pragma unroll
                for (int j = 0; j < 4; ++j)
                    if (cb + j < p.F) p.Vhat[(size_t)r * p.F + cb + j] = acc[i][4 * h + j];
            }
        }
    } else {  // RECON_SEPARATE
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const int r = m0 + row_of(i, tr);
            if (r >= p.M) continue;
            const float sc = p.row_scale[r];
            const int m = r / p.T, t = r - m * p.T;
            float *out = p.out_src + ((size_t)(m * p.S + p.s) * p.T + t) * p.F;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int cb = n0 + h * (BN / 2) + 4 * tc;
#pragma unroll
                for (int j = 0; j < 4; ++j)
                    if (cb + j < p.F) out[cb + j] = acc[i][4 * h + j] * sc;
            }
        }
    }
}

template <int NTC>
__global__ void __launch_bounds__(Cfg<NTC>::NT, Cfg<NTC>::MINB) backproj_kernel(BackprojArgs p, int n_tiles) {
    constexpr int BN = Cfg<NTC>::BN;
    __shared__ __align__(16) Smem<NTC> sm;
    const int tid = threadIdx.x;
    const int tr = tid / NTC, tc = tid % NTC;
    const int ntile = blockIdx.x % n_tiles;
    const int mtile = blockIdx.x / n_tiles;
    const int m0 = mtile * BM, n0 = ntile * BN;

    float acc[8][8];
    mainloop<NTC>(acc, sm, p.A, p.lda, p.B, p.ldb, p.M, m0, n0, 0, p.Kpad);

#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const int r = m0 + row_of(i, tr);
        if (r >= p.M) continue;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int cb = n0 + h * (BN / 2) + 4 * tc;
            const size_t off = (size_t)r * p.ldb + cb;
            const float4 th = *reinterpret_cast<const float4 *>(p.theta + off);
            float4 o;
            o.x = th.x * acc[i][4 * h + 0];
            o.y = th.y * acc[i][4 * h + 1];
            o.z = th.z * acc[i][4 * h + 2];
            o.w = th.w * acc[i][4 * h + 3];
            *reinterpret_cast<float4 *>(p.n_out + off) = o;
        }
    }
}

template <int NTC>
cudaError_t launch_recon_t(const ReconArgs &a, cudaStream_t st) {
    const int mt = (a.M + BM - 1) / BM;
    const long long grid = (long long)mt * a.n_tiles;
    recon_kernel<NTC><<<(unsigned)grid, Cfg<NTC>::NT, 0, st>>>(a, a.R ? RECON_RATIO : (a.out_src ? RECON_SEPARATE : RECON_STORE));
    return cudaGetLastError();
}

template <int NTC>
cudaError_t launch_backproj_t(const BackprojArgs &a, cudaStream_t st) {
    const int mt = (a.M + BM - 1) / BM;
    const int nt = a.ldb / Cfg<NTC>::BN;
    const long long grid = (long long)mt * nt;
    backproj_kernel<NTC><<<(unsigned)grid, Cfg<NTC>::NT, 0, st>>>(a, nt);
    return cudaGetLastError();
}

}  // namespace

#define NFHMM_BN_CASES(X) X(3) X(5) X(8) X(10) X(11) X(13) X(15) X(16) X(20)

cudaError_t launch_recon(int bn, const ReconArgs &a, cudaStream_t st) {
    switch (bn / 8) {
#define X(n) \
    case n:  \
        return launch_recon_t<n>(a, st);
        NFHMM_BN_CASES(X)
#undef X
        default:
            return cudaErrorInvalidValue;
    }
}

cudaError_t launch_backproj(int bn, const BackprojArgs &a, cudaStream_t st) {
    switch (bn / 8) {
#define X(n) \
    case n:  \
        return launch_backproj_t<n>(a, st);
        NFHMM_BN_CASES(X)
#undef X
        default:
            return cudaErrorInvalidValue;
    }
}

}  // namespace nfk
