// fb.cu -- kernel (e): scaled forward-backward per source chain, batched over all mixtures.
//
// q(D^(s)) is the chain posterior with log-likelihood gamma * phi (DESIGN R1).  One warp
// per chain (m, s); lane l owns states j = l + 32 q (q < NQ).  The recursion is latency-bound (2T
// dependent steps per chain), so each step is built to be short:
//   * A_s (row-stochastic, A[i][j] = P(j | i), DESIGN R4) lives in REGISTERS for N <= 64 (lane j holds
//     column j for the forward pass, row j for the backward pass), zero-padded to a compile-time NMAX
//     so the dot products are fully unrolled with 4 independent FMA chains per state;
//     for 64 < N <= 128 it is read from shared memory in the same unrolled pattern;
//   * the previous message is broadcast through shared memory with 128-bit loads;
//   * the normaliser is deferred:  u_0 = pi .* e_0;  w_t = (u_{t-1} A) .* e_t;  c_{t-1} = sum u_{t-1};
//     u_t = w_t / c_{t-1}  -- the warp reduction for c_{t-1} runs alongside the dot product;
//     a_{t-1} = u_{t-1} / c_{t-1} is the normalised message (stored for the backward pass);
//     log Z = sum_t log c_t + sum_t eoff_t (FP64; the product of c_t kept as mantissa * 2^exponent);
//   * backward: b_{T-1} = 1;  b_t = A (e_{t+1} .* b_{t+1}) / c_{t+1};  d_t = a_t .* b_t / sum;
//   * emissions e = exp(ec) (ec <= 0: the centred gamma*phi from the Dirichlet kernel) and the stored
//     messages are staged CH steps ahead into shared memory with cp.async (double-buffered chunks).
#include <cuda_runtime.h>
#include <math.h>

#include "nfhmm_internal.cuh"

namespace nfk {

namespace {

template <int NMAX>
struct FBCfg {
    static constexpr int WPB = NMAX <= 64 ? 4 : 2;  // chains (warps) per CTA, sharing the CTA's copy of A_s
    static constexpr int NQ = (NMAX + 31) / 32;
    static constexpr bool REG = NMAX <= 64;        // A in registers
    static constexpr int CH = NMAX <= 64 ? 32 : 16; // time steps per staged chunk
};

__device__ __forceinline__ void cp_async4(float *smem_dst, const float *gsrc) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem_dst);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(s), "l"(gsrc));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::); }

// Stage rows [t0, t0 + n) of a [T][W] array into dst[n][W] (warp-cooperative, async).
__device__ __forceinline__ void stage_rows(float *dst, const float *src, int W, int t0, int n, int lane) {
    const int cnt = n * W;
    const float *s = src + (size_t)t0 * W;
    for (int i = lane; i < cnt; i += 32) cp_async4(dst + i, s + i);
    cp_async_commit();
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// acc[q] = sum_i x[i] * M(i, j_q) over i < NMAX, x broadcast from shared memory (zero-padded).
// REG: M(i, j_q) = reg[q][i];  else M(i, j_q) = Ms[i * NMAX + j_q].
template <int NMAX, int RQ, int RN>
__device__ __forceinline__ void dot_bcast(float (&acc)[FBCfg<NMAX>::NQ], const float *x, const float (&reg)[RQ][RN],
                                          const float *Ms, const int (&js)[FBCfg<NMAX>::NQ]) {
    constexpr int NQ = FBCfg<NMAX>::NQ;
    float a[NQ][4];
#pragma unroll
    for (int q = 0; q < NQ; ++q) a[q][0] = a[q][1] = a[q][2] = a[q][3] = 0.f;
    const float4 *x4 = reinterpret_cast<const float4 *>(x);
#pragma unroll
    for (int i4 = 0; i4 < NMAX / 4; ++i4) {
        const float4 v = x4[i4];
        const float xv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            const int i = 4 * i4 + r;
#pragma unroll
            for (int q = 0; q < NQ; ++q) {
                const float m = FBCfg<NMAX>::REG ? reg[RQ > 1 ? q : 0][RN > 1 ? i : 0] : Ms[i * NMAX + js[q]];
                a[q][r] = fmaf(xv[r], m, a[q][r]);
            }
        }
    }
#pragma unroll
    for (int q = 0; q < NQ; ++q) acc[q] = (a[q][0] + a[q][1]) + (a[q][2] + a[q][3]);
}

template <int NMAX>
__global__ void __launch_bounds__(FBCfg<NMAX>::WPB * 32) fb_kernel(FBArgs p) {
    constexpr int WPB = FBCfg<NMAX>::WPB;
    constexpr int NQ = FBCfg<NMAX>::NQ;
    constexpr int CH = FBCfg<NMAX>::CH;
    constexpr bool REG = FBCfg<NMAX>::REG;
    extern __shared__ __align__(16) float sm[];
    const int N = p.N;
    float *As = sm;                       // [NMAX][NMAX]  As[i][j] = A[i][j]  (zero-padded)
    float *AT = As + NMAX * NMAX;         // [NMAX][NMAX]  AT[j][i] = A[i][j]
    float *wbase = AT + NMAX * NMAX;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // per warp: u[2][NMAX] | e chunks [2][CH][N] | a chunks [2][CH][N] | cinv chunks [2][CH]
    const int per_warp = 2 * NMAX + 4 * CH * N + 2 * CH;
    float *ubuf = wbase + warp * per_warp;
    float *ech = ubuf + 2 * NMAX;
    float *ach = ech + 2 * CH * N;
    float *cch = ach + 2 * CH * N;

    const int s = blockIdx.y;
    const int m = blockIdx.x * WPB + warp;
    const float *Ag = p.trans + (size_t)s * N * N;
    for (int idx = threadIdx.x; idx < NMAX * NMAX; idx += blockDim.x) {
        const int r = idx / NMAX, c = idx - r * NMAX;
        const float v = (r < N && c < N) ? Ag[r * N + c] : 0.f;
        As[idx] = v;
        AT[c * NMAX + r] = v;
    }
    for (int idx = lane; idx < 2 * NMAX; idx += 32) ubuf[idx] = 0.f;
    __syncthreads();
    if (m >= p.M) return;

    const int T = p.T;
    const size_t chain = (size_t)m * p.S + s;
    const float *ec = p.ec + chain * T * N;
    float *fwd = p.fwd + chain * T * N;
    float *cinv = p.cinv + chain * T;
    float *dh = p.d_hat + chain * T * N;
    unsigned bad = 0;

    int js[NQ];
    bool jv[NQ];
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
        js[q] = lane + 32 * q;
        jv[q] = js[q] < N;
    }
    float Areg[REG ? NQ : 1][REG ? NMAX : 1];
    if (REG) {   // forward: column j_q of A
#pragma unroll
        for (int q = 0; q < NQ; ++q)
#pragma unroll
            for (int i = 0; i < NMAX; ++i) Areg[q][i] = js[q] < NMAX ? As[i * NMAX + js[q]] : 0.f;
    }

    // sum of the FP64 emission offsets (lane-parallel, fixed order)
    double offsum = 0.0;
    for (int t = lane; t < T; t += 32) offsum += p.eoff[chain * T + t];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) offsum += __shfl_xor_sync(0xffffffffu, offsum, o);

    // ---------------- forward ----------------
    const int nch = (T + CH - 1) / CH;
    stage_rows(ech, ec, N, 0, min(CH, T), lane);
    double mant = 1.0;   // running product of c_t as mantissa * 2^expo (FP64)
    long long expo = 0;
    float u[NQ];
    for (int c = 0; c < nch; ++c) {
        const int t0 = c * CH, n = min(CH, T - t0);
        const float *ecur = ech + (c & 1) * CH * N;
        cp_async_wait_all();
        __syncwarp();
        if (c + 1 < nch) stage_rows(ech + ((c + 1) & 1) * CH * N, ec, N, t0 + CH, min(CH, T - t0 - CH), lane);
        for (int tt = 0; tt < n; ++tt) {
            const int t = t0 + tt;
            float e[NQ];
#pragma unroll
            for (int q = 0; q < NQ; ++q) e[q] = jv[q] ? expf(ecur[tt * N + js[q]]) : 0.f;
            if (t == 0) {
#pragma unroll
                for (int q = 0; q < NQ; ++q) u[q] = jv[q] ? p.prior[s * N + js[q]] * e[q] : 0.f;
            } else {
                float acc[NQ];
                dot_bcast<NMAX>(acc, ubuf + ((t - 1) & 1) * NMAX, Areg, As, js);
                // c_{t-1} from the previous (unnormalised) message, reduced alongside the dot product
                float ps = 0.f;
#pragma unroll
                for (int q = 0; q < NQ; ++q) ps += u[q];
                const float ct = warp_sum(ps);
                const float ic = 1.f / ct;
                if (!(ct > 0.f)) bad |= FLAG_NONFINITE;
#pragma unroll
                for (int q = 0; q < NQ; ++q)
                    if (jv[q]) fwd[(size_t)(t - 1) * N + js[q]] = u[q] * ic;
                if (lane == 0) {
                    cinv[t - 1] = ic;
                    int ex;
                    mant = frexp(mant * (double)ct, &ex);
                    expo += ex;
                }
#pragma unroll
                for (int q = 0; q < NQ; ++q) u[q] = acc[q] * e[q] * ic;
            }
            float *un = ubuf + (t & 1) * NMAX;
#pragma unroll
            for (int q = 0; q < NQ; ++q)
                if (jv[q]) un[js[q]] = u[q];
            __syncwarp();
        }
    }
    {   // last step's normaliser
        float ps = 0.f;
#pragma unroll
        for (int q = 0; q < NQ; ++q) ps += u[q];
        const float ct = warp_sum(ps);
        const float ic = 1.f / ct;
        if (!(ct > 0.f)) bad |= FLAG_NONFINITE;
#pragma unroll
        for (int q = 0; q < NQ; ++q)
            if (jv[q]) fwd[(size_t)(T - 1) * N + js[q]] = u[q] * ic;
        if (lane == 0) {
            cinv[T - 1] = ic;
            int ex;
            mant = frexp(mant * (double)ct, &ex);
            expo += ex;
            const double lz = log(mant) + (double)expo * 0.69314718055994530942 + offsum;
            p.logZ[chain] = lz;
            if (!isfinite(lz)) bad |= FLAG_NONFINITE;
        }
    }
    __threadfence_block();
    __syncwarp();

    // ---------------- backward ----------------
    if (REG) {   // backward: row j_q of A  (b_t[j] = sum_k A[j][k] x[k])
#pragma unroll
        for (int q = 0; q < NQ; ++q)
#pragma unroll
            for (int k = 0; k < NMAX; ++k) Areg[q][k] = js[q] < NMAX ? AT[k * NMAX + js[q]] : 0.f;
    }
    float b[NQ];
#pragma unroll
    for (int q = 0; q < NQ; ++q) b[q] = 1.f;
    // chunk c covers t in [t0, t0 + n), processed in descending t; needs e_{t+1}, cinv_{t+1}, a_t
    auto stage_back = [&](int cc, int buf) {
        const int t0 = cc * CH, n = min(CH, T - t0);
        stage_rows(ach + buf * CH * N, fwd, N, t0, n, lane);
        const int ne = min(n, T - 1 - t0);   // rows t0+1 .. t0+ne
        if (ne > 0) {
            stage_rows(ech + buf * CH * N, ec, N, t0 + 1, ne, lane);
            stage_rows(cch + buf * CH, cinv, 1, t0 + 1, ne, lane);
        }
    };
    stage_back(nch - 1, (nch - 1) & 1);
    for (int c = nch - 1; c >= 0; --c) {
        const int t0 = c * CH, n = min(CH, T - t0);
        const int buf = c & 1;
        const float *acur = ach + buf * CH * N;
        const float *ecur = ech + buf * CH * N;   // row r holds e_{t0 + 1 + r}
        const float *ccur = cch + buf * CH;       // ccur[r] = cinv_{t0 + 1 + r}
        cp_async_wait_all();
        __syncwarp();
        if (c > 0) stage_back(c - 1, buf ^ 1);
        for (int tt = n - 1; tt >= 0; --tt) {
            const int t = t0 + tt;
            if (t < T - 1) {
                float *xb = ubuf + (t & 1) * NMAX;
#pragma unroll
                for (int q = 0; q < NQ; ++q)
                    if (jv[q]) xb[js[q]] = expf(ecur[tt * N + js[q]]) * b[q];
                __syncwarp();
                float acc[NQ];
                dot_bcast<NMAX>(acc, xb, Areg, AT, js);
                const float ic = ccur[tt];
#pragma unroll
                for (int q = 0; q < NQ; ++q) b[q] = acc[q] * ic;
            }
            float dv[NQ];
            float ps = 0.f;
#pragma unroll
            for (int q = 0; q < NQ; ++q) {
                dv[q] = jv[q] ? acur[tt * N + js[q]] * b[q] : 0.f;
                ps += dv[q];
            }
            const float z = warp_sum(ps);
            const float iz = 1.f / z;
            if (!(z > 0.f)) bad |= FLAG_NONFINITE;
#pragma unroll
            for (int q = 0; q < NQ; ++q)
                if (jv[q]) dh[(size_t)t * N + js[q]] = dv[q] * iz;
        }
    }
    if (bad) atomicOr(p.flags, bad);
}

template <int NMAX>
cudaError_t launch_fb_t(const FBArgs &a, cudaStream_t st) {
    const int N = a.N;
    constexpr int CH = FBCfg<NMAX>::CH;
    constexpr int WPB = FBCfg<NMAX>::WPB;
    const size_t smem = ((size_t)2 * NMAX * NMAX + (size_t)WPB * (2 * NMAX + 4 * CH * N + 2 * CH)) * sizeof(float);
    static size_t attr = 0;
    if (smem > 48 * 1024 && attr < smem) {
        cudaError_t e = cudaFuncSetAttribute(fb_kernel<NMAX>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        attr = smem;
    }
    dim3 grid((a.M + WPB - 1) / WPB, a.S);
    fb_kernel<NMAX><<<grid, WPB * 32, smem, st>>>(a);
    return cudaGetLastError();
}

}  // namespace

cudaError_t launch_fb(const FBArgs &a, cudaStream_t st) {
    const int N = a.N;
    if (N <= 8) return launch_fb_t<8>(a, st);
    if (N <= 16) return launch_fb_t<16>(a, st);
    if (N <= 24) return launch_fb_t<24>(a, st);
    if (N <= 32) return launch_fb_t<32>(a, st);
    if (N <= 40) return launch_fb_t<40>(a, st);
    if (N <= 48) return launch_fb_t<48>(a, st);
    if (N <= 64) return launch_fb_t<64>(a, st);
    if (N <= 96) return launch_fb_t<96>(a, st);
    if (N <= 128) return launch_fb_t<128>(a, st);
    return cudaErrorInvalidValue;
}

}  // namespace nfk
