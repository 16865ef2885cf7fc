// fb.cu -- kernel (e): scaled forward-backward per source chain, batched over all mixtures.
//
// q(D^(s)) is the chain posterior with log-likelihood gamma * phi (DESIGN R1).  One warp
// per chain (m, s); lane l owns states j = l + 32 q (q < NQ).  The recursion is latency-bound (2T
// dependent steps per chain), so a step is kept to: broadcast the previous message through shared
// memory (128-bit loads) -> fully unrolled dot products -> one multiply -> store.
//   * A_s (row-stochastic, A[i][j] = P(j | i), DESIGN R4) lives in REGISTERS for N <= 64 (lane j holds
//     column j for the forward pass, row j for the backward pass), zero-padded to a compile-time NMAX;
//     for 64 < N <= 128 it is read from shared memory in the same unrolled pattern.
//   * Scaling is by exact powers of two (no division, no FP64, no warp reduction on the critical path):
//     every lane also sums the broadcast message it just loaded, and the next message is multiplied by
//     2^-E with E the binary exponent of that sum.  Forward:
//       u_0 = pi .* e_0;   u_t = ((u_{t-1} A) .* e_t) 2^-E_t,  E_t = exponent(sum u_{t-1});
//       a_t = u_t / sum u_t (stored, off the critical path);
//       log Z = ln(sum u_{T-1}) + ln 2 * sum_t E_t + sum_t eoff_t   (FP64, after the loop).
//     Backward: b_{T-1} = 1;  b_t = (A (e_{t+1} .* b_{t+1})) 2^-E'_t;  d_t = a_t .* b_t / sum(a_t .* b_t).
//   * Emissions e = exp(gamma (phi - max_n phi)) in (0, 1] come precomputed from the Dirichlet kernel;
//     the eoff are their FP64 per-frame offsets.  Inputs for the next CH steps are staged into shared
//     memory with cp.async (double-buffered chunks).
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

// binary exponent E of x > 0 (x = m 2^E, m in [1, 2)) and the exact scale 2^-E
__device__ __forceinline__ int exponent_of(float x) { return (int)((__float_as_uint(x) >> 23) & 0xFF) - 127; }
__device__ __forceinline__ float pow2_neg(int E) { return __uint_as_float((uint32_t)(127 - E) << 23); }

// acc[q] = sum_i x[i] * M(i, j_q) over i < NMAX with x broadcast from shared memory (zero-padded), and
// xsum = sum_i x[i] (every lane computes it from the values it loaded).
template <int NMAX, int RQ, int RN>
__device__ __forceinline__ void dot_bcast(float (&acc)[FBCfg<NMAX>::NQ], float &xsum, const float *x,
                                          const float (&reg)[RQ][RN], const float *Ms,
                                          const int (&js)[FBCfg<NMAX>::NQ]) {
    constexpr int NQ = FBCfg<NMAX>::NQ;
    float a[NQ][4];
    float s4[4] = {0.f, 0.f, 0.f, 0.f};
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
            s4[r] += xv[r];
#pragma unroll
            for (int q = 0; q < NQ; ++q) {
                const float m = FBCfg<NMAX>::REG ? reg[RQ > 1 ? q : 0][RN > 1 ? i : 0] : Ms[i * NMAX + js[q]];
                a[q][r] = fmaf(xv[r], m, a[q][r]);
            }
        }
    }
#pragma unroll
    for (int q = 0; q < NQ; ++q) acc[q] = (a[q][0] + a[q][1]) + (a[q][2] + a[q][3]);
    xsum = (s4[0] + s4[1]) + (s4[2] + s4[3]);
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
    // per warp: u[2][NMAX] | e chunks [2][CH][N] | a chunks [2][CH][N]
    const int per_warp = 2 * NMAX + 4 * CH * N;
    float *ubuf = wbase + warp * per_warp;
    float *ech = ubuf + 2 * NMAX;
    float *ach = ech + 2 * CH * N;

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
    const float *em = p.ec + chain * T * N;     // emissions e_t(n)
    float *fwd = p.fwd + chain * T * N;
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

    // ---------------- forward ----------------
    const int nch = (T + CH - 1) / CH;
    stage_rows(ech, em, N, 0, min(CH, T), lane);
    float u[NQ];
    int esum = 0;            // sum of the power-of-two scale exponents applied
    for (int c = 0; c < nch; ++c) {
        const int t0 = c * CH, n = min(CH, T - t0);
        const float *ecur = ech + (c & 1) * CH * N;
        cp_async_wait_all();
        __syncwarp();
        if (c + 1 < nch) stage_rows(ech + ((c + 1) & 1) * CH * N, em, N, t0 + CH, min(CH, T - t0 - CH), lane);
        for (int tt = 0; tt < n; ++tt) {
            const int t = t0 + tt;
            if (t == 0) {
#pragma unroll
                for (int q = 0; q < NQ; ++q) u[q] = jv[q] ? p.prior[s * N + js[q]] * ecur[js[q]] : 0.f;
            } else {
                float acc[NQ], sprev;
                dot_bcast<NMAX>(acc, sprev, ubuf + ((t - 1) & 1) * NMAX, Areg, As, js);
                if (!(sprev > 0.f) || !(sprev < INFINITY)) bad |= FLAG_NONFINITE;
                const int E = exponent_of(sprev);
                const float sc = pow2_neg(E);
                esum += E;
                // off the critical path: the normalised message a_{t-1} for the backward pass
                const float inv = 1.f / sprev;
#pragma unroll
                for (int q = 0; q < NQ; ++q)
                    if (jv[q]) fwd[(size_t)(t - 1) * N + js[q]] = u[q] * inv;
#pragma unroll
                for (int q = 0; q < NQ; ++q) u[q] = jv[q] ? acc[q] * ecur[tt * N + js[q]] * sc : 0.f;
            }
            float *un = ubuf + (t & 1) * NMAX;
#pragma unroll
            for (int q = 0; q < NQ; ++q)
                if (jv[q]) un[js[q]] = u[q];
            __syncwarp();
        }
    }
    {   // last message and log Z
        float ps = 0.f;
#pragma unroll
        for (int q = 0; q < NQ; ++q) ps += u[q];
        const float sl = warp_sum(ps);
        if (!(sl > 0.f) || !(sl < INFINITY)) bad |= FLAG_NONFINITE;
        const float inv = 1.f / sl;
#pragma unroll
        for (int q = 0; q < NQ; ++q)
            if (jv[q]) fwd[(size_t)(T - 1) * N + js[q]] = u[q] * inv;
        double offsum = 0.0;   // lane-parallel, fixed order
        for (int t = lane; t < T; t += 32) offsum += p.eoff[chain * T + t];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) offsum += __shfl_xor_sync(0xffffffffu, offsum, o);
        if (lane == 0) {
            const double lz = log((double)sl) + (double)esum * 0.69314718055994530942 + offsum;
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
    // chunk c covers t in [t0, t0 + n), processed in descending t; needs e_{t+1} and a_t
    auto stage_back = [&](int cc, int buf) {
        const int t0 = cc * CH, n = min(CH, T - t0);
        stage_rows(ach + buf * CH * N, fwd, N, t0, n, lane);
        const int ne = min(n, T - 1 - t0);   // rows t0+1 .. t0+ne
        if (ne > 0) stage_rows(ech + buf * CH * N, em, N, t0 + 1, ne, lane);
    };
    stage_back(nch - 1, (nch - 1) & 1);
    for (int c = nch - 1; c >= 0; --c) {
        const int t0 = c * CH, n = min(CH, T - t0);
        const int buf = c & 1;
        const float *acur = ach + buf * CH * N;
        const float *ecur = ech + buf * CH * N;   // row r holds e_{t0 + 1 + r}
        cp_async_wait_all();
        __syncwarp();
        if (c > 0) stage_back(c - 1, buf ^ 1);
        for (int tt = n - 1; tt >= 0; --tt) {
            const int t = t0 + tt;
            if (t < T - 1) {
                float *xb = ubuf + (t & 1) * NMAX;
#pragma unroll
                for (int q = 0; q < NQ; ++q)
                    if (jv[q]) xb[js[q]] = ecur[tt * N + js[q]] * b[q];
                __syncwarp();
                float acc[NQ], xs;
                dot_bcast<NMAX>(acc, xs, xb, Areg, AT, js);
                if (!(xs > 0.f) || !(xs < INFINITY)) bad |= FLAG_NONFINITE;
                const float sc = pow2_neg(exponent_of(xs));
#pragma unroll
                for (int q = 0; q < NQ; ++q) b[q] = acc[q] * sc;
            }
            // off the critical path: d_t = a_t .* b_t / sum
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
    const size_t smem = ((size_t)2 * NMAX * NMAX + (size_t)WPB * (2 * NMAX + 4 * CH * N)) * sizeof(float);
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
