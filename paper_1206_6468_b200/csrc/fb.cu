// fb.cu -- kernel (e): scaled forward-backward per source chain, batched over all mixtures.
//
// q(D^(s)) is the chain posterior with log-likelihood gamma * phi (DESIGN R1).  The two
// recursions are independent -- the backward messages b_t never read the forward messages u_t, only the
// marginals d_t ~ u_t .* b_t combine them -- so each chain gets TWO warps that run concurrently: warp 2c
// the forward pass, warp 2c+1 the backward pass.  Both store their messages and the consumers (the
// Dirichlet kernel, nfhmm_posteriors) form d_t = u_t .* b_t / sum_n(u_t .* b_t).
//
// Each recursion is latency-bound (T dependent steps), so one step is kept to: broadcast the previous
// message through shared memory (128-bit loads) -> unrolled dot products in packed FP32 pairs (FFMA2) ->
// one multiply -> store; no division, no FP64 and no warp reduction inside the loop.  Lane l owns states
// 32 q + l, q < ceil(NMAX / 32) (for N = 40: 2 x 20 FFMA2 per lane per step).  Splitting the N % 32
// remainder states over lane groups (fewer FMAs, a shuffle butterfly per step) measured ~1.7x slower.
// A_s (row-stochastic, A[i][j] = P(j | i), DESIGN R4) lives in registers when it fits (columns for the
// forward pass, rows for the backward pass), else is read from shared memory in the same pattern.
// Scaling is by exact powers of two: every lane also sums the broadcast vector it loads, and the next
// message is multiplied by 2^-E with E the binary exponent of that sum:
//   u_0 = pi .* e_0;   u_t = ((u_{t-1} A) .* e_t) 2^-E_t,  E_t = exponent(sum u_{t-1});
//   log Z = ln(sum u_{T-1}) + ln 2 * sum_t E_t + sum_t eoff_t   (FP64, after the loop);
//   b_{T-1} = 1;  x_t = e_{t+1} .* b_{t+1};  b_t = (A x_t) 2^-E'_t,  E'_t = exponent(sum x_t).
// Emissions e = exp(gamma (phi - max_n phi)) in (0, 1] come precomputed from the Dirichlet kernel; eoff
// are their FP64 per-frame offsets.  The emissions of the next CH steps are staged into shared memory
// with cp.async (double-buffered chunks).
#include <cuda_runtime.h>
#include <math.h>

#include "nfhmm_internal.cuh"

namespace nfk {

namespace {

template <int NMAX>
struct FBCfg {
    static constexpr int NQ = (NMAX + 31) / 32;       // rounds of 32 states per lane
    static constexpr bool REG = NQ * NMAX <= 96;      // A (packed pairs) in registers
    static constexpr int CPB = REG ? 2 : 1;           // chains per CTA (2 warps each)
    static constexpr int WPB = 2 * CPB;
    static constexpr int CH = NMAX <= 64 ? 32 : 16;   // time steps per staged chunk
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

// Packed FP32 pairs (sm_100 FFMA2 / FADD2: two FP32 lanes per instruction, each IEEE round-to-nearest).
__device__ __forceinline__ uint64_t pk2(float a, float b) {
    uint64_t r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
    return r;
}
__device__ __forceinline__ void fma2(uint64_t &d, uint64_t a, uint64_t b) {
    asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(d) : "l"(a), "l"(b));
}
__device__ __forceinline__ void add2(uint64_t &d, uint64_t a) { asm("add.rn.f32x2 %0, %1, %0;" : "+l"(d) : "l"(a)); }
__device__ __forceinline__ float hsum2(uint64_t v) {
    float a, b;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v));
    return a + b;
}

// One message step.  x: broadcast vector in shared memory (NMAX floats, zero-padded).
//   out[q] = sum_i x[i] M(i, 32 q + lane),  xsum = sum_i x[i] (every lane, from the values it loads)
// M(i, j): packed register pairs Mr[q][i/2] = (M(i, j), M(i+1, j)), or shared Ms[i * NMAX + j].
template <int NMAX>
__device__ __forceinline__ void step_products(float (&out)[FBCfg<NMAX>::NQ], float &xsum, const float *x,
                                              const uint64_t (&Mr)[FBCfg<NMAX>::REG ? FBCfg<NMAX>::NQ : 1][FBCfg<NMAX>::REG ? NMAX / 2 : 1],
                                              const float *Ms, int lane) {
    using C = FBCfg<NMAX>;
    constexpr int NQ = C::NQ;
    uint64_t a[NQ][2];
    uint64_t s2[2] = {0ull, 0ull};
#pragma unroll
    for (int q = 0; q < NQ; ++q) a[q][0] = a[q][1] = 0ull;
    const ulonglong2 *x4 = reinterpret_cast<const ulonglong2 *>(x);
#pragma unroll
    for (int i4 = 0; i4 < NMAX / 4; ++i4) {
        const ulonglong2 v = x4[i4];   // (x[4i4], x[4i4+1]) | (x[4i4+2], x[4i4+3])
        add2(s2[0], v.x);
        add2(s2[1], v.y);
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
            uint64_t m0, m1;
            if (C::REG) {
                m0 = Mr[C::REG ? q : 0][C::REG ? 2 * i4 : 0];
                m1 = Mr[C::REG ? q : 0][C::REG ? 2 * i4 + 1 : 0];
            } else {
                const int j = min(32 * q + lane, NMAX - 1), i = 4 * i4;   // (lanes past NMAX: discarded)
                m0 = pk2(Ms[i * NMAX + j], Ms[(i + 1) * NMAX + j]);
                m1 = pk2(Ms[(i + 2) * NMAX + j], Ms[(i + 3) * NMAX + j]);
            }
            fma2(a[q][0], v.x, m0);
            fma2(a[q][1], v.y, m1);
        }
    }
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
        add2(a[q][0], a[q][1]);
        out[q] = hsum2(a[q][0]);
    }
    add2(s2[0], s2[1]);
    xsum = hsum2(s2[0]);
}

template <int NMAX>
__global__ void __launch_bounds__(FBCfg<NMAX>::WPB * 32) fb_kernel(FBArgs p) {
    using C = FBCfg<NMAX>;
    constexpr int CPB = C::CPB, NQ = C::NQ, CH = C::CH;
    constexpr bool REG = C::REG;
    extern __shared__ __align__(16) float sm[];
    const int N = p.N;
    float *As = sm;                       // [NMAX][NMAX]  As[i][j] = A[i][j]  (zero-padded)
    float *AT = As + NMAX * NMAX;         // [NMAX][NMAX]  AT[j][i] = A[i][j]
    float *wbase = AT + NMAX * NMAX;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const bool backward = warp & 1;
    // per warp: message broadcast buffer [2][NMAX] | emission chunks [2][CH][N]
    const int per_warp = 2 * NMAX + 2 * CH * N;
    float *ubuf = wbase + warp * per_warp;
    float *ech = ubuf + 2 * NMAX;

    const int s = blockIdx.y;
    const int m = blockIdx.x * CPB + (warp >> 1);
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
    unsigned bad = 0;
    bool jv[NQ];
#pragma unroll
    for (int q = 0; q < NQ; ++q) jv[q] = 32 * q + lane < N;

    // forward: columns of A; backward: b_t[j] = sum_k A[j][k] x[k] = sum_k AT[k][j] x[k]
    const float *M = backward ? AT : As;
    uint64_t Mr[REG ? NQ : 1][REG ? NMAX / 2 : 1];
    if (REG) {
#pragma unroll
        for (int q = 0; q < NQ; ++q)
#pragma unroll
            for (int i = 0; i < NMAX; i += 2)
                Mr[REG ? q : 0][REG ? i / 2 : 0] =
                    32 * q + lane < NMAX ? pk2(M[i * NMAX + 32 * q + lane], M[(i + 1) * NMAX + 32 * q + lane]) : 0ull;
    }
    const int nch = (T + CH - 1) / CH;

    if (!backward) {
        // ---------------- forward: u_t -> p.fwd, log Z ----------------
        float *fwd = p.fwd + chain * T * N;
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
                const float *et = ecur + tt * N;
                if (t == 0) {
#pragma unroll
                    for (int q = 0; q < NQ; ++q) u[q] = jv[q] ? p.prior[s * N + 32 * q + lane] * et[32 * q + lane] : 0.f;
                } else {
                    float acc[NQ], usum;
                    step_products<NMAX>(acc, usum, ubuf + ((t - 1) & 1) * NMAX, Mr, M, lane);
                    if (!(usum > 0.f) || !(usum < INFINITY)) bad |= FLAG_NONFINITE;
                    const int E = exponent_of(usum);
                    const float sc = pow2_neg(E);
                    esum += E;
#pragma unroll
                    for (int q = 0; q < NQ; ++q) u[q] = jv[q] ? acc[q] * et[32 * q + lane] * sc : 0.f;
                }
                float *un = ubuf + (t & 1) * NMAX;
#pragma unroll
                for (int q = 0; q < NQ; ++q) {
                    if (jv[q]) {
                        un[32 * q + lane] = u[q];
                        fwd[(size_t)t * N + 32 * q + lane] = u[q];
                    }
                }
                __syncwarp();
            }
        }
        float part = 0.f;
#pragma unroll
        for (int q = 0; q < NQ; ++q) part += u[q];
        const float usum = warp_sum(part);
        if (!(usum > 0.f) || !(usum < INFINITY)) bad |= FLAG_NONFINITE;
        double offsum = 0.0;   // lane-parallel, fixed order
        for (int t = lane; t < T; t += 32) offsum += p.eoff[chain * T + t];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) offsum += __shfl_xor_sync(0xffffffffu, offsum, o);
        if (lane == 0) {
            const double lz = log((double)usum) + (double)esum * 0.69314718055994530942 + offsum;
            p.logZ[chain] = lz;
            if (!isfinite(lz)) bad |= FLAG_NONFINITE;
        }
    } else {
        // ---------------- backward: b_t -> p.bwd ----------------
        float *bwd = p.bwd + chain * T * N;
        float b[NQ];
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
            b[q] = jv[q] ? 1.f : 0.f;
            if (jv[q]) bwd[(size_t)(T - 1) * N + 32 * q + lane] = 1.f;
        }
        // chunk c covers x_t for t in [t0, t0 + n) in descending t: needs e_{t+1}, rows t0+1 .. t0+n
        auto stage_back = [&](int cc, int buf) {
            const int t0 = cc * CH, ne = min(CH, T - 1 - t0);
            stage_rows(ech + buf * CH * N, em, N, t0 + 1, ne, lane);
        };
        const int ncb = (T - 1 + CH - 1) / CH;   // chunks of t in [0, T-1)
        if (ncb > 0) stage_back(ncb - 1, (ncb - 1) & 1);
        for (int c = ncb - 1; c >= 0; --c) {
            const int t0 = c * CH, n = min(CH, T - 1 - t0);
            const int buf = c & 1;
            const float *ecur = ech + buf * CH * N;   // row r holds e_{t0 + 1 + r}
            cp_async_wait_all();
            __syncwarp();
            if (c > 0) stage_back(c - 1, buf ^ 1);
            for (int tt = n - 1; tt >= 0; --tt) {
                const int t = t0 + tt;
                const float *en = ecur + tt * N;
                float *xb = ubuf + (t & 1) * NMAX;
#pragma unroll
                for (int q = 0; q < NQ; ++q)
                    if (jv[q]) xb[32 * q + lane] = en[32 * q + lane] * b[q];
                __syncwarp();
                float acc[NQ], xsum;
                step_products<NMAX>(acc, xsum, xb, Mr, M, lane);
                if (!(xsum > 0.f) || !(xsum < INFINITY)) bad |= FLAG_NONFINITE;
                const float sc = pow2_neg(exponent_of(xsum));
#pragma unroll
                for (int q = 0; q < NQ; ++q) {
                    b[q] = jv[q] ? acc[q] * sc : 0.f;
                    if (jv[q]) bwd[(size_t)t * N + 32 * q + lane] = b[q];
                }
            }
        }
    }
    if (bad) atomicOr(p.flags, bad);
}

template <int NMAX>
cudaError_t launch_fb_t(const FBArgs &a, cudaStream_t st) {
    using C = FBCfg<NMAX>;
    const int N = a.N;
    const size_t smem = ((size_t)2 * NMAX * NMAX + (size_t)C::WPB * (2 * NMAX + 2 * C::CH * N)) * sizeof(float);
    static size_t attr = 0;
    if (smem > 48 * 1024 && attr < smem) {
        cudaError_t e = cudaFuncSetAttribute(fb_kernel<NMAX>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        attr = smem;
    }
    dim3 grid((a.M + C::CPB - 1) / C::CPB, a.S);
    fb_kernel<NMAX><<<grid, C::WPB * 32, smem, st>>>(a);
    return cudaGetLastError();
}

}  // namespace

cudaError_t launch_fb(const FBArgs &a, cudaStream_t st) {
    const int N = a.N;
    if (N <= 4) return launch_fb_t<4>(a, st);
    if (N <= 8) return launch_fb_t<8>(a, st);
    if (N <= 16) return launch_fb_t<16>(a, st);
    if (N <= 24) return launch_fb_t<24>(a, st);
    if (N <= 32) return launch_fb_t<32>(a, st);
    if (N <= 40) return launch_fb_t<40>(a, st);
    if (N <= 48) return launch_fb_t<48>(a, st);
    if (N <= 64) return launch_fb_t<64>(a, st);
    if (N <= 96) return launch_fb_t<96>(a, st);
    if (N <= 104) return launch_fb_t<104>(a, st);
    if (N <= 128) return launch_fb_t<128>(a, st);
    return cudaErrorInvalidValue;
}

}  // namespace nfk
