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
#include <limits.h>
#include <math.h>
#include <stdlib.h>

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
    // independent FFMA2 chains per output: the step is a latency chain, and 4 partial sums (5 dependent
    // FFMA2 each at N = 40) measured 24 % / 11 % faster than 2 at 64 / 256 mixtures (5: -18 %, 8: -12 %,
    // 10: as 4)
    constexpr int NA = 4;
    uint64_t a[NQ][NA];
    uint64_t s2[2] = {0ull, 0ull};
#pragma unroll
    for (int q = 0; q < NQ; ++q)
#pragma unroll
        for (int k = 0; k < NA; ++k) a[q][k] = 0ull;
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
            fma2(a[q][(2 * i4) % NA], v.x, m0);
            fma2(a[q][(2 * i4 + 1) % NA], v.y, m1);
        }
    }
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
#pragma unroll
        for (int k = 1; k < NA; ++k) add2(a[q][0], a[q][k]);
        out[q] = hsum2(a[q][0]);
    }
    add2(s2[0], s2[1]);
    xsum = hsum2(s2[0]);
}

// CHUNKED = false: one sequential pass over [0, T) per chain (compiled exactly for that case);
// CHUNKED = true: phase 3 of the parallel-in-time path -- one unit per (chain, time chunk), started from
// the exact chunk-start messages of fbp_scan_kernel.
template <int NMAX, bool CHUNKED>
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
    // unit = (mixture, chunk of the time axis); one chunk [0, T) unless the parallel-in-time path
    // (fbp_* kernels) supplies exact chunk-start messages
    const int unit = blockIdx.x * CPB + (warp >> 1);
    const int nchunk = CHUNKED ? p.nchunk : 1;
    const int m = CHUNKED ? unit / nchunk : unit, chunk = CHUNKED ? unit - m * nchunk : 0;
    const float *Ag = p.trans + (size_t)s * N * N;
    for (int idx = threadIdx.x; idx < NMAX * NMAX; idx += blockDim.x) {
        const int r = idx / NMAX, c = idx - r * NMAX;
        const float v = (r < N && c < N) ? Ag[r * N + c] : 0.f;
        As[idx] = v;
        AT[c * NMAX + r] = v;
    }
    for (int idx = lane; idx < 2 * NMAX; idx += 32) ubuf[idx] = 0.f;
    __syncthreads();
    if (m >= p.M) return;   // (unit beyond M * nchunk)

    const int T = p.T;
    const int ta = CHUNKED ? chunk * p.chunk_len : 0, tb = CHUNKED ? min(T, ta + p.chunk_len) : T;   // [ta, tb)
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
    const int nch = (tb - ta + CH - 1) / CH;

    if (!backward) {
        // ---------------- forward: u_t -> p.fwd, log Z ----------------
        float *fwd = p.fwd + chain * T * N;
        stage_rows(ech, em, N, ta, min(CH, tb - ta), lane);
        float u[NQ];
        int esum = 0;            // sum of the power-of-two scale exponents applied
        for (int c = 0; c < nch; ++c) {
            const int t0 = ta + c * CH, n = min(CH, tb - t0);
            const float *ecur = ech + (c & 1) * CH * N;
            cp_async_wait_all();
            __syncwarp();
            if (c + 1 < nch) stage_rows(ech + ((c + 1) & 1) * CH * N, em, N, t0 + CH, min(CH, tb - t0 - CH), lane);
            for (int tt = 0; tt < n; ++tt) {
                const int t = t0 + tt;
                const float *et = ecur + tt * N;
                if (t == ta) {
                    if (CHUNKED) {   // exact chunk-start message u_ta from the scan (fbp_scan_kernel)
                        const float *f0 = p.fstart + (chain * nchunk + chunk) * NMAX;
#pragma unroll
                        for (int q = 0; q < NQ; ++q) u[q] = jv[q] ? f0[32 * q + lane] : 0.f;
                    } else {
#pragma unroll
                        for (int q = 0; q < NQ; ++q) u[q] = jv[q] ? p.prior[s * N + 32 * q + lane] * et[32 * q + lane] : 0.f;
                    }
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
        if (CHUNKED) goto done;   // log Z comes from the scan (fbp_scan_kernel)
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
        // b_{tb-1}: 1 at the end of the sequence, else the exact message from the scan
        const float *b0 = CHUNKED ? p.bstart + (chain * nchunk + chunk) * NMAX : nullptr;
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
            b[q] = jv[q] ? (b0 ? b0[32 * q + lane] : 1.f) : 0.f;
            if (jv[q]) bwd[(size_t)(tb - 1) * N + 32 * q + lane] = b[q];
        }
        // staging chunk c covers x_t for t in [t0, t0 + n) in descending t: needs e_{t+1}, rows t0+1 .. t0+n
        auto stage_back = [&](int cc, int buf) {
            const int t0 = ta + cc * CH, ne = min(CH, tb - 1 - t0);
            stage_rows(ech + buf * CH * N, em, N, t0 + 1, ne, lane);
        };
        const int ncb = (tb - 1 - ta + CH - 1) / CH;   // staging chunks of t in [ta, tb-1)
        if (ncb > 0) stage_back(ncb - 1, (ncb - 1) & 1);
        for (int c = ncb - 1; c >= 0; --c) {
            const int t0 = ta + c * CH, n = min(CH, tb - 1 - t0);
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
done:
    if (bad) atomicOr(p.flags, bad);
}

// ---------------------------------------------------------------------------------------------------
// Large state spaces (N > 64, config 4: N = 100): one warp per chain and direction would hold
// ceil(N/32) x N coefficients of A per lane -- too many registers, so the sequential kernel reads A from
// shared memory every step (416 loads per lane per step at N = 100).  Here a CTA runs ONE direction of
// one chain with W = ceil(N/32) warps: lane j of warp w owns state j = 32 w + lane and keeps column j
// (forward) or row j (backward) of A in registers as packed pairs; per step every warp reads the whole
// previous message (broadcast, 128-bit shared loads), forms its 32 outputs and publishes them to a
// double-buffered message vector, and a named barrier over the W warps closes the step.  Same scaling
// and arithmetic as fb_kernel (power-of-two rescale from the broadcast vector's sum).  Each warp stages
// only its own 32 emission columns (cp.async, double-buffered chunks of CH steps).
template <int NMAX>
struct WideCfg {
    static constexpr int W = (NMAX + 31) / 32;   // warps per direction
    static constexpr int CH = 16;                // time steps per staged chunk
    static_assert(NMAX % 8 == 0, "NMAX must be a multiple of 8");
};

template <int NMAX>
__global__ void __launch_bounds__(WideCfg<NMAX>::W * 32, 3) fb_wide_kernel(FBArgs p) {
    using C = WideCfg<NMAX>;
    constexpr int W = C::W, CH = C::CH;
    extern __shared__ __align__(16) float sm[];
    float *mb = sm;                                   // [2][NMAX] message (forward u / backward x), zero-padded
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    float *eb = sm + 2 * NMAX + warp * 2 * CH * 32;   // this warp's [2][CH][32] emission slices
    const int N = p.N, T = p.T, s = blockIdx.y, m = blockIdx.x;
    const bool backward = blockIdx.z == 1;
    const int j = 32 * warp + lane;
    const bool jv = j < N;
    const size_t chain = (size_t)m * p.S + s;
    const float *Ag = p.trans + (size_t)s * N * N;
    const float *em = p.ec + chain * T * N;
    for (int i = threadIdx.x; i < 2 * NMAX; i += blockDim.x) mb[i] = 0.f;
    // forward: u_t[j] = sum_i u[i] A[i][j] (column j); backward: b_t[j] = sum_k A[j][k] x[k] (row j)
    uint64_t Mr[NMAX / 2];
#pragma unroll
    for (int i = 0; i < NMAX; i += 2) {
        float a0 = 0.f, a1 = 0.f;
        if (jv) {
            if (i < N) a0 = backward ? Ag[j * N + i] : Ag[i * N + j];
            if (i + 1 < N) a1 = backward ? Ag[j * N + i + 1] : Ag[(i + 1) * N + j];
        }
        Mr[i / 2] = pk2(a0, a1);
    }
    __syncthreads();
    auto step_sync = [&]() { asm volatile("bar.sync 1, %0;\n" ::"r"(W * 32) : "memory"); };
    auto stage = [&](int buf, int t0, int n) {   // rows [t0, t0 + n) of this warp's 32 columns
        if (jv)
            for (int r = 0; r < n; ++r) cp_async4(eb + (buf * CH + r) * 32 + lane, em + (size_t)(t0 + r) * N + j);
        cp_async_commit();
    };
    // out = sum_i x[i] M(i, j), xsum = sum_i x[i]; four independent FFMA2 chains
    auto products = [&](const float *x, float &out, float &xsum) {
        uint64_t a[4] = {0ull, 0ull, 0ull, 0ull}, s2[2] = {0ull, 0ull};
        const ulonglong2 *x4 = reinterpret_cast<const ulonglong2 *>(x);
#pragma unroll
        for (int i4 = 0; i4 < NMAX / 4; ++i4) {
            const ulonglong2 v = x4[i4];
            add2(s2[0], v.x);
            add2(s2[1], v.y);
            fma2(a[2 * (i4 & 1)], v.x, Mr[2 * i4]);
            fma2(a[2 * (i4 & 1) + 1], v.y, Mr[2 * i4 + 1]);
        }
        add2(a[0], a[1]);
        add2(a[2], a[3]);
        add2(a[0], a[2]);
        out = hsum2(a[0]);
        add2(s2[0], s2[1]);
        xsum = hsum2(s2[0]);
    };
    unsigned bad = 0;
    if (!backward) {
        float *fwd = p.fwd + chain * T * N;
        int esum = 0;
        const int nch = (T + CH - 1) / CH;
        stage(0, 0, min(CH, T));
        for (int c = 0; c < nch; ++c) {
            const int t0 = c * CH, n = min(CH, T - t0);
            cp_async_wait_all();
            __syncwarp();
            if (c + 1 < nch) stage((c + 1) & 1, t0 + CH, min(CH, T - t0 - CH));
            const float *ecur = eb + (c & 1) * CH * 32;
            for (int tt = 0; tt < n; ++tt) {
                const int t = t0 + tt;
                const float e = ecur[tt * 32 + lane];
                float u;
                if (t == 0) {
                    u = jv ? p.prior[s * N + j] * e : 0.f;
                } else {
                    float acc, usum;
                    products(mb + ((t - 1) & 1) * NMAX, acc, usum);
                    if (!(usum > 0.f) || !(usum < INFINITY)) bad |= FLAG_NONFINITE;
                    const int E = exponent_of(usum);
                    esum += E;
                    u = jv ? acc * e * pow2_neg(E) : 0.f;
                }
                if (jv) {
                    mb[(t & 1) * NMAX + j] = u;
                    fwd[(size_t)t * N + j] = u;
                }
                step_sync();
            }
        }
        if (warp == 0) {   // log Z = ln(sum u_{T-1}) + ln 2 sum_t E_t + sum_t eoff_t
            const float *x = mb + ((T - 1) & 1) * NMAX;
            float part = 0.f;
            for (int i = lane; i < N; i += 32) part += x[i];
            const float usum = warp_sum(part);
            if (!(usum > 0.f) || !(usum < INFINITY)) bad |= FLAG_NONFINITE;
            double offsum = 0.0;
            for (int t = lane; t < T; t += 32) offsum += p.eoff[chain * T + t];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) offsum += __shfl_xor_sync(0xffffffffu, offsum, o);
            if (lane == 0) {
                const double lz = log((double)usum) + (double)esum * 0.69314718055994530942 + offsum;
                p.logZ[chain] = lz;
                if (!isfinite(lz)) bad |= FLAG_NONFINITE;
            }
        }
    } else {
        float *bwd = p.bwd + chain * T * N;
        float b = jv ? 1.f : 0.f;
        if (jv) bwd[(size_t)(T - 1) * N + j] = b;
        // chunk c covers t in [c CH, c CH + n) of [0, T - 1), descending; row r holds e_{c CH + 1 + r}
        const int ncb = (T - 1 + CH - 1) / CH;
        auto stage_back = [&](int cc, int buf) { stage(buf, cc * CH + 1, min(CH, T - 1 - cc * CH)); };
        if (ncb > 0) stage_back(ncb - 1, (ncb - 1) & 1);
        for (int c = ncb - 1; c >= 0; --c) {
            const int t0 = c * CH, n = min(CH, T - 1 - t0);
            cp_async_wait_all();
            __syncwarp();
            if (c > 0) stage_back(c - 1, (c - 1) & 1);
            const float *ecur = eb + (c & 1) * CH * 32;
            for (int tt = n - 1; tt >= 0; --tt) {
                const int t = t0 + tt;
                float *xb = mb + (t & 1) * NMAX;
                if (jv) xb[j] = ecur[tt * 32 + lane] * b;
                step_sync();
                float acc, xsum;
                products(xb, acc, xsum);
                if (!(xsum > 0.f) || !(xsum < INFINITY)) bad |= FLAG_NONFINITE;
                b = jv ? acc * pow2_neg(exponent_of(xsum)) : 0.f;
                if (jv) bwd[(size_t)t * N + j] = b;
            }
        }
    }
    if (bad) atomicOr(p.flags, bad);
}

template <int NMAX>
cudaError_t launch_fb_wide(const FBArgs &a, cudaStream_t st) {
    using C = WideCfg<NMAX>;
    const size_t smem = ((size_t)2 * NMAX + (size_t)C::W * 2 * C::CH * 32) * sizeof(float);
    fb_wide_kernel<NMAX><<<dim3(a.M, a.S, 2), C::W * 32, smem, st>>>(a);
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------------------------------
// Parallel-in-time forward-backward, for few chains (single-mixture configurations):
// the time axis is cut into chunks [t0, t1) of L steps and ONE transfer matrix per chunk serves both
// directions,  P_c = prod_{t = t0+1}^{t1-1} A diag(e_t)  (empty product = I):
//   forward   u_{t1-1} = u_{t0} P_c,        next chunk   u_{t1} = (u_{t1-1} A) .* e_{t1};
//   backward  b_{t0}   = P_c b_{t1-1},      previous     b_{t0-1} = A (e_{t0} .* b_{t0}).
// Phase 1 (fbp_transfer_kernel) forms every P_c in parallel -- its rows are independent vector
// recursions of the basis vectors, one warp each, with per-row power-of-two exponents; phase 2
// (fbp_scan_kernel) walks the chunks once per chain and direction -- C vector-matrix products instead of
// T dependent steps -- giving the exact chunk-start messages and log Z; phase 3 re-runs each chunk from
// its start message in parallel (fb_kernel<NMAX, true>).  Exact up to FP32 rounding: the same products
// in a different association order.

// Phase 1: row i of P_c is the forward recursion of the basis vector e_i through the chunk
// (P'[i][:] = P[i][:] A diag(e_t)), so every row is an independent warp running the same vector step as
// the sequential kernel (A columns in registers, broadcast through shared memory, power-of-two rescale).
// Rows carry their own exponents PE[row] (the scan folds them in exactly); P is written row-major and
// transposed.  Block = FBP_ROWS warps (rows) of one (chain, chunk).
constexpr int FBP_ROWS = 4;

template <int NMAX>
__global__ void __launch_bounds__(FBP_ROWS * 32) fbp_transfer_kernel(FBArgs p, float *P, float *PT, int *PE) {
    using C = FBCfg<NMAX>;
    constexpr int NQ = C::NQ;
    extern __shared__ __align__(16) float sm[];
    float *As = sm;                                   // [NMAX][NMAX]  A[i][j]
    float *es = As + NMAX * NMAX;                     // [L][NMAX] emissions of the chunk
    float *xb = es + p.chunk_len * NMAX;              // [FBP_ROWS][2][NMAX] broadcast buffers
    const int N = p.N, T = p.T, L = p.chunk_len;
    const int rows_blocks = (NMAX + FBP_ROWS - 1) / FBP_ROWS;
    const int c = blockIdx.x / rows_blocks, rb = blockIdx.x - c * rows_blocks;
    const int chain = blockIdx.y, s = chain % p.S;
    const int t0 = c * L, t1 = min(T, t0 + L);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int row = rb * FBP_ROWS + warp;
    const float *Ag = p.trans + (size_t)s * N * N;
    for (int idx = threadIdx.x; idx < NMAX * NMAX; idx += blockDim.x) {
        const int r = idx / NMAX, cc = idx - r * NMAX;
        As[idx] = (r < N && cc < N) ? Ag[r * N + cc] : 0.f;
    }
    const float *em = p.ec + (size_t)chain * T * N;
    for (int idx = threadIdx.x; idx < (t1 - t0) * NMAX; idx += blockDim.x) {
        const int r = idx / NMAX, cc = idx - r * NMAX;
        es[idx] = (cc < N) ? em[(size_t)(t0 + r) * N + cc] : 0.f;
    }
    float *bx = xb + warp * 2 * NMAX;
    for (int idx = lane; idx < 2 * NMAX; idx += 32) bx[idx] = 0.f;
    __syncthreads();
    if (row >= NMAX) return;
    bool jv[NQ];
#pragma unroll
    for (int q = 0; q < NQ; ++q) jv[q] = 32 * q + lane < N;
    uint64_t Mr[C::REG ? NQ : 1][C::REG ? NMAX / 2 : 1];
    if (C::REG) {
#pragma unroll
        for (int q = 0; q < NQ; ++q)
#pragma unroll
            for (int i = 0; i < NMAX; i += 2)
                Mr[C::REG ? q : 0][C::REG ? i / 2 : 0] =
                    32 * q + lane < NMAX ? pk2(As[i * NMAX + 32 * q + lane], As[(i + 1) * NMAX + 32 * q + lane]) : 0ull;
    }
    float v[NQ];
#pragma unroll
    for (int q = 0; q < NQ; ++q) v[q] = (32 * q + lane == row && row < N) ? 1.f : 0.f;
    int etot = 0;
    for (int t = t0 + 1; t < t1; ++t) {
        float *un = bx + ((t - t0) & 1) * NMAX;
#pragma unroll
        for (int q = 0; q < NQ; ++q)
            if (jv[q]) un[32 * q + lane] = v[q];
        __syncwarp();
        float acc[NQ], xs;
        step_products<NMAX>(acc, xs, un, Mr, As, lane);
        // row of a state no path leaves (or a padded row): stays zero, no rescale
        const int E = xs > 0.f ? exponent_of(xs) : 0;
        const float sc = pow2_neg(E);
        etot += E;
        const float *et = es + (t - t0) * NMAX;
#pragma unroll
        for (int q = 0; q < NQ; ++q) v[q] = jv[q] ? acc[q] * et[32 * q + lane] * sc : 0.f;
    }
    // the exponents of the first step's input were 0 (a basis vector); the last step's output carries
    // the scale of its input sum only: fold the row's remaining magnitude into etot via one more rescale
    float part = 0.f;
#pragma unroll
    for (int q = 0; q < NQ; ++q) part += v[q];
    const float rs = warp_sum(part);
    const int E = rs > 0.f ? exponent_of(rs) : 0;
    const float sc = pow2_neg(E);
    etot += E;
    float *Pc = P + ((size_t)chain * p.nchunk + c) * NMAX * NMAX;
    float *PTc = PT + ((size_t)chain * p.nchunk + c) * NMAX * NMAX;
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
        const int j = 32 * q + lane;
        if (j < NMAX) {
            const float x = jv[q] ? v[q] * sc : 0.f;
            Pc[(size_t)row * NMAX + j] = x;
            PTc[(size_t)j * NMAX + row] = x;
        }
    }
    if (lane == 0) PE[((size_t)chain * p.nchunk + c) * NMAX + row] = etot;
}

// Phase 2: warp 0 = forward scan (chunk-start u, log Z), warp 1 = backward scan (chunk-end b).  Each
// chunk's inputs -- P_c (forward) or P_c^T (backward), its row exponents and the emission row that links
// to the neighbouring chunk -- arrive together in a FBP_RING-deep cp.async ring, so the walk over the
// chunks is bound by its own arithmetic rather than by one L2 round trip per chunk.
constexpr int FBP_RING = 4;

template <int NMAX>
struct ScanSlot {   // floats: P [NMAX][NMAX] | exponents [NMAX] (int bits) | emission row [NMAX]
    static constexpr int FLOATS = NMAX * NMAX + 2 * NMAX;
};

template <int NMAX>
__global__ void __launch_bounds__(64) fbp_scan_kernel(FBArgs p, const float *P, const float *PT, const int *PE,
                                                      float *fstart, float *bstart) {
    using C = FBCfg<NMAX>;
    constexpr int NQ = C::NQ, SLOT = ScanSlot<NMAX>::FLOATS;
    extern __shared__ __align__(16) float sm[];
    float *As = sm;                                   // [NMAX][NMAX] A[i][j]
    float *AT = As + NMAX * NMAX;                     // [NMAX][NMAX] AT[j][i]
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nc = p.nchunk;
    float *wall = AT + NMAX * NMAX + warp * ((size_t)nc * NMAX + FBP_RING * SLOT + 2 * NMAX);   // [nc][NMAX]
    float *ring = wall + (size_t)nc * NMAX;
    float *xb = ring + FBP_RING * SLOT;               // broadcast buffers [2][NMAX]
    const int N = p.N, T = p.T, L = p.chunk_len;
    const int chain = blockIdx.x, s = chain % p.S;
    const float *Ag = p.trans + (size_t)s * N * N;
    for (int idx = threadIdx.x; idx < NMAX * NMAX; idx += blockDim.x) {
        const int r = idx / NMAX, cc = idx - r * NMAX;
        const float v = (r < N && cc < N) ? Ag[r * N + cc] : 0.f;
        As[idx] = v;
        AT[cc * NMAX + r] = v;
    }
    for (int idx = lane; idx < 2 * NMAX; idx += 32) xb[idx] = 0.f;
    for (int idx = lane; idx < FBP_RING * SLOT; idx += 32) ring[idx] = 0.f;   // (padded emission entries)
    __syncthreads();
    const float *em = p.ec + (size_t)chain * T * N;
    bool jv[NQ];
#pragma unroll
    for (int q = 0; q < NQ; ++q) jv[q] = 32 * q + lane < N;
    unsigned bad = 0;
    const bool fwd = warp == 0;
    const float *M = fwd ? As : AT;                   // the linking step: u A (forward), A x (backward)
    uint64_t Mr[C::REG ? NQ : 1][C::REG ? NMAX / 2 : 1];
    if (C::REG) {
#pragma unroll
        for (int q = 0; q < NQ; ++q)
#pragma unroll
            for (int i = 0; i < NMAX; i += 2)
                Mr[C::REG ? q : 0][C::REG ? i / 2 : 0] =
                    32 * q + lane < NMAX ? pk2(M[i * NMAX + 32 * q + lane], M[(i + 1) * NMAX + 32 * q + lane]) : 0ull;
    }
    // every chunk's row scales w[c][i] = 2^(E_i - Emax_c) up front (independent of the messages), with the
    // total of the Emax_c (forward: chunks 0..nc-1; backward: nc-1..1) kept for log Z
    long long ls = 0;
    for (int c = 0; c < nc; ++c) {
        const int *pe = PE + ((size_t)chain * nc + c) * NMAX;
        int e[NQ], emax = INT_MIN;
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
            e[q] = jv[q] ? pe[32 * q + lane] : INT_MIN;
            emax = max(emax, e[q]);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) emax = max(emax, __shfl_xor_sync(0xffffffffu, emax, o));
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
            const int d = jv[q] ? e[q] - emax : -1000;
            if (32 * q + lane < NMAX) wall[c * NMAX + 32 * q + lane] = d < -126 ? 0.f : __uint_as_float((uint32_t)(127 + d) << 23);
        }
        if (fwd || c > 0) ls += emax;
    }
    // slot for chunk c: matrix, (unused exponent row), linking emission row (forward e_{t1}; backward e_{t0})
    auto stage = [&](int c) {
        float *dst = ring + (c % FBP_RING) * SLOT;
        const float *src = (fwd ? P : PT) + ((size_t)chain * nc + c) * NMAX * NMAX;
        for (int i = lane; i < NMAX * NMAX / 4; i += 32) {
            const unsigned sa = (unsigned)__cvta_generic_to_shared(dst + 4 * i);
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(src + 4 * i));
        }
        const int te = fwd ? (c + 1) * L : c * L;
        if (te < T)
            for (int i = lane; i < N; i += 32) cp_async4(dst + NMAX * NMAX + NMAX + i, em + (size_t)te * N + i);
        cp_async_commit();
    };
    // x (broadcast in smem) times the slot matrix Ms (lane-owned columns); xsum = sum of x
    auto vecmat = [&](const float *x, const float *Ms, float (&out)[NQ], float &xsum) {
        uint64_t acc[NQ][4];   // four independent FFMA2 chains per output (as step_products)
        uint64_t s2[2] = {0ull, 0ull};
#pragma unroll
        for (int q = 0; q < NQ; ++q) acc[q][0] = acc[q][1] = acc[q][2] = acc[q][3] = 0ull;
        const ulonglong2 *x4 = reinterpret_cast<const ulonglong2 *>(x);
#pragma unroll
        for (int i4 = 0; i4 < NMAX / 4; ++i4) {
            const ulonglong2 v = x4[i4];
            add2(s2[0], v.x);
            add2(s2[1], v.y);
#pragma unroll
            for (int q = 0; q < NQ; ++q) {
                const int j = min(32 * q + lane, NMAX - 1), i = 4 * i4;
                fma2(acc[q][(2 * i4) & 3], v.x, pk2(Ms[i * NMAX + j], Ms[(i + 1) * NMAX + j]));
                fma2(acc[q][(2 * i4 + 1) & 3], v.y, pk2(Ms[(i + 2) * NMAX + j], Ms[(i + 3) * NMAX + j]));
            }
        }
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
            add2(acc[q][0], acc[q][1]);
            add2(acc[q][2], acc[q][3]);
            add2(acc[q][0], acc[q][2]);
            out[q] = hsum2(acc[q][0]);
        }
        add2(s2[0], s2[1]);
        xsum = hsum2(s2[0]);
    };
    auto put = [&](const float (&v)[NQ], int b) {
        __syncwarp();
#pragma unroll
        for (int q = 0; q < NQ; ++q)
            if (jv[q]) xb[b * NMAX + 32 * q + lane] = v[q];
        __syncwarp();
    };
    float v[NQ], y[NQ];
    const int npre = min(FBP_RING - 1, nc);
    if (fwd) {
        for (int c = 0; c < npre; ++c) stage(c);
        float part = 0.f;
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
            v[q] = jv[q] ? p.prior[s * N + 32 * q + lane] * em[32 * q + lane] : 0.f;
            part += v[q];
        }
        {   // u_0 normalised exactly once; later rescales come from the lane-local input sums
            const float s0 = warp_sum(part);
            const int E = exponent_of(s0);
            const float sc = pow2_neg(E);
#pragma unroll
            for (int q = 0; q < NQ; ++q) v[q] *= sc;
            ls += E;
        }
        for (int c = 0; c < nc; ++c) {
            // v = u_{t0} of chunk c (scaled)
#pragma unroll
            for (int q = 0; q < NQ; ++q)
                if (jv[q]) fstart[((size_t)chain * nc + c) * NMAX + 32 * q + lane] = v[q];
            if (c + FBP_RING - 1 < nc) stage(c + FBP_RING - 1);
            else cp_async_commit();
            asm volatile("cp.async.wait_group %0;\n" ::"n"(FBP_RING - 1));
            __syncwarp();
            const float *slot = ring + (c % FBP_RING) * SLOT;
            float w[NQ], xs;
#pragma unroll
            for (int q = 0; q < NQ; ++q) w[q] = jv[q] ? v[q] * wall[c * NMAX + 32 * q + lane] : 0.f;
            put(w, 0);
            vecmat(xb, slot, y, xs);                               // u_{t1-1} = u_{t0} P_c (row-scaled)
            if (c + 1 < nc) {
                put(y, 1);
                float an[NQ], ys;
                step_products<NMAX>(an, ys, xb + NMAX, Mr, M, lane);   // u_{t1} = (u_{t1-1} A) .* e_{t1}
                const int E = exponent_of(ys);                     // rescale by the input's sum
                const float sc = pow2_neg(E);
                ls += E;
                const float *e1 = slot + NMAX * NMAX + NMAX;
#pragma unroll
                for (int q = 0; q < NQ; ++q) v[q] = jv[q] ? an[q] * e1[32 * q + lane] * sc : 0.f;
                if (!(ys > 0.f) || !(ys < INFINITY)) bad |= FLAG_NONFINITE;
            } else {
                float part2 = 0.f;
#pragma unroll
                for (int q = 0; q < NQ; ++q) part2 += jv[q] ? y[q] : 0.f;
                const float us = warp_sum(part2);
                if (!(us > 0.f) || !(us < INFINITY)) bad |= FLAG_NONFINITE;
                double offsum = 0.0;
                for (int t = lane; t < T; t += 32) offsum += p.eoff[(size_t)chain * T + t];
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) offsum += __shfl_xor_sync(0xffffffffu, offsum, o);
                if (lane == 0) {
                    const double lz = log((double)us) + (double)ls * 0.69314718055994530942 + offsum;
                    p.logZ[chain] = lz;
                    if (!isfinite(lz)) bad |= FLAG_NONFINITE;
                }
            }
        }
    } else {
        // chunks in descending order: ring position k holds chunk nc - 1 - k
        auto cid = [&](int k) { return nc - 1 - k; };
        for (int k = 0; k < npre; ++k) stage(cid(k));
#pragma unroll
        for (int q = 0; q < NQ; ++q) v[q] = jv[q] ? 1.f : 0.f;
        for (int k = 0; k < nc; ++k) {
            const int c = cid(k);
            // v = b_{t1-1} of chunk c (scaled)
#pragma unroll
            for (int q = 0; q < NQ; ++q)
                if (jv[q]) bstart[((size_t)chain * nc + c) * NMAX + 32 * q + lane] = v[q];
            if (k + FBP_RING - 1 < nc) stage(cid(k + FBP_RING - 1));
            else cp_async_commit();
            if (c == 0) break;
            asm volatile("cp.async.wait_group %0;\n" ::"n"(FBP_RING - 1));
            __syncwarp();
            const float *slot = ring + (c % FBP_RING) * SLOT;
            float xs;
            put(v, 0);
            vecmat(xb, slot, y, xs);                               // b_{t0} = P_c b_{t1-1} (slot holds P^T)
            const int E = exponent_of(xs);                         // rescale by the input's sum
            const float sc = pow2_neg(E);
            if (!(xs > 0.f) || !(xs < INFINITY)) bad |= FLAG_NONFINITE;
            const float *e0 = slot + NMAX * NMAX + NMAX;
#pragma unroll
            for (int q = 0; q < NQ; ++q) y[q] = jv[q] ? y[q] * wall[c * NMAX + 32 * q + lane] * e0[32 * q + lane] * sc : 0.f;
            put(y, 1);
            float ys;
            step_products<NMAX>(v, ys, xb + NMAX, Mr, M, lane);   // b_{t0-1} = A (e_{t0} .* b_{t0})
        }
    }
    cp_async_wait_all();
    if (bad) atomicOr(p.flags, bad);
}

template <int NMAX>
cudaError_t launch_fb_t(const FBArgs &a, cudaStream_t st) {
    using C = FBCfg<NMAX>;
    const int N = a.N;
    const size_t smem = ((size_t)2 * NMAX * NMAX + (size_t)C::WPB * (2 * NMAX + 2 * C::CH * N)) * sizeof(float);
    const bool chunked = a.nchunk > 1;
    auto kern = chunked ? fb_kernel<NMAX, true> : fb_kernel<NMAX, false>;
    {
        cudaError_t e = ensure_dyn_smem((const void *)kern, smem);
        if (e != cudaSuccess) return e;
    }
    if (chunked) {   // phases 1 and 2 of the parallel-in-time path (NMAX <= 64)
        if (NMAX > 64 || !a.P || !a.PT || !a.PE) return cudaErrorInvalidValue;
        const size_t sm1 = ((size_t)NMAX * NMAX + (size_t)a.chunk_len * NMAX + FBP_ROWS * 2 * NMAX) * sizeof(float);
        const size_t sm2 = ((size_t)2 * NMAX * NMAX +
                            2 * ((size_t)a.nchunk * NMAX + (size_t)FBP_RING * ScanSlot<NMAX>::FLOATS + 2 * NMAX)) * sizeof(float);
        {
            cudaError_t e = ensure_dyn_smem((const void *)fbp_transfer_kernel<NMAX>, sm1);
            if (e == cudaSuccess) e = ensure_dyn_smem((const void *)fbp_scan_kernel<NMAX>, sm2);
            if (e != cudaSuccess) return e;
        }
        const int rows_blocks = (NMAX + FBP_ROWS - 1) / FBP_ROWS;
        fbp_transfer_kernel<NMAX><<<dim3(a.nchunk * rows_blocks, a.M * a.S), FBP_ROWS * 32, sm1, st>>>(a, a.P, a.PT, a.PE);
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
        fbp_scan_kernel<NMAX><<<a.M * a.S, 64, sm2, st>>>(a, a.P, a.PT, a.PE, a.fstart, a.bstart);
        e = cudaGetLastError();
        if (e != cudaSuccess) return e;
    }
    const int units = a.M * (chunked ? a.nchunk : 1);
    dim3 grid((units + C::CPB - 1) / C::CPB, a.S);
    kern<<<grid, C::WPB * 32, smem, st>>>(a);
    return cudaGetLastError();
}

}  // namespace

// ---------------------------------------------------------------------------------------------------
// Many chains per source (batched configurations): C chains of ONE source and ONE direction per warp,
// sharing that source's A in registers.  For N = 32 Q + R (R = 32 / C, e.g. N = 40 = 32 + 8 with C = 4):
// lane l owns state l of every chain in each full round q < Q, and state 32 Q + l % R of chain l / R in
// the remainder round, so the remainder's lanes are not idle (the one-chain kernel leaves 24 of 32 lanes
// idle in its second round at N = 40).  A step: the C previous messages are broadcast through shared
// memory (LDS.128), each lane forms its Q C + 1 dot products with packed FFMA2 (C Q + 1 independent
// chains -- the latency is hidden by the other chains instead of by split accumulators), the scale
// 2^-E of each chain comes from the sum of that chain's broadcast vector (computed by its remainder lane
// group, shared by a shuffle), and the outputs are multiplied by the emissions (forward) or turned into
// the next step's e .* b (backward).  Same recursions and scaling as fb_kernel:
//   u_0 = pi .* e_0,  u_t = ((u_{t-1} A) .* e_t) 2^-E(sum u_{t-1});
//   b_{T-1} = 1,  b_t = (A (e_{t+1} .* b_{t+1})) 2^-E(sum e_{t+1} .* b_{t+1});
//   log Z = ln(sum u_{T-1}) + ln 2 sum_t E_t + sum_t eoff_t.
// The emissions of the next FBM_D steps (all C chains) are staged in a per-warp cp.async ring.
constexpr int FBM_D = 8;   // emission ring depth (steps)
#ifndef FBM_MINB
#define FBM_MINB 1   // min resident warps per SM asked of ptxas (16: <= 128 registers)
#endif

template <int Q, int R>
struct FBMCfg {
    static constexpr int C = 32 / R;          // chains per warp
    static constexpr int NM = 32 * Q + R;     // states
    static constexpr int SLOT = C * NM;       // floats per emission slot (one step, all chains)
    static constexpr int SMEM = (2 * C * NM + FBM_D * SLOT) * 4;   // per warp: 2 broadcast buffers + ring
    static_assert(NM % 4 == 0, "states must be a multiple of 4");
};

template <int Q, int R>
__global__ void __launch_bounds__(32, FBM_MINB) fb_multi_kernel(FBArgs p) {
    using C_ = FBMCfg<Q, R>;
    constexpr int C = C_::C, NM = C_::NM, SLOT = C_::SLOT;
    constexpr int CHUNKS = SLOT / 4, CPL = (CHUNKS + 31) / 32;   // 16-byte emission chunks per step, per lane
    extern __shared__ __align__(16) float sm[];
    float *xb = sm;                          // [2][C][NM] broadcast messages
    float *ring = sm + 2 * C * NM;           // [FBM_D][C][NM] emissions
    const int lane = threadIdx.x;
    const int groups = (p.M + C - 1) / C;
    const int s = blockIdx.x / (2 * groups), rem = blockIdx.x - s * 2 * groups;
    const bool backward = rem >= groups;
    const int grp0 = backward ? rem - groups : rem;
    const int m0 = grp0 * C;
    const int T = p.T, N = NM;
    const int g = lane / R, jr = 32 * Q + lane % R;   // remainder round: chain g, state jr
    const float *Ag = p.trans + (size_t)s * N * N;
    // A in registers: forward u A -> column j; backward A x -> row j (pairs over the input index)
    uint64_t Mq[Q > 0 ? Q : 1][NM / 2], Mr[NM / 2];
#pragma unroll
    for (int i = 0; i < NM; i += 2) {
#pragma unroll
        for (int q = 0; q < Q; ++q) {
            const int j = 32 * q + lane;
            Mq[q][i / 2] = backward ? pk2(Ag[j * N + i], Ag[j * N + i + 1]) : pk2(Ag[i * N + j], Ag[(i + 1) * N + j]);
        }
        Mr[i / 2] = backward ? pk2(Ag[jr * N + i], Ag[jr * N + i + 1]) : pk2(Ag[i * N + jr], Ag[(i + 1) * N + jr]);
    }
    // per-chain message rows (chains past M write nothing; they compute on a valid chain's emissions)
    const int cm = p.M - 1 - m0;             // last valid chain index in the group
    float *outp = backward ? p.bwd : p.fwd;
    float *orow[C];
#pragma unroll
    for (int c = 0; c < C; ++c) orow[c] = outp + ((size_t)(m0 + (c <= cm ? c : cm)) * p.S + s) * T * N;
    const bool gv = g <= cm;
    float *grow = orow[0];   // chain g's row (selected without indexing the register array)
#pragma unroll
    for (int c = 1; c < C; ++c)
        if (c == g) grow = orow[c];
    // emission staging: this lane's chunks (chain, 16-byte offset), source rows advanced by one step each
    const float *esrc[CPL];
    unsigned edst[CPL];
    bool eok[CPL];
#pragma unroll
    for (int u = 0; u < CPL; ++u) {
        const int k = lane + 32 * u;
        eok[u] = k < CHUNKS;
        const int c = eok[u] ? k / (NM / 4) : 0, o = eok[u] ? k - c * (NM / 4) : 0;
        const int cc = c <= cm ? c : cm;
        esrc[u] = p.ec + ((size_t)(m0 + cc) * p.S + s) * T * N + 4 * o;
        edst[u] = (unsigned)__cvta_generic_to_shared(ring + c * NM + 4 * o);
    }
    auto stage = [&](int t) {
        const unsigned slot = (unsigned)((t % FBM_D) * SLOT * 4);
#pragma unroll
        for (int u = 0; u < CPL; ++u)
            if (eok[u]) asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(edst[u] + slot), "l"(esrc[u] + (size_t)t * N));
        cp_async_commit();
    };
    unsigned bad = 0;
    const int t_first = backward ? T - 1 : 0, dt = backward ? -1 : 1;
    for (int k = 0; k < FBM_D - 1; ++k) {
        const int t = t_first + dt * k;
        if (t >= 0 && t < T) stage(t);
        else cp_async_commit();
    }
    int esum = 0;            // (forward) exponent sum of chain g (the remainder group's chain)
    float vq[Q > 0 ? Q : 1][C], vr = 0.f;   // this lane's current outputs
    int t = t_first;
    for (int k = 0; k < T; ++k, t += dt) {
        {   // keep FBM_D - 1 steps in flight
            const int tn = t + dt * (FBM_D - 1);
            if (tn >= 0 && tn < T) stage(tn);
            else cp_async_commit();
        }
        asm volatile("cp.async.wait_group %0;\n" ::"n"(FBM_D - 1));
        __syncwarp();
        const float *et = ring + (t % FBM_D) * SLOT;
        float *xo = xb + (k & 1) * C * NM;          // this step's outputs (broadcast for the next step)
        float eq[Q > 0 ? Q : 1][C], er;
#pragma unroll
        for (int q = 0; q < Q; ++q)
#pragma unroll
            for (int c = 0; c < C; ++c) eq[q][c] = et[c * NM + 32 * q + lane];
        er = et[g * NM + jr];
        if (k == 0) {
            if (!backward) {   // u_0 = pi .* e_0 (unscaled)
#pragma unroll
                for (int q = 0; q < Q; ++q)
#pragma unroll
                    for (int c = 0; c < C; ++c) vq[q][c] = p.prior[s * N + 32 * q + lane] * eq[q][c];
                vr = p.prior[s * N + jr] * er;
            } else {           // b_{T-1} = 1
#pragma unroll
                for (int q = 0; q < Q; ++q)
#pragma unroll
                    for (int c = 0; c < C; ++c) vq[q][c] = 1.f;
                vr = 1.f;
            }
        } else {
            const float *xi = xb + ((k - 1) & 1) * C * NM;   // previous step's broadcast vectors
            uint64_t aq[Q > 0 ? Q : 1][C], ar = 0ull, xs2[2] = {0ull, 0ull};
#pragma unroll
            for (int q = 0; q < Q; ++q)
#pragma unroll
                for (int c = 0; c < C; ++c) aq[q][c] = 0ull;
#pragma unroll
            for (int i4 = 0; i4 < NM / 4; ++i4) {
#pragma unroll
                for (int c = 0; c < C; ++c) {
                    if (Q == 0) break;
                    const ulonglong2 v = reinterpret_cast<const ulonglong2 *>(xi + c * NM)[i4];
#pragma unroll
                    for (int q = 0; q < Q; ++q) {
                        fma2(aq[q][c], v.x, Mq[q][2 * i4]);
                        fma2(aq[q][c], v.y, Mq[q][2 * i4 + 1]);
                    }
                }
                const ulonglong2 w = reinterpret_cast<const ulonglong2 *>(xi + g * NM)[i4];
                fma2(ar, w.x, Mr[2 * i4]);
                fma2(ar, w.y, Mr[2 * i4 + 1]);
                add2(xs2[0], w.x);
                add2(xs2[1], w.y);
            }
            add2(xs2[0], xs2[1]);
            const float xsum = hsum2(xs2[0]);          // sum of chain g's broadcast vector
            if (gv && (!(xsum > 0.f) || !(xsum < INFINITY))) bad |= FLAG_NONFINITE;
            const int E = exponent_of(xsum);
            if (!backward) esum += E;
#pragma unroll
            for (int c = 0; c < C; ++c) {
                if (Q == 0) break;
                const float sc = pow2_neg(__shfl_sync(0xffffffffu, E, c * R));
#pragma unroll
                for (int q = 0; q < Q; ++q) vq[q][c] = hsum2(aq[q][c]) * sc;
            }
            vr = hsum2(ar) * pow2_neg(E);
            if (!backward) {   // u_t = (u_{t-1} A) .* e_t  2^-E
#pragma unroll
                for (int q = 0; q < Q; ++q)
#pragma unroll
                    for (int c = 0; c < C; ++c) vq[q][c] *= eq[q][c];
                vr *= er;
            }
        }
        // store the messages (u_t or b_t) and publish the next broadcast vector (u_t, or e_t .* b_t)
        const int to = t * N;
#pragma unroll
        for (int q = 0; q < Q; ++q)
#pragma unroll
            for (int c = 0; c < C; ++c) {
                if (c <= cm) orow[c][to + 32 * q + lane] = vq[q][c];
                xo[c * NM + 32 * q + lane] = backward ? vq[q][c] * eq[q][c] : vq[q][c];
            }
        if (gv) grow[to + jr] = vr;
        xo[g * NM + jr] = backward ? vr * er : vr;
        __syncwarp();
    }
    cp_async_wait_all();
    if (!backward) {   // log Z of chain g (its R lanes agree): ln(sum u_{T-1}) + ln 2 sum E + sum eoff
        const float *xl = xb + ((T - 1) & 1) * C * NM + g * NM;
        float us = 0.f;
        for (int i = lane % R; i < NM; i += R) us += xl[i];
        double off = 0.0;
        const size_t chain = (size_t)(m0 + (gv ? g : 0)) * p.S + s;
        if (gv)
            for (int tt = lane % R; tt < T; tt += R) off += p.eoff[chain * T + tt];
#pragma unroll
        for (int o = R / 2; o > 0; o >>= 1) {
            us += __shfl_xor_sync(0xffffffffu, us, o);
            off += __shfl_xor_sync(0xffffffffu, off, o);
        }
        if (gv && lane % R == 0) {
            if (!(us > 0.f) || !(us < INFINITY)) bad |= FLAG_NONFINITE;
            const double lz = log((double)us) + (double)esum * 0.69314718055994530942 + off;
            p.logZ[chain] = lz;
            if (!isfinite(lz)) bad |= FLAG_NONFINITE;
        }
    }
    if (bad) atomicOr(p.flags, bad);
}

template <int Q, int R>
cudaError_t launch_fb_multi(const FBArgs &a, cudaStream_t st) {
    using C_ = FBMCfg<Q, R>;
    const int groups = (a.M + C_::C - 1) / C_::C;
    cudaError_t e = ensure_dyn_smem((const void *)fb_multi_kernel<Q, R>, C_::SMEM);
    if (e != cudaSuccess) return e;
    fb_multi_kernel<Q, R><<<a.S * 2 * groups, 32, C_::SMEM, st>>>(a);
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------------------------------
// Tensor-core forward-backward for many chains per source (round 2): the chains of one source share A_s,
// so one step of 16 chains is a [16 x N] x [N x N] matrix product -- warp-level mma.sync m16n8k8 TF32 with
// the 3xTF32 split (a_lo b_hi + a_hi b_lo + a_hi b_hi, as the GEMMs; FP32 accumulation).  One CTA per
// (source, direction, 16 chains) with one warp per 8-state column tile (N = 8 NT: NT warps); each warp
// keeps its column tile of A (hi / lo fragments) in registers for the whole recursion, reads the previous
// messages of all 16 chains from a shared tile as A-operand fragments, and publishes its 8 columns of the
// new messages and their row-sum partials; one named barrier per step.  The three products accumulate
// separately (mma.sync's latency on sm_100 is long: NT-deep chains).  Same recursions and scaling as
// fb_kernel (power-of-two scale from the previous message's row sum):
//   forward u_t = ((u_{t-1} A) 2^-E) .* e_t;  backward b_t = (x_{t+1} A^T) 2^-E, x_t = e_t .* b_t.
constexpr int FBT_D = 8;   // emission ring depth (steps)

__device__ __forceinline__ void mma_tf32(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
    asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                 : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
                 : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
// hi = x rounded to TF32 (nearest, ties away: two integer ops); lo = x - hi exactly (the MMA reads its top
// 19 bits -- a truncation 2^-11 below lo, i.e. 2^-22 of x)
__device__ __forceinline__ uint32_t tf32_hi_bits(float x) { return (__float_as_uint(x) + 0x1000u) & 0xFFFFE000u; }

template <int NT>   // N = 8 NT states, NT warps
struct FBTCfg {
    static constexpr int N = 8 * NT, LD = N + 4;   // operand tile row pitch (floats; +4 staggers the banks)
    static constexpr int OP = 16 * LD;
    static constexpr int RING = 16 * 8;            // one warp's emission slot: 16 rows x its 8 columns
    static constexpr int FLOATS = 4 * OP + 2 * NT * 16 + NT * FBT_D * RING;   // op tiles (hi, lo) x 2 | row sums | rings
};

template <int NT>
__global__ void __launch_bounds__(NT * 32) fb_mma_kernel(FBArgs p) {
    using C_ = FBTCfg<NT>;
    constexpr int N = C_::N, LD = C_::LD, OP = C_::OP, RING = C_::RING;
    extern __shared__ __align__(16) float sm[];
    uint32_t *opb = reinterpret_cast<uint32_t *>(sm);   // [2][hi, lo][16][LD] operand tiles, already split
    float *rsp = sm + 4 * OP;                     // [2][NT][16] row-sum partials
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    float *ring = rsp + 2 * NT * 16 + warp * FBT_D * RING;   // this warp's [FBT_D][16][8] emissions
    const int groups = (p.M + 15) / 16;
    const int s = blockIdx.x / (2 * groups), rem = blockIdx.x - s * 2 * groups;
    const bool backward = rem >= groups;
    const int m0 = (backward ? rem - groups : rem) * 16;
    const int T = p.T;
    const int g = lane >> 2, tq = lane & 3;
    const int rows_valid = min(16, p.M - m0);
    const int col = 8 * warp + 2 * tq;            // this thread's two columns
    const float *Ag = p.trans + (size_t)s * N * N;
    // B fragments of column tile `warp`: forward B[k][n] = A[k][n]; backward B[k][n] = A[n][k];
    // b0 = (k = 8j + tq, n = 8 warp + g), b1 = (k = 8j + tq + 4, n = 8 warp + g)
    uint32_t bh[NT][2], bl[NT][2];
#pragma unroll
    for (int j = 0; j < NT; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int k = 8 * j + tq + 4 * h, n = 8 * warp + g;
            const float v = backward ? Ag[n * N + k] : Ag[k * N + n];
            const uint32_t hi = tf32_hi_bits(v);
            bh[j][h] = hi;
            bl[j][h] = __float_as_uint(v - __uint_as_float(hi));
        }
    const int rA = g, rB = g + 8;
    const bool vA = rA < rows_valid, vB = rB < rows_valid;
    const size_t chA = (size_t)(m0 + (vA ? rA : 0)) * p.S + s, chB = (size_t)(m0 + (vB ? rB : 0)) * p.S + s;
    float *outp = backward ? p.bwd : p.fwd;
    const int dtN = backward ? -N : N;   // message pointers advance one row per step
    float *oA = outp + chA * T * N + col + (size_t)(backward ? T - 1 : 0) * N;
    float *oB = outp + chB * T * N + col + (size_t)(backward ? T - 1 : 0) * N;
    const float pr0 = backward ? 0.f : p.prior[s * N + col], pr1 = backward ? 0.f : p.prior[s * N + col + 1];
    // emission ring: lane = (row lane / 2, half lane % 2) -> one 16-byte chunk of its row's 8 columns
    const int er = lane >> 1;
    const int err = er < rows_valid ? er : 0;
    // step kk's emission row e_t (t = t_first + dt kk) goes to ring slot kk % FBT_D
    const int t_first = backward ? T - 1 : 0;
    const float *esrc = p.ec + ((size_t)(m0 + err) * p.S + s) * T * N + 8 * warp + 4 * (lane & 1) + (size_t)t_first * N;
    const unsigned edst = (unsigned)__cvta_generic_to_shared(ring + er * 8 + 4 * (lane & 1));
    auto stage = [&](int kk) {
        if (kk < T)
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(edst + (unsigned)((kk & (FBT_D - 1)) * RING * 4)),
                         "l"(esrc + (ptrdiff_t)kk * dtN));
        cp_async_commit();
    };
    for (int kk = 0; kk < FBT_D - 1; ++kk) stage(kk);
    unsigned bad = 0;
    int EA = 0, EB = 0;              // exponents of the operand rows' sums (applied at the next step)
    int esumA = 0, esumB = 0;        // forward: applied exponents (log Z)
    float sumA = 0.f, sumB = 0.f;    // the last operand row sums (forward: sum u_{T-1})
    const unsigned bar_n = NT * 32;
    for (int k = 0; k < T; ++k) {
        stage(k + FBT_D - 1);
        asm volatile("cp.async.wait_group %0;\n" ::"n"(FBT_D - 1));
        __syncwarp();
        const float *et = ring + (k & (FBT_D - 1)) * RING;
        const float2 ea = *reinterpret_cast<const float2 *>(et + rA * 8 + 2 * tq);
        const float2 eb = *reinterpret_cast<const float2 *>(et + rB * 8 + 2 * tq);
        float c[4];   // (rA, col), (rA, col+1), (rB, col), (rB, col+1)
        if (k == 0) {
            if (backward) {
                c[0] = c[1] = c[2] = c[3] = 1.f;
            } else {   // u_0 = pi .* e_0 (unscaled)
                c[0] = pr0 * ea.x;
                c[1] = pr1 * ea.y;
                c[2] = pr0 * eb.x;
                c[3] = pr1 * eb.y;
            }
        } else {
            const uint32_t *oph = opb + ((k - 1) & 1) * 2 * OP, *opl = oph + OP;
            float ch[4] = {0.f, 0.f, 0.f, 0.f}, cl[4] = {0.f, 0.f, 0.f, 0.f}, cm[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
            for (int j = 0; j < NT; ++j) {
                const int o0 = rA * LD + 8 * j + tq, o1 = rB * LD + 8 * j + tq;
                const uint32_t ah[4] = {oph[o0], oph[o1], oph[o0 + 4], oph[o1 + 4]};
                const uint32_t al[4] = {opl[o0], opl[o1], opl[o0 + 4], opl[o1 + 4]};
                mma_tf32(cl, al, bh[j][0], bh[j][1]);
                mma_tf32(cm, ah, bl[j][0], bl[j][1]);
                mma_tf32(ch, ah, bh[j][0], bh[j][1]);
            }
            const float scA = pow2_neg(EA), scB = pow2_neg(EB);
            if (!backward) {
                esumA += EA;
                esumB += EB;
            }
#pragma unroll
            for (int r = 0; r < 4; ++r) c[r] = (ch[r] + (cl[r] + cm[r])) * (r < 2 ? scA : scB);
            if (!backward) {   // u_t = (u_{t-1} A) 2^-E .* e_t
                c[0] *= ea.x;
                c[1] *= ea.y;
                c[2] *= eb.x;
                c[3] *= eb.y;
            }
        }
        // messages out; the next operand (u_t, or x_t = e_t .* b_t) into the tile; row-sum partials
        if (vA) *reinterpret_cast<float2 *>(oA) = make_float2(c[0], c[1]);
        if (vB) *reinterpret_cast<float2 *>(oB) = make_float2(c[2], c[3]);
        oA += dtN;
        oB += dtN;
        if (backward) {
            c[0] *= ea.x;
            c[1] *= ea.y;
            c[2] *= eb.x;
            c[3] *= eb.y;
        }
        {   // the producer splits its own values: the consumers read hi and lo fragments directly
            uint32_t *oh = opb + (k & 1) * 2 * OP, *ol = oh + OP;
            uint32_t h[4], l[4];
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                h[r] = tf32_hi_bits(c[r]);
                l[r] = __float_as_uint(c[r] - __uint_as_float(h[r]));
            }
            *reinterpret_cast<uint2 *>(oh + rA * LD + col) = make_uint2(h[0], h[1]);
            *reinterpret_cast<uint2 *>(oh + rB * LD + col) = make_uint2(h[2], h[3]);
            *reinterpret_cast<uint2 *>(ol + rA * LD + col) = make_uint2(l[0], l[1]);
            *reinterpret_cast<uint2 *>(ol + rB * LD + col) = make_uint2(l[2], l[3]);
        }
        float pa = c[0] + c[1], pb = c[2] + c[3];
        pa += __shfl_xor_sync(0xffffffffu, pa, 1);
        pa += __shfl_xor_sync(0xffffffffu, pa, 2);
        pb += __shfl_xor_sync(0xffffffffu, pb, 1);
        pb += __shfl_xor_sync(0xffffffffu, pb, 2);
        float *rp = rsp + (k & 1) * NT * 16;
        if (tq == 0) {
            rp[warp * 16 + rA] = pa;
            rp[warp * 16 + rB] = pb;
        }
        asm volatile("bar.sync 1, %0;\n" ::"r"(bar_n) : "memory");
        float ta = 0.f, tb = 0.f;   // the rows' full sums, column tiles in a fixed order
#pragma unroll
        for (int i = 0; i < NT; ++i) {
            ta += rp[i * 16 + rA];
            tb += rp[i * 16 + rB];
        }
        if ((vA && (!(ta > 0.f) || !(ta < INFINITY))) || (vB && (!(tb > 0.f) || !(tb < INFINITY)))) bad |= FLAG_NONFINITE;
        EA = ta > 0.f ? exponent_of(ta) : 0;
        EB = tb > 0.f ? exponent_of(tb) : 0;
        sumA = ta;
        sumB = tb;
    }
    cp_async_wait_all();
    if (!backward && warp == 0) {   // log Z = ln(sum u_{T-1}) + ln 2 sum E + sum_t eoff_t, per row
        double oa = 0.0, ob = 0.0;
        for (int tt = tq; tt < T; tt += 4) {
            if (vA) oa += p.eoff[chA * T + tt];
            if (vB) ob += p.eoff[chB * T + tt];
        }
        oa += __shfl_xor_sync(0xffffffffu, oa, 1);
        oa += __shfl_xor_sync(0xffffffffu, oa, 2);
        ob += __shfl_xor_sync(0xffffffffu, ob, 1);
        ob += __shfl_xor_sync(0xffffffffu, ob, 2);
        if (tq == 0) {
            if (vA) {
                const double lz = log((double)sumA) + (double)esumA * 0.69314718055994530942 + oa;
                p.logZ[chA] = lz;
                if (!isfinite(lz)) bad |= FLAG_NONFINITE;
            }
            if (vB) {
                const double lz = log((double)sumB) + (double)esumB * 0.69314718055994530942 + ob;
                p.logZ[chB] = lz;
                if (!isfinite(lz)) bad |= FLAG_NONFINITE;
            }
        }
    }
    if (bad) atomicOr(p.flags, bad);
}

template <int NT>
cudaError_t launch_fb_mma(const FBArgs &a, cudaStream_t st) {
    using C_ = FBTCfg<NT>;
    const size_t smem = (size_t)C_::FLOATS * 4;
    cudaError_t e = ensure_dyn_smem((const void *)fb_mma_kernel<NT>, smem);
    if (e != cudaSuccess) return e;
    fb_mma_kernel<NT><<<a.S * 2 * ((a.M + 15) / 16), NT * 32, smem, st>>>(a);
    return cudaGetLastError();
}

bool fb_mma_supported(int N, int64_t M, int nchunk) { return nchunk <= 1 && M >= 16 && (N == 40 || N == 48 || N == 32 || N == 64 || N == 24 || N == 16); }

bool fb_multi_supported(int N, int64_t M, int nchunk) {
    return nchunk <= 1 && M >= 2 && (N == 40 || N == 36 || N == 48 || N == 8 || N == 4 || N == 16);
}

int fb_pick_chunks(int64_t chains, int64_t T, int N, int *chunk_len) {
    // Parallel in time only while the sequential recursion would leave most of the GPU idle (at most
    // 32 chains -- e.g. single-mixture configurations), for N <= 64 (phase-2 smem) and long enough sequences.  Chunk length ~ sqrt(T): phase 1
    // costs ~L matrix products per chunk, phase 2 ~T/L vector-matrix products per chain.
    int max_chains = 32;
    if (const char *e = getenv("NFHMM_FB_PARALLEL_MAX")) max_chains = atoi(e);   // experiments (chain bound)
    if (chains > max_chains || N > 64 || T < 96) return 0;
    // chunk length ~ sqrt(2.3 T) in multiples of 16 (round 2 sweep, frame-iterations/s: config 1 (T = 1000)
    // L = 24 / 32 / 48 / 64 / 96 -> 7.3 / 7.6 / 8.2 / 7.9 / 7.4 M; config 2 (T = 2000) 32 / 48 / 64 / 96 ->
    // 9.5 / 10.2 / 10.3 / 10.2 M): the transfer and re-run phases cost ~L steps, the scan ~T / L chunks
    int L = 16 * (int)lround(sqrt(2.3 * (double)T) / 16.0);
    if (L < 32) L = 32;
    if (L > 256) L = 256;
    if (const char *e = getenv("NFHMM_FB_CHUNK")) {   // experiments (chunk length)
        const int l = atoi(e);
        if (l >= 8 && l <= 1024) L = l;
    }
    // phase 2 keeps every chunk's row scales in shared memory: grow the chunks until it fits (the
    // template bucket NMAX of N as in launch_fb); past L = 4096 keep the sequential kernel
    const int NMAX = N <= 4 ? 4 : N <= 8 ? 8 : N <= 16 ? 16 : N <= 24 ? 24 : N <= 32 ? 32 : N <= 40 ? 40 : N <= 48 ? 48 : 64;
    auto scan_smem = [&](int64_t nc) {
        return ((int64_t)2 * NMAX * NMAX + 2 * (nc * NMAX + (int64_t)FBP_RING * (NMAX * NMAX + 2 * NMAX) + 2 * NMAX)) * 4;
    };
    // phase 1 stages one chunk of emissions: (NMAX^2 + L NMAX + 8 NMAX) floats
    auto transfer_smem = [&](int64_t l) { return ((int64_t)NMAX * NMAX + l * NMAX + (int64_t)FBP_ROWS * 2 * NMAX) * 4; };
    const int64_t limit = 227 * 1024;
    while (scan_smem((T + L - 1) / L) > limit && L < 4096) L *= 2;
    if (scan_smem((T + L - 1) / L) > limit || transfer_smem(L) > limit) return 0;
    *chunk_len = L;
    return (int)((T + L - 1) / L);
}

cudaError_t launch_fb(const FBArgs &a, cudaStream_t st) {
    const int N = a.N;
    // many chains per source: 16 chains per warp on the tensor cores (multi == 2, default), or C chains per
    // warp with the remainder states spread over the lanes (multi == 1)
    if (a.multi == 2 && fb_mma_supported(N, a.M, a.nchunk)) {
        if (N == 40) return launch_fb_mma<5>(a, st);
        if (N == 48) return launch_fb_mma<6>(a, st);
        if (N == 32) return launch_fb_mma<4>(a, st);
        if (N == 64) return launch_fb_mma<8>(a, st);
        if (N == 24) return launch_fb_mma<3>(a, st);
        if (N == 16) return launch_fb_mma<2>(a, st);
    }
    if (a.multi && fb_multi_supported(N, a.M, a.nchunk)) {
        if (N == 40) return launch_fb_multi<1, 8>(a, st);
        if (N == 36) return launch_fb_multi<1, 4>(a, st);
        if (N == 48) return launch_fb_multi<1, 16>(a, st);
        if (N == 8) return launch_fb_multi<0, 8>(a, st);
        if (N == 4) return launch_fb_multi<0, 4>(a, st);
        if (N == 16) return launch_fb_multi<0, 16>(a, st);
    }
    if (a.wide == 2 && a.nchunk <= 1 && N > 32 && N <= 64) {   // experiment: multi-warp kernel for few chains
        if (N <= 40) return launch_fb_wide<40>(a, st);
        if (N <= 64) return launch_fb_wide<64>(a, st);
    }
    if (N <= 4) return launch_fb_t<4>(a, st);
    if (N <= 8) return launch_fb_t<8>(a, st);
    if (N <= 16) return launch_fb_t<16>(a, st);
    if (N <= 24) return launch_fb_t<24>(a, st);
    if (N <= 32) return launch_fb_t<32>(a, st);
    if (N <= 40) return launch_fb_t<40>(a, st);
    if (N <= 48) return launch_fb_t<48>(a, st);
    if (N <= 64) return launch_fb_t<64>(a, st);
    // N > 64 (never parallel in time): a CTA of ceil(N/32) warps per chain and direction (fb_wide_kernel,
    // 6.3x faster at N = 100); a.wide = 0 (NFHMM_FB_WIDE=0) keeps the one-warp kernel with A in shared
    // memory.  (The multi-warp kernel at N = 40 measured 3 % slower than fb_kernel<40>.)
    if (a.wide && a.nchunk <= 1) {
        if (N <= 96) return launch_fb_wide<96>(a, st);
        if (N <= 104) return launch_fb_wide<104>(a, st);
        if (N <= 128) return launch_fb_wide<128>(a, st);
    }
    if (N <= 96) return launch_fb_t<96>(a, st);
    if (N <= 104) return launch_fb_t<104>(a, st);
    if (N <= 128) return launch_fb_t<128>(a, st);
    return cudaErrorInvalidValue;
}

}  // namespace nfk
