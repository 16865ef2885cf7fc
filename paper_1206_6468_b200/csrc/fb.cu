// fb.cu -- kernel (e): scaled forward-backward per source chain, batched over all mixtures.
//
// q(D^(s)) is the chain posterior with log-likelihood gamma * phi (DESIGN R1).  One warp
// per chain (m, s); lane l owns states j = l + 32 q (q < NQ).  Chains of the same source share a CTA
// so A_s (row-stochastic, A[i][j] = P(j | i), DESIGN R4) is staged once in shared memory in both
// orientations (conflict-free lane access in the forward and backward recursions).
//
// Forward with a deferred normaliser (keeps the warp reduction off the dependency chain):
//   u_0 = pi .* e_0;  w_t = (u_{t-1} A) .* e_t;  c_{t-1} = sum u_{t-1};  u_t = w_t / c_{t-1};
//   a_{t-1} = u_{t-1} / c_{t-1} (normalised message, stored);  log Z = sum_t log c_t + sum_t eoff_t.
// Backward: b_{T-1} = 1;  b_t = A (e_{t+1} .* b_{t+1}) / c_{t+1};  d_t = a_t .* b_t / sum.
// Emissions e = exp(ec) with ec <= 0 the centred gamma*phi; their FP64 offsets eoff enter log Z only.
// Inputs for the next CH steps are staged into shared memory with cp.async (double-buffered chunks).
#include <cuda_runtime.h>
#include <math.h>

#include "nfhmm_internal.cuh"

namespace nfk {

namespace {

constexpr int WPB = 4;     // chains (warps) per CTA
template <int NQ>
struct Chunk { static constexpr int CH = NQ <= 2 ? 32 : 16; };   // time steps per staged chunk

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

template <int NQ>
__global__ void __launch_bounds__(WPB * 32) fb_kernel(FBArgs p) {
    constexpr int CH = Chunk<NQ>::CH;
    extern __shared__ __align__(16) float sm[];
    const int N = p.N;
    float *As = sm;                      // [N][N]   A[i][j]
    float *AT = As + N * N;              // [N][N]   A[j][i] at AT[j*N + i]... i.e. AT[i][j] = A[j][i]
    float *wbase = AT + N * N;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // per-warp: u[2][N] | e chunks [2][CH][N] | a chunks [2][CH][N] | cinv chunks [2][CH]
    const int per_warp = 2 * N + 4 * CH * N + 2 * CH;
    float *ubuf = wbase + warp * per_warp;
    float *ech = ubuf + 2 * N;
    float *ach = ech + 2 * CH * N;
    float *cch = ach + 2 * CH * N;

    const int s = blockIdx.y;
    const int m = blockIdx.x * WPB + warp;
    const float *Ag = p.trans + (size_t)s * N * N;
    for (int i = threadIdx.x; i < N * N; i += blockDim.x) {
        const float v = Ag[i];
        As[i] = v;
        const int r = i / N, c = i - r * N;
        AT[c * N + r] = v;
    }
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

    // sum of the FP64 emission offsets (lane-parallel, fixed order)
    double offsum = 0.0;
    for (int t = lane; t < T; t += 32) offsum += p.eoff[chain * T + t];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) offsum += __shfl_xor_sync(0xffffffffu, offsum, o);

    // ---------------- forward ----------------
    const int nch = (T + CH - 1) / CH;
    stage_rows(ech, ec, N, 0, min(CH, T), lane);
    double mant = 1.0;   // running product of c_t as mantissa * 2^expo (exact scaling, FP64)
    long long expo = 0;
    float u[NQ];
    for (int c = 0; c < nch; ++c) {
        const int t0 = c * CH, n = min(CH, T - t0);
        float *ecur = ech + (c & 1) * CH * N;
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
                const float *up = ubuf + ((t - 1) & 1) * N;
                float acc0[NQ], acc1[NQ];
#pragma unroll
                for (int q = 0; q < NQ; ++q) acc0[q] = acc1[q] = 0.f;
                int i = 0;
                for (; i + 1 < N; i += 2) {
                    const float x0 = up[i], x1 = up[i + 1];
#pragma unroll
                    for (int q = 0; q < NQ; ++q)
                        if (jv[q]) {
                            acc0[q] = fmaf(x0, As[i * N + js[q]], acc0[q]);
                            acc1[q] = fmaf(x1, As[(i + 1) * N + js[q]], acc1[q]);
                        }
                }
                if (i < N) {
                    const float x0 = up[i];
#pragma unroll
                    for (int q = 0; q < NQ; ++q)
                        if (jv[q]) acc0[q] = fmaf(x0, As[i * N + js[q]], acc0[q]);
                }
                // c_{t-1} from the previous (unnormalised) message, reduced while the dot ran
                float ps = 0.f;
#pragma unroll
                for (int q = 0; q < NQ; ++q) ps += u[q];
                const float ct = warp_sum(ps);
                const float ic = 1.f / ct;
                if (!(ct > 0.f)) bad |= FLAG_NONFINITE;
                // store normalised a_{t-1} and 1/c_{t-1}
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
                for (int q = 0; q < NQ; ++q) u[q] = (acc0[q] + acc1[q]) * e[q] * ic;
            }
            float *un = ubuf + (t & 1) * N;
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
    // chunk c covers t in [t0, t0 + n) processed in descending t; needs e_{t+1}, cinv_{t+1}, a_t.
    float b[NQ];
#pragma unroll
    for (int q = 0; q < NQ; ++q) b[q] = 1.f;
    // stage the last chunk: a rows [t0, T), e rows [t0+1, T) shifted, cinv [t0+1, T)
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
        float *acur = ach + buf * CH * N;
        float *ecur = ech + buf * CH * N;   // row r holds e_{t0 + 1 + r}
        float *ccur = cch + buf * CH;       // ccur[r] = cinv_{t0 + 1 + r}
        cp_async_wait_all();
        __syncwarp();
        if (c > 0) stage_back(c - 1, buf ^ 1);
        for (int tt = n - 1; tt >= 0; --tt) {
            const int t = t0 + tt;
            if (t < T - 1) {
                // x_{t+1} = e_{t+1} .* b_{t+1}; b_t = A x / c_{t+1}
                float *xb = ubuf + (t & 1) * N;
#pragma unroll
                for (int q = 0; q < NQ; ++q)
                    if (jv[q]) xb[js[q]] = expf(ecur[tt * N + js[q]]) * b[q];
                __syncwarp();
                float acc0[NQ], acc1[NQ];
#pragma unroll
                for (int q = 0; q < NQ; ++q) acc0[q] = acc1[q] = 0.f;
                int j = 0;
                for (; j + 1 < N; j += 2) {
                    const float x0 = xb[j], x1 = xb[j + 1];
#pragma unroll
                    for (int q = 0; q < NQ; ++q)
                        if (jv[q]) {
                            acc0[q] = fmaf(AT[j * N + js[q]], x0, acc0[q]);
                            acc1[q] = fmaf(AT[(j + 1) * N + js[q]], x1, acc1[q]);
                        }
                }
                if (j < N) {
                    const float x0 = xb[j];
#pragma unroll
                    for (int q = 0; q < NQ; ++q)
                        if (jv[q]) acc0[q] = fmaf(AT[j * N + js[q]], x0, acc0[q]);
                }
                const float ic = ccur[tt];
#pragma unroll
                for (int q = 0; q < NQ; ++q) b[q] = (acc0[q] + acc1[q]) * ic;
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

template <int NQ>
cudaError_t launch_fb_t(const FBArgs &a, cudaStream_t st) {
    const int N = a.N;
    constexpr int CH = Chunk<NQ>::CH;
    const size_t smem = ((size_t)2 * N * N + (size_t)WPB * (2 * N + 4 * CH * N + 2 * CH)) * sizeof(float);
    static size_t attr = 0;
    if (smem > 48 * 1024 && attr < smem) {
        cudaError_t e = cudaFuncSetAttribute(fb_kernel<NQ>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        attr = smem;
    }
    dim3 grid((a.M + WPB - 1) / WPB, a.S);
    fb_kernel<NQ><<<grid, WPB * 32, smem, st>>>(a);
    return cudaGetLastError();
}

}  // namespace

cudaError_t launch_fb(const FBArgs &a, cudaStream_t st) {
    const int nq = (a.N + 31) / 32;
    switch (nq) {
        case 1: return launch_fb_t<1>(a, st);
        case 2: return launch_fb_t<2>(a, st);
        case 3: return launch_fb_t<3>(a, st);
        case 4: return launch_fb_t<4>(a, st);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace nfk
