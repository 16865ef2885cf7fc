// misc.cu -- small kernels around the VB sweep: (g) the FP64 bound reduction, Section 4's ratio mask
// (part of (f)), initial state, observation statistics, the dictionary transpose.
#include <cuda_runtime.h>
#include <math.h>

#include <map>
#include <mutex>
#include <tuple>

#include "nfhmm_internal.cuh"

namespace nfk {

namespace {

__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// (g) L_i[m] = sum_t (sum_tiles data_part[t] + hdir[t]) + sum_s log Z[m][s] + T c_prior   (DESIGN R8)
// One CTA per mixture, fixed-order FP64 reduction: bitwise independent of how mixtures are sharded.
// The sweep index comes from a device counter (so that a CUDA graph of one sweep can be replayed): every
// block reads it, and the last block to finish advances it.
__global__ void __launch_bounds__(256) elbo_kernel(ElboArgs p) {
    __shared__ double scratch[8];
    __shared__ bool last_m;
    const int m = blockIdx.x, nb = gridDim.y, b = blockIdx.y;   // mixtures on x (no 65535 cap)
    const int iter = *p.iter_ctr;
    const int chunk = (p.T + nb - 1) / nb, t0 = b * chunk, t1 = min(p.T, t0 + chunk);
    double acc = 0.0;
    for (int t = t0 + threadIdx.x; t < t1; t += blockDim.x) {
        const size_t f = (size_t)m * p.T + t;
        // data term: integer-valued partials in units of 2^-20 nats (exact sum, any tiling)
        double q = 0.0;
        for (int c = 0; c < p.n_tiles; ++c) q += p.data_part[f * p.n_tiles + c];
        acc += p.hdir[f] + q * (1.0 / 1048576.0);
    }
    acc = warp_sum_d(acc);
    if ((threadIdx.x & 31) == 0) scratch[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        double s = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += scratch[w];
        p.part[(size_t)m * ELBO_MAX_BLOCKS + b] = s;
        __threadfence();
        last_m = atomicAdd(&p.mix_ctr[m], 1u) == (unsigned)nb - 1;
    }
    __syncthreads();
    if (!last_m || threadIdx.x != 0) return;
    // the mixture's last block: partials in block order (deterministic), then the chain and prior terms
    __threadfence();
    double s = 0.0;
    for (int k = 0; k < nb; ++k) s += ((volatile double *)p.part)[(size_t)m * ELBO_MAX_BLOCKS + k];
    for (int k = 0; k < p.S; ++k) s += p.logZ[(size_t)m * p.S + k];
    s += p.c_prior_T;
    if (iter < p.max_iters) p.fe[(size_t)m * p.max_iters + iter] = s;
    p.mix_ctr[m] = 0u;
    __threadfence();
    if (atomicAdd(p.done_ctr, 1u) == gridDim.x - 1) {   // the last mixture advances the sweep counter
        *p.done_ctr = 0u;
        *p.iter_ctr = iter + 1;
        __threadfence();
    }
}

__device__ double digamma_fp64(double x);

// DESIGN R5: alpha = a0 = 1 + gamma/N, theta~ = exp(psi(a0) - psi(Kt a0)) (uniform; FP64 digamma below)
__global__ void init_state_kernel(int frames, int ld, int Kt, double a0, float *alpha, float *theta) {
    __shared__ float th0_s;
    if (threadIdx.x == 0) th0_s = (float)exp(digamma_fp64(a0) - digamma_fp64(a0 * (double)Kt));
    __syncthreads();
    const float th0 = th0_s, a0f = (float)a0;
    const size_t n = (size_t)frames * ld;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        const int k = (int)(i % ld);
        alpha[i] = k < Kt ? a0f : 0.f;
        theta[i] = k < Kt ? th0 : 0.f;
    }
}

// d[r][n] = u[r][n] b[r][n] / sum_n u[r][n] b[r][n]: q(D) marginals from the FB messages (warp per row)
__global__ void marginals_kernel(const float *__restrict__ u, const float *__restrict__ b, float *__restrict__ d,
                                 long long rows, int N) {
    const long long r = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (r >= rows) return;
    float s = 0.f;
    for (int n = lane; n < N; n += 32) s += u[r * N + n] * b[r * N + n];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    const float is = 1.f / s;
    for (int n = lane; n < N; n += 32) d[r * N + n] = u[r * N + n] * b[r * N + n] * is;
}

__global__ void fill_kernel(float *p, long long n, float v) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        p[i] = v;
}

__global__ void transpose_kernel(const float *__restrict__ src, int rows, int cols, int lds, float *__restrict__ dst,
                                 int ldd) {
    __shared__ float tile[32][33];
    const int c0 = blockIdx.x * 32, r0 = blockIdx.y * 32;
    for (int i = threadIdx.y; i < 32; i += blockDim.y) {
        const int r = r0 + i, c = c0 + threadIdx.x;
        tile[i][threadIdx.x] = (r < rows && c < cols) ? src[(size_t)r * lds + c] : 0.f;
    }
    __syncthreads();
    for (int i = threadIdx.y; i < 32; i += blockDim.y) {
        const int c = c0 + i, r = r0 + threadIdx.x;
        if (c < cols && r < rows) dst[(size_t)c * ldd + r] = tile[threadIdx.x][i];
    }
}

// v_t = sum_l V_lt (FP64 accumulation) and input checks (V >= 0, finite) -- one warp per frame.
__global__ void obs_stats_kernel(const float *__restrict__ V, int frames, int F, int ld, float *vt, unsigned *flags) {
    const long long w = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (w >= frames) return;
    double s = 0.0;
    unsigned bad = 0;
    for (int l = lane; l < F; l += 32) {
        const float v = V[(size_t)w * ld + l];
        if (!(v >= 0.f) || !isfinite(v)) bad = FLAG_BAD_INPUT;
        s += (double)v;
    }
    s = warp_sum_d(s);
    if (lane == 0) vt[w] = (float)s;
    if (bad) atomicOr(flags, bad);
}

// scale_t = v_t / alpha_0 (posterior mean E[theta] = alpha / alpha_0, DESIGN R9; v_t from S:408).
__device__ double digamma_fp64(double x) {
    double r = 0.0;
    while (x < 10.0) {
        r -= 1.0 / x;
        x += 1.0;
    }
    const double f = 1.0 / (x * x);
    const double t = f * (-1.0 / 12 + f * (1.0 / 120 + f * (-1.0 / 252 + f * (1.0 / 240 + f * (-1.0 / 132 +
                     f * (691.0 / 32760 + f * (-1.0 / 12)))))));
    return r + log(x) - 0.5 / x + t;
}

// alpha_0 = v_t + Kt + gamma S K (Eq. 6 summed over k; DESIGN R19) and the frame's scalar bound terms
__global__ void frame_consts_kernel(const float *__restrict__ vt, int frames, int Kt, double gamma, int S, int K,
                                    double *fc) {
    const int f = blockIdx.x * blockDim.x + threadIdx.x;
    if (f >= frames) return;
    const double a0 = (double)vt[f] + (double)Kt + gamma * (double)S * (double)K;
    const double psi0 = digamma_fp64(a0);
    fc[4 * (size_t)f + 0] = a0;
    fc[4 * (size_t)f + 1] = psi0;
    fc[4 * (size_t)f + 2] = -a0 - lgamma(a0) + (a0 - (double)Kt) * psi0;
    fc[4 * (size_t)f + 3] = exp(-psi0);
}

__global__ void sep_scale_kernel(const float *__restrict__ alpha, int frames, int Kt, int ld, const float *vt, float *scale) {
    const long long w = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (w >= frames) return;
    double s = 0.0;
    for (int k = lane; k < Kt; k += 32) s += (double)alpha[(size_t)w * ld + k];
    s = warp_sum_d(s);
    if (lane == 0) scale[w] = (float)((double)vt[w] / s);
}

// P:203  V*^(s) = V V_src^(s) / sum_s' V_src^(s');  1/S where the denominator is 0.
__global__ void wiener_kernel(const float *__restrict__ V, int ldv, const float *vsrc, float *vstar, int M, int S,
                              int T, int F) {
    const size_t n = (size_t)M * T * F;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        const int l = (int)(i % F);
        const size_t mt = i / F;
        const int t = (int)(mt % T), m = (int)(mt / T);
        const float v = V[mt * ldv + l];
        float den = 0.f;
        for (int s = 0; s < S; ++s) den += vsrc[((size_t)(m * S + s) * T + t) * F + l];
        for (int s = 0; s < S; ++s) {
            const size_t o = ((size_t)(m * S + s) * T + t) * F + l;
            vstar[o] = den > 0.f ? v * (vsrc[o] / den) : v / (float)S;
        }
    }
}

int grid_for(size_t n, int block) {
    size_t g = (n + block - 1) / block;
    if (g > 148 * 32) g = 148 * 32;
    if (g < 1) g = 1;
    return (int)g;
}

}  // namespace

cudaError_t launch_elbo(const ElboArgs &a, cudaStream_t st) {
    int nb = (a.T + 255) / 256;
    nb = nb < 1 ? 1 : (nb > ELBO_MAX_BLOCKS ? ELBO_MAX_BLOCKS : nb);
    elbo_kernel<<<dim3(a.M, nb), 256, 0, st>>>(a);
    return cudaGetLastError();
}

// alpha, theta of DESIGN R5; u = b = 1 so that the marginals u .* b / sum are the uniform d = 1/N
cudaError_t launch_init_state(int frames, int ld, int Kt, double alpha0, float *alpha, float *theta, float *u_fwd,
                              float *b_bwd, long long d_count, cudaStream_t st) {
    init_state_kernel<<<grid_for((size_t)frames * ld, 256), 256, 0, st>>>(frames, ld, Kt, alpha0, alpha, theta);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    fill_kernel<<<grid_for((size_t)d_count, 256), 256, 0, st>>>(u_fwd, d_count, 1.f);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    fill_kernel<<<grid_for((size_t)d_count, 256), 256, 0, st>>>(b_bwd, d_count, 1.f);
    return cudaGetLastError();
}

cudaError_t launch_marginals(const float *u, const float *b, float *d, long long rows, int N, cudaStream_t st) {
    marginals_kernel<<<(unsigned)((rows * 32 + 255) / 256), 256, 0, st>>>(u, b, d, rows, N);
    return cudaGetLastError();
}

cudaError_t launch_transpose(const float *src, int rows, int cols, int ld_src, float *dst, int ld_dst, cudaStream_t st) {
    dim3 grid((cols + 31) / 32, (rows + 31) / 32), block(32, 8);
    transpose_kernel<<<grid, block, 0, st>>>(src, rows, cols, ld_src, dst, ld_dst);
    return cudaGetLastError();
}

cudaError_t launch_obs_stats(const float *V, int frames, int F, int ld, float *vt, unsigned *flags, cudaStream_t st) {
    obs_stats_kernel<<<(unsigned)(((long long)frames * 32 + 255) / 256), 256, 0, st>>>(V, frames, F, ld, vt, flags);
    return cudaGetLastError();
}

cudaError_t launch_frame_consts(const float *vt, int frames, int Kt, double gamma, int S, int K, double *fc,
                                cudaStream_t st) {
    frame_consts_kernel<<<(frames + 127) / 128, 128, 0, st>>>(vt, frames, Kt, gamma, S, K, fc);
    return cudaGetLastError();
}

cudaError_t launch_sep_scale(const float *alpha, int frames, int Kt, int ld, const float *vt, float *scale,
                             cudaStream_t st) {
    sep_scale_kernel<<<(unsigned)(((long long)frames * 32 + 255) / 256), 256, 0, st>>>(alpha, frames, Kt, ld, vt, scale);
    return cudaGetLastError();
}

cudaError_t launch_wiener(const float *V, int ldv, const float *vsrc, float *vstar, int M, int S, int T, int F,
                          cudaStream_t st) {
    wiener_kernel<<<grid_for((size_t)M * T * F, 256), 256, 0, st>>>(V, ldv, vsrc, vstar, M, S, T, F);
    return cudaGetLastError();
}

namespace {
std::mutex g_launch_mu;
std::map<std::pair<const void *, int>, size_t> g_smem_attr;
std::map<int, int> g_sms;
std::map<std::tuple<const void *, int, int, size_t>, int> g_occ;
int current_device() {
    int dev = 0;
    cudaGetDevice(&dev);
    return dev;
}
}  // namespace

cudaError_t ensure_dyn_smem(const void *func, size_t bytes) {
    if (bytes <= 48 * 1024) return cudaSuccess;
    const int dev = current_device();
    std::lock_guard<std::mutex> lk(g_launch_mu);
    size_t &done = g_smem_attr[{func, dev}];
    if (done >= bytes) return cudaSuccess;
    cudaError_t e = cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    if (e == cudaSuccess) done = bytes;
    return e;
}

int device_sms() {
    const int dev = current_device();
    std::lock_guard<std::mutex> lk(g_launch_mu);
    int &n = g_sms[dev];
    if (!n) {
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        if (n < 1) n = 1;
    }
    return n;
}

int occupancy_ctas(const void *func, int threads, size_t smem) {
    const int dev = current_device();
    std::lock_guard<std::mutex> lk(g_launch_mu);
    int &n = g_occ[std::make_tuple(func, dev, threads, smem)];
    if (!n) {
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, func, threads, smem);
        if (n < 1) n = 1;
    }
    return n;
}

}  // namespace nfk
