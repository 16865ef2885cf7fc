// stft.cu -- the spectrogram front end and the resynthesis back end around the VB path (SURVEY §8(f)
// NEXT-4): nfhmm_stft (waveform -> complex STFT and the quanta V = gain |X|) and nfhmm_istft (separated
// magnitudes + the mixture's phase -> waveforms).
//
//   P:30   "A spectrogram is the magnitude of the short-time Fourier transform (STFT) of a signal";
//   P:219  "a window size of 64ms and a hop size of 16ms (the sampling rate was 16KHz)"  (L = 1024, H = 256);
//   P:201  "go back to the time domain with these estimates using the phase of the original mixture".
// Window: periodic Hann w[n] = 1/2 - 1/2 cos(2 pi n / L), DFT length = window length (DESIGN R23).
//   X_t[k] = sum_n w[n] x[t H + n] e^{-2 pi i k n / L},  k <= L/2;   V = gain |X|;
//   Y_t[k] = M_t[k] X_t[k] / |X_t[k]| (0 where X = 0), Hermitian;  y_t = real IDFT(Y_t) / L;
//   y[n] = sum_t w[n - t H] y_t[n - t H] / sum_t w[n - t H]^2   (weighted overlap-add, fixed frame order).
// Each frame is a radix-2 FFT in shared memory (one CTA per frame, log2 L barrier-separated butterfly
// stages, twiddles from sincospif); the overlap-add is a separate gather kernel (one thread per output
// sample, frames in ascending order), so the results are deterministic.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "nfhmm_internal.cuh"

namespace nfk {
namespace {

constexpr int FFT_THREADS = 256;

__device__ __forceinline__ float hann_w(int n, int L) { return 0.5f - 0.5f * cospif(2.f * (float)n / (float)L); }

__device__ __forceinline__ unsigned bitrev(unsigned x, int bits) { return __brev(x) >> (32 - bits); }

// in-place radix-2 FFT of s[L] (bit-reversed input order); sign = +1 forward (twiddles e^{-2 pi i k / L}),
// -1 inverse (their conjugates; unscaled)
__device__ void fft_smem(float2 *s, const float2 *tw, int L, int bits, float sign) {
    for (int st = 1; st <= bits; ++st) {
        const int half = 1 << (st - 1), stride = L >> st;   // twiddle index step
        for (int j = threadIdx.x; j < L / 2; j += blockDim.x) {
            const int g = j >> (st - 1), pos = j & (half - 1);
            const int i0 = (g << st) + pos, i1 = i0 + half;
            float2 w = tw[pos * stride];
            w.y *= sign;
            const float2 a = s[i0], b = s[i1];
            const float2 bw = make_float2(b.x * w.x - b.y * w.y, b.x * w.y + b.y * w.x);
            s[i0] = make_float2(a.x + bw.x, a.y + bw.y);
            s[i1] = make_float2(a.x - bw.x, a.y - bw.y);
        }
        __syncthreads();
    }
}

__device__ void twiddles(float2 *tw, int L) {   // tw[k] = e^{-2 pi i k / L}, k < L/2
    for (int k = threadIdx.x; k < L / 2; k += blockDim.x) {
        float sn, cs;
        sincospif(-2.f * (float)k / (float)L, &sn, &cs);
        tw[k] = make_float2(cs, sn);
    }
}

// one CTA per (signal, frame): windowed frame -> X [sig][T][F] (complex interleaved), V = gain |X|
__global__ void __launch_bounds__(FFT_THREADS) stft_kernel(const float *x, int64_t n_samples, int L, int bits, int H,
                                                           int T, float gain, float2 *X, float *V) {
    extern __shared__ __align__(16) float2 ssm[];
    float2 *s = ssm, *tw = ssm + L;
    const int t = blockIdx.x;
    const int64_t sig = blockIdx.y;
    const float *xs = x + sig * n_samples + (int64_t)t * H;
    twiddles(tw, L);
    for (int n = threadIdx.x; n < L; n += blockDim.x) s[bitrev(n, bits)] = make_float2(hann_w(n, L) * xs[n], 0.f);
    __syncthreads();
    fft_smem(s, tw, L, bits, 1.f);
    const int F = L / 2 + 1;
    const int64_t row = (sig * T + t) * F;
    for (int k = threadIdx.x; k < F; k += blockDim.x) {
        const float2 v = s[k];
        if (X) X[row + k] = v;
        if (V) V[row + k] = gain * hypotf(v.x, v.y);
    }
}

// one CTA per (mixture, source, frame): Y = M X / |X| (Hermitian), inverse FFT, / L, times the window
// -> frames [mix][src][T][L]
__global__ void __launch_bounds__(FFT_THREADS) istft_frame_kernel(const float2 *X, const float *M, int S, int T, int L,
                                                                  int bits, float inv_gain, float *frames) {
    extern __shared__ __align__(16) float2 ssm[];
    float2 *s = ssm, *tw = ssm + L;
    const int t = blockIdx.x, src = blockIdx.y;
    const int64_t mix = blockIdx.z;
    const int F = L / 2 + 1;
    const float2 *xr = X + (mix * T + t) * F;
    const float *mr = M + ((mix * S + src) * T + t) * F;
    twiddles(tw, L);
    for (int k = threadIdx.x; k < L; k += blockDim.x) {
        const int kk = k < F ? k : L - k;
        const float2 xc = xr[kk];
        const float mag = hypotf(xc.x, xc.y);
        const float m = mr[kk] * inv_gain;
        float2 y = mag > 0.f ? make_float2(m * (xc.x / mag), m * (xc.y / mag)) : make_float2(0.f, 0.f);
        if (k >= F) y.y = -y.y;   // Y[L - k] = conj(Y[k])
        s[bitrev(k, bits)] = y;
    }
    __syncthreads();
    fft_smem(s, tw, L, bits, -1.f);
    float *fo = frames + ((mix * S + src) * T + t) * (int64_t)L;
    const float il = 1.f / (float)L;
    for (int n = threadIdx.x; n < L; n += blockDim.x) fo[n] = s[n].x * il * hann_w(n, L);
}

// weighted overlap-add: y[n] = sum_t frame_t[n - t H] / sum_t w[n - t H]^2 (frames in ascending t)
__global__ void ola_kernel(const float *frames, int64_t n_out, int T, int L, int H, float *y) {
    const int64_t n = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (n >= n_out) return;
    const int64_t row = blockIdx.y;   // (mix, src)
    const float *fr = frames + row * (int64_t)T * L;
    int64_t t_lo = n - L + 1 <= 0 ? 0 : (n - L + 1 + H - 1) / H;
    int64_t t_hi = n / H;
    if (t_hi > T - 1) t_hi = T - 1;
    float num = 0.f, den = 0.f;
    for (int64_t t = t_lo; t <= t_hi; ++t) {
        const int off = (int)(n - t * H);
        const float w = hann_w(off, L);
        num += fr[t * L + off];
        den += w * w;
    }
    y[row * n_out + n] = den > 0.f ? num / den : 0.f;
}

bool is_device_ptr(const void *p) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

int log2_exact(int L) {
    int b = 0;
    while ((1 << b) < L) ++b;
    return (1 << b) == L ? b : -1;
}

// device copy of a (possibly host) input; *owned set when a temporary was allocated
template <typename Tp>
cudaError_t stage_in(const Tp *p, size_t count, cudaStream_t st, const Tp **dev, Tp **owned) {
    *owned = nullptr;
    if (is_device_ptr(p)) {
        *dev = p;
        return cudaSuccess;
    }
    Tp *d = nullptr;
    cudaError_t e = cudaMallocAsync(&d, count * sizeof(Tp), st);
    if (e != cudaSuccess) return e;
    e = cudaMemcpyAsync(d, p, count * sizeof(Tp), cudaMemcpyHostToDevice, st);
    *dev = d;
    *owned = d;
    return e;
}

}  // namespace
}  // namespace nfk

using namespace nfk;

extern "C" {

int nfhmm_stft(const float *x, int64_t n_sig, int64_t n_samples, int32_t win, int32_t hop, float gain, float *X, float *V,
               int32_t device, void *stream) {
    const int bits = log2_exact(win);
    if (!x || n_sig < 1 || win < 2 || win > 4096 || bits < 0 || hop < 1 || hop > win || n_samples < win ||
        !(gain > 0.f) || (!X && !V) || n_sig > 65535)
        return NFHMM_EINVAL;
    if (cudaSetDevice(device) != cudaSuccess) return NFHMM_ECUDA;
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t T64 = 1 + (n_samples - win) / hop;
    if (T64 > (int64_t)1 << 30) return NFHMM_EINVAL;
    const int T = (int)T64, F = win / 2 + 1;
    const size_t nout = (size_t)n_sig * T * F;
    const float *xd = nullptr;
    float *xo = nullptr, *Xd = X, *Vd = V, *Xo = nullptr, *Vo = nullptr;
    cudaError_t e = stage_in(x, (size_t)n_sig * n_samples, st, &xd, &xo);
    const bool xh = X && !is_device_ptr(X), vh = V && !is_device_ptr(V);
    if (e == cudaSuccess && xh) e = cudaMallocAsync(&Xo, nout * 8, st), Xd = Xo;
    if (e == cudaSuccess && vh) e = cudaMallocAsync(&Vo, nout * 4, st), Vd = Vo;
    if (e == cudaSuccess) {
        const size_t smem = (size_t)win * 8 + (size_t)win / 2 * 8;
        e = ensure_dyn_smem((const void *)stft_kernel, smem);
        if (e == cudaSuccess) {
            stft_kernel<<<dim3(T, (unsigned)n_sig), FFT_THREADS, smem, st>>>(xd, n_samples, win, bits, hop, T, gain,
                                                                            reinterpret_cast<float2 *>(Xd), Vd);
            e = cudaGetLastError();
        }
    }
    if (e == cudaSuccess && xh) e = cudaMemcpyAsync(X, Xo, nout * 8, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess && vh) e = cudaMemcpyAsync(V, Vo, nout * 4, cudaMemcpyDeviceToHost, st);
    if (xo) cudaFreeAsync(xo, st);
    if (Xo) cudaFreeAsync(Xo, st);
    if (Vo) cudaFreeAsync(Vo, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    return e == cudaSuccess ? NFHMM_OK : NFHMM_ECUDA;
}

int nfhmm_istft(const float *X, const float *M, int64_t n_mix, int32_t S, int64_t T, int32_t win, int32_t hop,
                float gain, float *y, int64_t n_samples, int32_t device, void *stream) {
    const int bits = log2_exact(win);
    if (!X || !M || !y || n_mix < 1 || n_mix > 65535 || S < 1 || S > 65535 || T < 1 || T > ((int64_t)1 << 30) ||
        win < 2 || win > 4096 || bits < 0 || hop < 1 || hop > win || n_samples < 1 || !(gain > 0.f))
        return NFHMM_EINVAL;
    if (cudaSetDevice(device) != cudaSuccess) return NFHMM_ECUDA;
    cudaStream_t st = (cudaStream_t)stream;
    const int F = win / 2 + 1;
    const float *Xd = nullptr, *Md = nullptr;
    float *Xo = nullptr, *Mo = nullptr, *frames = nullptr, *yo = nullptr, *yd = y;
    cudaError_t e = stage_in(X, (size_t)n_mix * T * F * 2, st, &Xd, &Xo);
    if (e == cudaSuccess) e = stage_in(M, (size_t)n_mix * S * T * F, st, &Md, &Mo);
    if (e == cudaSuccess) e = cudaMallocAsync(&frames, (size_t)n_mix * S * T * win * 4, st);
    const bool yh = !is_device_ptr(y);
    const size_t ny = (size_t)n_mix * S * n_samples;
    if (e == cudaSuccess && yh) e = cudaMallocAsync(&yo, ny * 4, st), yd = yo;
    if (e == cudaSuccess) {
        const size_t smem = (size_t)win * 8 + (size_t)win / 2 * 8;
        e = ensure_dyn_smem((const void *)istft_frame_kernel, smem);
        if (e == cudaSuccess) {
            istft_frame_kernel<<<dim3((unsigned)T, S, (unsigned)n_mix), FFT_THREADS, smem, st>>>(
                reinterpret_cast<const float2 *>(Xd), Md, S, (int)T, win, bits, 1.f / gain, frames);
            e = cudaGetLastError();
        }
        if (e == cudaSuccess) {
            ola_kernel<<<dim3((unsigned)((n_samples + 255) / 256), (unsigned)(n_mix * S)), 256, 0, st>>>(
                frames, n_samples, (int)T, win, hop, yd);
            e = cudaGetLastError();
        }
    }
    if (e == cudaSuccess && yh) e = cudaMemcpyAsync(y, yo, ny * 4, cudaMemcpyDeviceToHost, st);
    if (Xo) cudaFreeAsync(Xo, st);
    if (Mo) cudaFreeAsync(Mo, st);
    if (frames) cudaFreeAsync(frames, st);
    if (yo) cudaFreeAsync(yo, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    return e == cudaSuccess ? NFHMM_OK : NFHMM_ECUDA;
}

}  // extern "C"
