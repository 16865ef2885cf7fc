/*
 * stft_oracle.c -- plain, slow, single-threaded FP64 CPU oracle of the spectrogram front end and the
 * resynthesis back end around the VB path (Mysore & Sahani, arXiv 1206.6468).
 *
 * ORACLE -- TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  The product path
 * (paper_1206_6468_b200/, libnfhmm.so) never links, imports or calls it, and it shares no code,
 * header, table or constant with the CUDA path.
 *
 * Citation keys as in nfhmm_oracle.c ("P:n" = PAPER.md line n, "S:n" = SPEC.md line n).
 *
 * Front end ("A spectrogram is the magnitude of the short-time Fourier transform"; "a
 * window size of 64ms and a hop size of 16ms (the sampling rate was 16KHz)"):
 *   w[n] = 1/2 - 1/2 cos(2 pi n / L)  (periodic Hann, L = window length = DFT length; DESIGN R23),
 *   X_t[k] = sum_{n<L} w[n] x[t H + n] exp(-2 pi i k n / L),   k = 0 .. L/2,   t = 0 .. T-1,
 *   T = 1 + (n_samples - L) / H,   V_t[k] = gain |X_t[k]|  (real-valued quanta).
 * Back end ("go back to the time domain with these estimates using the phase of the original
 * mixture"):
 *   Y_t[k] = M_t[k] X_t[k] / |X_t[k]|  (0 where X_t[k] = 0),   Y_t[L-k] = conj(Y_t[k]),
 *   y_t[n] = (1/L) sum_{k<L} Y_t[k] exp(2 pi i k n / L)   (real),
 *   y[n] = sum_t w[n - t H] y_t[n - t H] / sum_t w[n - t H]^2   (weighted overlap-add; 0 where no frame
 *          covers n or the window sum is 0), so istft(stft(x)) = x wherever sum_t w^2 > 0.
 * Every DFT is the definition written out (O(L^2) per frame, FP64 twiddles from the angle).
 *
 * Parity pins: tests/test_stft_oracle.py (numpy.fft on the same frames; round trip; bin-centred
 * sinusoid and DC; Parseval; identity and zero masks; disjoint-band masks).
 */
#include <math.h>
#include <stdlib.h>

#define OR_OK 0
#define OR_EINVAL (-1)

static const double PI = 3.14159265358979323846;

static double hann(int n, int L) { return 0.5 - 0.5 * cos(2.0 * PI * (double)n / (double)L); }

/* x [n_samples] (one signal) -> X [T][F][2] (re, im), V [T][F] (nullable) */
int or_stft(const float *x, int n_samples, int L, int H, double gain, double *X, double *V) {
    if (L < 2 || H < 1 || n_samples < L) return OR_EINVAL;
    const int T = 1 + (n_samples - L) / H, F = L / 2 + 1;
    for (int t = 0; t < T; ++t)
        for (int k = 0; k < F; ++k) {
            double re = 0.0, im = 0.0;
            for (int n = 0; n < L; ++n) {
                const double v = hann(n, L) * (double)x[(size_t)t * H + n];
                const double ang = -2.0 * PI * (double)(((long long)k * n) % L) / (double)L;
                re += v * cos(ang);
                im += v * sin(ang);
            }
            double *o = X + ((size_t)t * F + k) * 2;
            o[0] = re;
            o[1] = im;
            if (V) V[(size_t)t * F + k] = gain * sqrt(re * re + im * im);
        }
    return OR_OK;
}

/* X [T][F][2] mixture STFT, M [T][F] magnitudes -> y [n_samples] (one source) */
int or_istft(const double *X, const double *M, int T, int L, int H, double *y, int n_samples) {
    if (L < 2 || H < 1 || T < 1) return OR_EINVAL;
    const int F = L / 2 + 1;
    double *num = (double *)calloc((size_t)n_samples, sizeof(double));
    double *den = (double *)calloc((size_t)n_samples, sizeof(double));
    double *Yre = (double *)malloc(sizeof(double) * L), *Yim = (double *)malloc(sizeof(double) * L);
    for (int t = 0; t < T; ++t) {
        for (int k = 0; k < F; ++k) {
            const double *xc = X + ((size_t)t * F + k) * 2;
            const double mag = sqrt(xc[0] * xc[0] + xc[1] * xc[1]);
            const double m = M[(size_t)t * F + k];
            Yre[k] = mag > 0.0 ? m * xc[0] / mag : 0.0;
            Yim[k] = mag > 0.0 ? m * xc[1] / mag : 0.0;
        }
        for (int k = F; k < L; ++k) {   /* Hermitian symmetry of a real frame */
            Yre[k] = Yre[L - k];
            Yim[k] = -Yim[L - k];
        }
        for (int n = 0; n < L; ++n) {
            double acc = 0.0;
            for (int k = 0; k < L; ++k) {
                const double ang = 2.0 * PI * (double)(((long long)k * n) % L) / (double)L;
                acc += Yre[k] * cos(ang) - Yim[k] * sin(ang);
            }
            const long long s = (long long)t * H + n;
            if (s < n_samples) {
                const double w = hann(n, L);
                num[s] += w * acc / (double)L;
                den[s] += w * w;
            }
        }
    }
    for (int s = 0; s < n_samples; ++s) y[s] = den[s] > 0.0 ? num[s] / den[s] : 0.0;
    free(num); free(den); free(Yre); free(Yim);
    return OR_OK;
}
