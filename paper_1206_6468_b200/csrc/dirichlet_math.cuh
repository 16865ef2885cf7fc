// dirichlet_math.cuh -- element arithmetic of the Dirichlet step (Eq. 6-8 per element, DESIGN R14),
// shared by the standalone Dirichlet kernel (dirichlet.cu) and the fused back-projection epilogue
// (gemm_tc.cu).  Product path only.
#pragma once
#include <stdint.h>

#include "digamma_u_poly.cuh"
#include "f32x2.cuh"

namespace nfk {

// ln of a pair, both >= 1 (normal): exponent ln 2 + lg2(mantissa) ln 2 (SFU), assembled packed
__device__ __forceinline__ uint64_t ln_sfu2(float x0, float x1) {
    const uint32_t b0 = __float_as_uint(x0), b1 = __float_as_uint(x1);
    float l0, l1;
    asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(l0) : "f"(__uint_as_float((b0 & 0x007FFFFFu) | 0x3F800000u)));
    asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(l1) : "f"(__uint_as_float((b1 & 0x007FFFFFu) | 0x3F800000u)));
    const uint64_t e = f2pack((float)((int)(b0 >> 23) - 127), (float)((int)(b1 >> 23) - 127));
    return f2fma(e, f2c(0.693147180559945309f), f2mul(f2pack(l0, l1), f2c(0.693147180559945309f)));
}
__device__ __forceinline__ float rcp_sfu(float x) {
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}
__device__ __forceinline__ float ex2_sfu(float x) {
    float r;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}
// Two elements at once (packed FFMA2 pipeline): alpha pair a -> psi, theta, and the running g~ sum
//   u = 1/a, t = 2u - 1, r = u/2 + u^2 G(t), psi = ln a - r, theta = a e^{-psi_0} exp(-r),
//   g~ = ln(a)/2 + ln(2 pi)/2 + 1/2 + u (H(t) - 1/2) + (u - u^2) G(t)
__device__ __forceinline__ void elem_pair(float a0, float a1, uint64_t e0_2, bool want_h, uint64_t &psi2,
                                          uint64_t &th2, uint64_t &g2t) {
    const uint64_t a2 = f2pack(a0, a1);
#ifdef NFHMM_EXP_NOMATH   // bandwidth experiment only: no element math
    psi2 = a2;
    th2 = f2mul(a2, e0_2);
    g2t = want_h ? a2 : 0ull;
    return;
#endif
    const uint64_t u2 = f2pack(rcp_sfu(a0), rcp_sfu(a1));
    const uint64_t lx2 = ln_sfu2(a0, a1);
    const uint64_t t2 = f2fma(u2, f2c(2.f), f2c(-1.f));
    const uint64_t G2 = dig_G2(t2);
    const uint64_t uu2 = f2mul(u2, u2);
    const uint64_t r2 = f2fma(uu2, G2, f2mul(u2, f2c(0.5f)));
    psi2 = f2sub(lx2, r2);
    float q0, q1;
    f2unpack(f2mul(r2, f2c(-1.44269504088896341f)), q0, q1);
    th2 = f2mul(f2mul(a2, e0_2), f2pack(ex2_sfu(q0), ex2_sfu(q1)));
    if (want_h) {
        const uint64_t H2 = lng_H2(t2);
        const uint64_t g2 = f2fma(f2c(0.5f), lx2, f2c(1.41893853320467274f));
        g2t = f2add(g2, f2fma(u2, f2sub(H2, f2c(0.5f)), f2mul(f2sub(u2, uu2), G2)));
    } else {
        g2t = 0ull;
    }
}


}  // namespace nfk
