// gemm_tc.cu -- the (a) reconstruction and (b) back-projection contractions on the 5th-generation tensor
// cores (tcgen05, sm_100a) with 3xTF32 splitting, so the products keep FP32 accuracy (BASELINE north_star:
// "SIMT FFMA tiles or 3xTF32 split tcgen05 with ... dictionary tiles in shared memory").
//
// C[M x N] = A[M x K] * B[N x K]^T with both operands K-major in global memory:
//   (a) recon:    A = theta [frames][Kt_pad], B = beta  [F_pad][Kt_pad]  -> V_hat          (Eq. 7)
//   (b) backproj: A = R     [frames][F_pad],  B = betaT [Kt_pad][F_pad]  -> sum_l R beta   (Eq. 6)
// Every FP32 operand x is split on the fly into x_hi = rn_tf32(x) and x_lo = rn_tf32(x - x_hi); the MMAs
// accumulate a_lo*b_hi + a_hi*b_lo + a_hi*b_hi (the dropped a_lo*b_lo is ~2^-22 relative; every term is
// non-negative, so there is no cancellation).
//
// Accuracy of the accumulation (DESIGN "3xTF32 on tcgen05"): the tensor core's FP32 accumulator loses
// about half an ulp per update (measured: the error grows linearly with K).  The MMAs therefore
// accumulate only CHUNK_KB k-blocks (64 k-elements, 24 updates) into a TMEM slot; the epilogue warps
// drain each slot into FP32 registers with round-to-nearest adds while the MMAs fill the other slot.
// The error is then independent of K (Kt = 800 ... 8000), and the register accumulator doubles as the
// output double-buffer: the MMAs of tile i+1 run while the epilogue of tile i computes.
//
// One persistent CTA per SM, warp-specialised (13 warps):
//   warps 0-3   converters: FP32 global loads (prefetched one stage ahead in registers) -> hi/lo split ->
//               shared memory in the canonical K-major no-swizzle UMMA layout (8-row x 16-byte core
//               matrices), multi-stage mbarrier ring;
//   warp  4     TMEM allocator + single-thread tcgen05.mma issuer (M=128, N=BN, K=8 per instruction);
//   warps 5-12  epilogue: two warps per TMEM lane quarter, each owning every other 32-column chunk;
//               thread = output row; 128-bit vector loads/stores of its row.
// Epilogues: RATIO (R = V / V_hat, FP64 row partials of sum V log V_hat, zero-support flag, optional
// V_hat), STORE (V_hat), SEPARATE (v_t/alpha_0 scaled V_src^(s)), BACKPROJ (n = theta .* C).
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "nfhmm_internal.cuh"

namespace nfk {

namespace {

constexpr int TC_BM = 128;
constexpr int TC_KB = 16;                  // k-elements per pipeline stage (2 MMAs of K=8 per split product)
constexpr int CHUNK_KB = 4;                // k-blocks accumulated in TMEM before the epilogue drains the slot
constexpr int TC_THREADS = 13 * 32;
constexpr int TC_SLOT_COLS = 256;          // TMEM columns per accumulation slot (2 slots)
constexpr int TC_MAX_BN = 192;             // 3 x 32-column chunks per epilogue warp (96 FP32 registers)
constexpr int EPI_CH = 3;                  // max chunks per epilogue warp

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@!P1 bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }

__device__ __forceinline__ void tc_commit(uint64_t *bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_u32(bar))
                 : "memory");
}

__device__ __forceinline__ void tc_mma_tf32(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                            uint32_t accumulate) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "setp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n"
        "}\n" ::"r"(d_tmem),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

// K-major, no-swizzle UMMA shared-memory descriptor.  Core matrix = 8 rows x 16 bytes (contiguous);
// LBO = byte distance between core matrices adjacent in K, SBO = between 8-row groups (M/N).
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
    d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
    d |= (uint64_t)1 << 46;   // descriptor version (sm_100)
    return d;                 // base offset 0, LBO mode 0, layout type 0 = SWIZZLE_NONE
}

// Instruction descriptor: D F32, A/B TF32, both K-major, M = 128, N = n.
__host__ __device__ constexpr uint32_t idesc_tf32(int n) {
    return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(TC_BM >> 4) << 24);
}

__device__ __forceinline__ float tf32_rn(float x) {
    uint32_t u = __float_as_uint(x);
    u = (u + 0x1000u) & 0xFFFFE000u;   // round to nearest (ties away) at 10 mantissa bits
    return __uint_as_float(u);
}

// add 32 (or 16) TMEM columns of this warp's 32 lanes into acc (thread = lane = row)
__device__ __forceinline__ void tmem_add32(uint32_t taddr, float (&acc)[32]) {
    uint32_t r[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
    for (int i = 0; i < 32; ++i) acc[i] += __uint_as_float(r[i]);
}
__device__ __forceinline__ void tmem_add16(uint32_t taddr, float (&acc)[32]) {
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
    for (int i = 0; i < 16; ++i) acc[i] += __uint_as_float(r[i]);
}

enum TcMode : int { TC_RATIO = 0, TC_STORE = 1, TC_SEPARATE = 2, TC_BACKPROJ = 3 };

struct TcParams {
    int mode;
    int M;                  // rows (frames)
    int n_valid;            // valid rows of B (columns of C)
    int n_tiles;            // ceil(n_valid / BN)
    int bn;                 // tile width (multiple of 16, <= TC_MAX_BN)
    int k_begin, k_end;     // contraction window (global element index)
    int stages;
    const float *A;
    int lda;
    const float *B;
    int ldb;
    // epilogue
    int ldc;                // row length of V / R (RATIO) or theta / n (BACKPROJ); a multiple of 8
    int F;                  // true bins (V_hat / V_src column bound)
    const float *V;
    float *R;
    float *Vhat;
    double *data_part;
    const float *theta;
    float *n_out;
    const float *row_scale;
    float *out_src;
    int T, S, s;
    unsigned *flags;
};

struct Smem {
    uint64_t full[8], empty[8], pfull[2], pempty[2];
    uint32_t tmem_base;
};

// One FP32 float4 of row `row` at column k, masked to the window [kb, ke) (zeros outside).
__device__ __forceinline__ float4 ld_masked(const float *row, int k, int kb, int ke) {
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    if (k < ke && k + 3 >= kb) {
        v = __ldg(reinterpret_cast<const float4 *>(row + k));
        if (k < kb || k + 4 > ke) {
            if (k + 0 < kb || k + 0 >= ke) v.x = 0.f;
            if (k + 1 < kb || k + 1 >= ke) v.y = 0.f;
            if (k + 2 < kb || k + 2 >= ke) v.z = 0.f;
            if (k + 3 < kb || k + 3 >= ke) v.w = 0.f;
        }
    }
    return v;
}

__device__ __forceinline__ void split_store(unsigned char *hi_base, unsigned char *lo_base, uint32_t off, float4 v) {
    float4 hi, lo;
    hi.x = tf32_rn(v.x); lo.x = tf32_rn(v.x - hi.x);
    hi.y = tf32_rn(v.y); lo.y = tf32_rn(v.y - hi.y);
    hi.z = tf32_rn(v.z); lo.z = tf32_rn(v.z - hi.z);
    hi.w = tf32_rn(v.w); lo.w = tf32_rn(v.w - hi.w);
    *reinterpret_cast<float4 *>(hi_base + off) = hi;
    *reinterpret_cast<float4 *>(lo_base + off) = lo;
}

__global__ void __launch_bounds__(TC_THREADS, 1) tc_gemm_kernel(TcParams p) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    Smem &S = *reinterpret_cast<Smem *>(smem_raw);
    const int BN = p.bn;
    const uint32_t a_bytes = TC_BM * TC_KB * 4;           // one of hi / lo
    const uint32_t b_bytes = (uint32_t)BN * TC_KB * 4;
    const uint32_t stage_bytes = 2 * a_bytes + 2 * b_bytes;
    unsigned char *ring = smem_raw + 2048;           // [0,1024): barriers; [1024,2048): row-partial exchange

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int n_mtiles = (p.M + TC_BM - 1) / TC_BM;
    const int n_total = n_mtiles * p.n_tiles;
    const int kstart = p.k_begin & ~3;
    const int n_kb = (p.k_end - kstart + TC_KB - 1) / TC_KB;
    const int n_chunks = (n_kb + CHUNK_KB - 1) / CHUNK_KB;

    if (threadIdx.x == 0) {
        for (int i = 0; i < p.stages; ++i) {
            mbar_init(&S.full[i], 128);
            mbar_init(&S.empty[i], 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&S.pfull[i], 1);
            mbar_init(&S.pempty[i], 256);
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    if (warp == 4) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(smem_u32(&S.tmem_base)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = S.tmem_base;

    if (warp < 4) {
        // ------------------------------------------------------------ converters
        const int t = threadIdx.x;   // 0..127: row t of the A tile; rows t, t+128 of the B tile
        float4 ra[TC_KB / 4], rb0[TC_KB / 4], rb1[TC_KB / 4];
        auto load = [&](int tile, int kb) {
            const int mt = tile / p.n_tiles, nt = tile - mt * p.n_tiles;
            const int k0 = kstart + kb * TC_KB;
            const float *arow = p.A + (size_t)min(mt * TC_BM + t, p.M - 1) * p.lda;
#pragma unroll
            for (int c4 = 0; c4 < TC_KB / 4; ++c4) ra[c4] = ld_masked(arow, k0 + 4 * c4, p.k_begin, p.k_end);
            const int n_a = nt * BN + t, n_b = nt * BN + t + 128;
            const float *b0 = p.B + (size_t)min(n_a, p.n_valid - 1) * p.ldb;
            const float *b1 = p.B + (size_t)min(n_b, p.n_valid - 1) * p.ldb;
#pragma unroll
            for (int c4 = 0; c4 < TC_KB / 4; ++c4) {
                rb0[c4] = (t < BN && n_a < p.n_valid) ? ld_masked(b0, k0 + 4 * c4, p.k_begin, p.k_end) : make_float4(0.f, 0.f, 0.f, 0.f);
                rb1[c4] = (t + 128 < BN && n_b < p.n_valid) ? ld_masked(b1, k0 + 4 * c4, p.k_begin, p.k_end) : make_float4(0.f, 0.f, 0.f, 0.f);
            }
        };
        int tile = blockIdx.x, kb = 0;
        if (tile < n_total) load(tile, kb);
        uint32_t it = 0;
        while (tile < n_total) {
            // keep this stage's data, prefetch the next one while waiting for a free slot
            float4 ca[TC_KB / 4], cb0[TC_KB / 4], cb1[TC_KB / 4];
#pragma unroll
            for (int c4 = 0; c4 < TC_KB / 4; ++c4) {
                ca[c4] = ra[c4];
                cb0[c4] = rb0[c4];
                cb1[c4] = rb1[c4];
            }
            int ntile = tile, nkb = kb + 1;
            if (nkb == n_kb) {
                nkb = 0;
                ntile += gridDim.x;
            }
            if (ntile < n_total) load(ntile, nkb);
            const uint32_t st = it % p.stages, ph = (it / p.stages) & 1;
            mbar_wait(&S.empty[st], ph ^ 1);
            unsigned char *sa_hi = ring + (size_t)st * stage_bytes;
            unsigned char *sa_lo = sa_hi + a_bytes;
            unsigned char *sb_hi = sa_lo + a_bytes;
            unsigned char *sb_lo = sb_hi + b_bytes;
#pragma unroll
            for (int c4 = 0; c4 < TC_KB / 4; ++c4) {
                split_store(sa_hi, sa_lo, (uint32_t)c4 * (TC_BM * 16) + (uint32_t)t * 16, ca[c4]);
                if (t < BN) split_store(sb_hi, sb_lo, (uint32_t)c4 * ((uint32_t)BN * 16) + (uint32_t)t * 16, cb0[c4]);
                if (t + 128 < BN)
                    split_store(sb_hi, sb_lo, (uint32_t)c4 * ((uint32_t)BN * 16) + (uint32_t)(t + 128) * 16, cb1[c4]);
            }
            fence_proxy_async_smem();
            mbar_arrive(&S.full[st]);
            ++it;
            tile = ntile;
            kb = nkb;
        }
    } else if (warp == 4) {
        // ------------------------------------------------------------ MMA issuer
        const uint32_t idesc = idesc_tf32(BN);
        uint32_t it = 0, ch_it = 0;
        for (int tile = blockIdx.x; tile < n_total; tile += gridDim.x) {
            for (int c = 0; c < n_chunks; ++c, ++ch_it) {
                const uint32_t slot = ch_it & 1, sph = (ch_it >> 1) & 1;
                mbar_wait(&S.pempty[slot], sph ^ 1);
                tc_fence_after();
                const uint32_t d = tmem + slot * TC_SLOT_COLS;
                const int kb_end = min(n_kb, (c + 1) * CHUNK_KB);
                for (int kb = c * CHUNK_KB; kb < kb_end; ++kb, ++it) {
                    const uint32_t st = it % p.stages, ph = (it / p.stages) & 1;
                    mbar_wait(&S.full[st], ph);
                    tc_fence_after();
                    if (lane == 0) {
                        const uint32_t a_hi = smem_u32(ring + (size_t)st * stage_bytes);
                        const uint32_t a_lo = a_hi + a_bytes;
                        const uint32_t b_hi = a_lo + a_bytes;
                        const uint32_t b_lo = b_hi + b_bytes;
#pragma unroll
                        for (int kk = 0; kk < TC_KB / 8; ++kk) {
                            // K = 8 per MMA = 2 core matrices along K = 2 * LBO bytes
                            const uint32_t ao = (uint32_t)kk * 2 * (TC_BM * 16), bo = (uint32_t)kk * 2 * ((uint32_t)BN * 16);
                            const uint64_t dah = umma_desc(a_hi + ao, TC_BM * 16, 128);
                            const uint64_t dal = umma_desc(a_lo + ao, TC_BM * 16, 128);
                            const uint64_t dbh = umma_desc(b_hi + bo, (uint32_t)BN * 16, 128);
                            const uint64_t dbl = umma_desc(b_lo + bo, (uint32_t)BN * 16, 128);
                            const uint32_t first = (kb == c * CHUNK_KB && kk == 0) ? 0u : 1u;
                            tc_mma_tf32(d, dal, dbh, idesc, first);   // small terms first
                            tc_mma_tf32(d, dah, dbl, idesc, 1u);
                            tc_mma_tf32(d, dah, dbh, idesc, 1u);
                        }
                        tc_commit(&S.empty[st]);
                    }
                    __syncwarp();
                }
                if (lane == 0) tc_commit(&S.pfull[slot]);
                __syncwarp();
            }
        }
    } else {
        // ------------------------------------------------------------ epilogue
        const int ew = warp - 5;                  // 0..7
        const int q = warp & 3;                   // TMEM lane quarter this warp may access
        const int half = ew >> 2;                 // owns 32-column chunks half, half+2, half+4
        const uint32_t lane_base = (uint32_t)(32 * q) << 16;
        uint32_t ch_it = 0;
        unsigned bad = 0;
        for (int tile = blockIdx.x; tile < n_total; tile += gridDim.x) {
            const int mt = tile / p.n_tiles, nt = tile - mt * p.n_tiles;
            const int m0 = mt * TC_BM, n0 = nt * BN;
            float acc[EPI_CH][32];
#pragma unroll
            for (int j = 0; j < EPI_CH; ++j)
#pragma unroll
                for (int i = 0; i < 32; ++i) acc[j][i] = 0.f;
            for (int c = 0; c < n_chunks; ++c, ++ch_it) {
                const uint32_t slot = ch_it & 1, sph = (ch_it >> 1) & 1;
                mbar_wait(&S.pfull[slot], sph);
                tc_fence_after();
#pragma unroll
                for (int j = 0; j < EPI_CH; ++j) {
                    const int c0 = 32 * (half + 2 * j);
                    const uint32_t ta = tmem + slot * TC_SLOT_COLS + lane_base + (uint32_t)c0;
                    if (c0 + 32 <= BN) tmem_add32(ta, acc[j]);
                    else if (c0 + 16 <= BN) tmem_add16(ta, acc[j]);
                }
                tc_fence_before();
                mbar_arrive(&S.pempty[slot]);
            }
            // the tile's full sum is in registers; the MMAs of the next tile are already running
            const int row = m0 + 32 * q + lane;
            const bool row_ok = row < p.M;
            double part = 0.0;
#pragma unroll
            for (int j = 0; j < EPI_CH; ++j) {
                const int c0 = 32 * (half + 2 * j);
                const int colb = n0 + c0;
                if (c0 >= BN || !row_ok) continue;
                const int w = min(32, BN - c0);
                if (p.mode == TC_RATIO || p.mode == TC_BACKPROJ) {
                    const float *src = p.mode == TC_RATIO ? p.V : p.theta;
                    float *dst = p.mode == TC_RATIO ? p.R : p.n_out;
#pragma unroll
                    for (int i4 = 0; i4 < 8; ++i4) {
                        const int col = colb + 4 * i4;
                        if (4 * i4 >= w || col >= p.ldc) continue;
                        const size_t o = (size_t)row * p.ldc + col;
                        const float4 x = *reinterpret_cast<const float4 *>(src + o);
                        const float xv[4] = {x.x, x.y, x.z, x.w};
                        float y[4];
#pragma unroll
                        for (int e = 0; e < 4; ++e) {
                            const float vh = acc[j][4 * i4 + e];
                            if (p.mode == TC_BACKPROJ) {
                                y[e] = xv[e] * vh;                       // n = theta .* (R beta)
                            } else {
                                y[e] = 0.f;                              // R = V / V_hat
                                if (xv[e] > 0.f) {
                                    if (vh > 0.f) {
                                        y[e] = xv[e] / vh;
                                        part += (double)xv[e] * (double)logf(vh);
                                    } else {
                                        bad |= FLAG_ZERO_SUPPORT;
                                    }
                                }
                                if (p.Vhat && col + e < p.F) p.Vhat[(size_t)row * p.F + col + e] = vh;
                            }
                        }
                        *reinterpret_cast<float4 *>(dst + o) = make_float4(y[0], y[1], y[2], y[3]);
                    }
                } else if (p.mode == TC_STORE) {
#pragma unroll
                    for (int i = 0; i < 32; ++i)
                        if (i < w && colb + i < p.F) p.Vhat[(size_t)row * p.F + colb + i] = acc[j][i];
                } else {   // TC_SEPARATE
                    const float sc = p.row_scale[row];
                    const int m = row / p.T, tt = row - m * p.T;
                    float *out = p.out_src + ((size_t)(m * p.S + p.s) * p.T + tt) * p.F;
#pragma unroll
                    for (int i = 0; i < 32; ++i)
                        if (i < w && colb + i < p.F) out[colb + i] = acc[j][i] * sc;
                }
            }
            if (p.mode == TC_RATIO) {
                // two warps share each row: combine their partials in a fixed order through shared memory
                double *xch = reinterpret_cast<double *>(smem_raw + 1024);   // [128] doubles
                const int rl = 32 * q + lane;
                if (half == 1) xch[rl] = part;
                asm volatile("bar.sync 1, 256;\n" ::: "memory");
                if (half == 0 && row_ok) p.data_part[(size_t)row * p.n_tiles + nt] = part + xch[rl];
                asm volatile("bar.sync 1, 256;\n" ::: "memory");
            }
        }
        if (bad) atomicOr(p.flags, bad);
    }

    tc_fence_before();
    __syncthreads();
    if (warp == 4) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem));
    }
}

int g_num_sms = 0;

int stages_for(int bn) {
    const size_t stage_bytes = 2 * (size_t)TC_BM * TC_KB * 4 + 2 * (size_t)bn * TC_KB * 4;
    const size_t budget = 227 * 1024 - 2048;
    int s = (int)(budget / stage_bytes);
    return s > 8 ? 8 : s;
}

cudaError_t launch_tc(const TcParams &p, cudaStream_t st) {
    if (g_num_sms == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
    }
    if (p.bn < 16 || p.bn > TC_MAX_BN || p.bn % 16) return cudaErrorInvalidValue;
    const size_t stage_bytes = 2 * (size_t)TC_BM * TC_KB * 4 + 2 * (size_t)p.bn * TC_KB * 4;
    const size_t smem = 2048 + (size_t)p.stages * stage_bytes;
    static bool attr = false;
    if (!attr) {
        cudaError_t e = cudaFuncSetAttribute(tc_gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
        if (e != cudaSuccess) return e;
        attr = true;
    }
    const int n_total = ((p.M + TC_BM - 1) / TC_BM) * p.n_tiles;
    const int grid = n_total < g_num_sms ? n_total : g_num_sms;
    tc_gemm_kernel<<<grid, TC_THREADS, smem, st>>>(p);
    return cudaGetLastError();
}

}  // namespace

int tc_pick_bn(int64_t n) {
    int best = 16;
    int64_t best_pad = INT64_MAX;
    // padded width plus a per-tile cost (each extra column tile re-reads the A rows from L2)
    for (int bn = 16; bn <= TC_MAX_BN; bn += 16) {
        const int64_t pad = (n + bn - 1) / bn * bn + 24 * ((n + bn - 1) / bn);
        if (pad < best_pad || (pad == best_pad && bn > best)) {
            best_pad = pad;
            best = bn;
        }
    }
    return best;
}

cudaError_t launch_recon_tc(int bn, const ReconArgs &a, cudaStream_t st) {
    TcParams p{};
    p.mode = a.R ? TC_RATIO : (a.out_src ? TC_SEPARATE : TC_STORE);
    p.M = a.M;
    p.n_valid = a.F;
    p.bn = bn;
    p.n_tiles = (a.F + bn - 1) / bn;
    p.k_begin = a.k_begin;
    p.k_end = a.k_end;
    p.stages = stages_for(bn);
    p.A = a.A;
    p.lda = a.lda;
    p.B = a.B;          // beta [F_pad][Kt_pad] (K-major rows of length ldb)
    p.ldb = a.ldb;
    p.ldc = a.ldv;
    p.F = a.F;
    p.V = a.V;
    p.R = a.R;
    p.Vhat = a.Vhat;
    p.data_part = a.data_part;
    p.row_scale = a.row_scale;
    p.out_src = a.out_src;
    p.T = a.T;
    p.S = a.S;
    p.s = a.s;
    p.flags = a.flags;
    return launch_tc(p, st);
}

cudaError_t launch_backproj_tc(int bn, int n_valid, const BackprojArgs &a, cudaStream_t st) {
    TcParams p{};
    p.mode = TC_BACKPROJ;
    p.M = a.M;
    p.n_valid = n_valid;
    p.bn = bn;
    p.n_tiles = (n_valid + bn - 1) / bn;
    p.k_begin = 0;
    p.k_end = a.Kpad;
    p.stages = stages_for(bn);
    p.A = a.A;
    p.lda = a.lda;
    p.B = a.B;          // betaT [Kt_pad][F_pad]
    p.ldb = a.Kpad;
    p.ldc = a.ldb;
    p.theta = a.theta;
    p.n_out = a.n_out;
    return launch_tc(p, st);
}

}  // namespace nfk
