// gemm_tc.cu -- the (a) reconstruction and (b) back-projection contractions on the 5th-generation tensor
// cores (tcgen05, sm_100a) with 3xTF32 splitting, so the products keep FP32 accuracy (BASELINE north_star:
// "SIMT FFMA tiles or 3xTF32 split tcgen05 with ... dictionary tiles in shared memory").
//
// C[M x N] = A[M x K] * B[N x K]^T:
//   (a) recon:    A = theta [frames][Kt_pad],  B = beta  (N = bins,     K = elements) -> V_hat   (Eq. 7)
//   (b) backproj: A = R     [frames][F_pad],   B = betaT (N = elements, K = bins)     -> R beta  (Eq. 6)
// Every FP32 operand x is split into x_hi = rn_tf32(x) and x_lo = rn_tf32(x - x_hi); the MMAs accumulate
// a_lo*b_hi + a_hi*b_lo + a_hi*b_hi (the dropped a_lo*b_lo is ~2^-22 relative; every term is non-negative,
// so there is no cancellation).  The dictionary (B) is static: it is split and re-tiled once, at
// set_model, into the exact shared-memory image of a pipeline stage, so each stage of B is ONE
// cp.async.bulk; the per-sweep operand A is split on the fly by converter warps.
//
// Accuracy of the accumulation (DESIGN "3xTF32 on tcgen05"): the tensor core's FP32 accumulator loses
// about half an ulp per update (measured: the error grows linearly with K).  The MMAs therefore
// accumulate only CHUNK_KB k-blocks (64 k-elements, 24 updates) into a TMEM slot; the epilogue warps
// drain each slot into FP32 registers with round-to-nearest adds while the MMAs fill the other slot.
// The error is then independent of K (Kt = 800 ... 8000), and the register accumulator doubles as the
// output double-buffer: the MMAs of tile i+1 run while the epilogue of tile i computes.
//
// One persistent CTA per SM, warp-specialised (22 warps):
//   warps 0-7   converters, two groups of 4 alternating pipeline stages: FP32 A rows (prefetched one
//               group-stage ahead in registers) -> hi/lo split -> shared memory in the canonical K-major
//               no-swizzle UMMA layout (8-row x 16-byte core matrices);
//   warp  8     TMEM allocator + single-thread tcgen05.mma issuer (M=128, N=BN, K=8 per instruction);
//   warp  9     B producer: one cp.async.bulk per stage (mbarrier complete_tx);
//   warps 10-21 epilogue: three warps per TMEM lane quarter, each owning every third 32-column chunk;
//               thread = output row; 128-bit vector loads/stores of its row.
// Epilogues: RATIO (R = V / V_hat, FP64 row partials of sum V log V_hat, zero-support flag, optional
// V_hat), STORE (V_hat), SEPARATE (v_t/alpha_0 scaled V_src^(s)), BACKPROJ (n = theta .* C).
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "nfhmm_internal.cuh"

namespace nfk {

namespace {

constexpr int TC_BM = 128;
constexpr int TC_KB = 16;                  // k-elements per pipeline stage (2 MMAs of K=8 per split product)
constexpr int CHUNK_KB = 4;                // k-blocks accumulated in TMEM before the epilogue drains the slot
// Warp roles: warps 0-3 converters, 4-15 epilogue, 16 MMA issuer + TMEM allocator, 17 B producer
constexpr int CONV_WARPS = 4;
constexpr int W_EPI0 = 4;
constexpr int EPI_PER_Q = 3;               // epilogue warps per TMEM lane quarter
constexpr int EPI_WARPS = 4 * EPI_PER_Q;   // 12
constexpr int W_MMA = 16;
constexpr int W_BLOAD = 17;
constexpr int TC_THREADS = 18 * 32;        // 576 -> up to 112 registers per thread
constexpr int TC_SLOT_COLS = 256;          // TMEM columns per accumulation slot (2 slots)
constexpr int TC_MAX_BN = 192;             // 6 x 32-column chunks = 2 per epilogue warp (64 FP32 registers)
constexpr int EPI_CH = 2;                  // chunks per epilogue warp
constexpr int RAW_DEPTH = 4;               // A stages in flight (cp.async) ahead of the converters
constexpr int RAW_SLOTS = RAW_DEPTH + 1;
constexpr int RAW_ROW = 20;                // floats per staged A row (16 + 4 pad: conflict-free 128-bit reads)
constexpr int RAW_OFF = 4096;              // [0,1024) barriers, [1024,4096) row-partial exchange
constexpr int RING_OFF = RAW_OFF + RAW_SLOTS * TC_BM * RAW_ROW * 4;   // then the hi/lo operand ring

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
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
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
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

__host__ __device__ __forceinline__ float tf32_rn_bits(float x) {
    uint32_t u;
    memcpy(&u, &x, 4);
    u = (u + 0x1000u) & 0xFFFFE000u;   // round to nearest (ties away) at 10 mantissa bits
    float y;
    memcpy(&y, &u, 4);
    return y;
}
__device__ __forceinline__ float tf32_rn(float x) {
    return __uint_as_float((__float_as_uint(x) + 0x1000u) & 0xFFFFE000u);
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
    int n_tiles;            // column tiles of C
    int bn;                 // tile width (multiple of 16, <= TC_MAX_BN)
    int k_begin, k_end;     // contraction window (global element index)
    int stages;
    const float *A;
    int lda;
    const float *Bsplit;    // pre-split, pre-tiled B: chunk (nt, kb) = [hi BN x 16][lo BN x 16] UMMA images
    int nkb_total;          // k-blocks per column tile in Bsplit
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
    int dbg;                // performance experiments only (NFHMM_TC_DEBUG): 1 no A loads, 2 no MMAs, 4 no epilogue I/O
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
    unsigned char *ring = smem_raw + RING_OFF;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int n_mtiles = (p.M + TC_BM - 1) / TC_BM;
    const int n_total = n_mtiles * p.n_tiles;
    const int kstart = p.k_begin & ~(TC_KB - 1);          // k-blocks on the global 16-element grid of Bsplit
    const int kb0 = kstart / TC_KB;
    const int n_kb = (p.k_end - kstart + TC_KB - 1) / TC_KB;
    const int n_chunks = (n_kb + CHUNK_KB - 1) / CHUNK_KB;

    if (threadIdx.x == 0) {
        for (int i = 0; i < p.stages; ++i) {
            mbar_init(&S.full[i], 128 + 1);   // the converters + the B producer's expect_tx arrive
            mbar_init(&S.empty[i], 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&S.pfull[i], 1);
            mbar_init(&S.pempty[i], EPI_WARPS * 32);
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    if (warp == W_MMA) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(smem_u32(&S.tmem_base)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = S.tmem_base;

    if (warp < CONV_WARPS) {
        // ------------------------------------------------------------ converters (A operand)
        // Thread t owns row t of every A tile: it copies the row's 16-float slab of stage it + RAW_DEPTH
        // into a private staging slot with cp.async (no registers held, RAW_DEPTH stages in flight),
        // then splits stage it from its slot into the hi/lo UMMA images.
        const int t = threadIdx.x;
        float *raw = reinterpret_cast<float *>(smem_raw + RAW_OFF);
        int tile = blockIdx.x, kb = 0, tile2 = blockIdx.x, kb2 = 0;
        auto advance = [&](int &tl, int &k_b) {
            if (++k_b == n_kb) {
                k_b = 0;
                tl += gridDim.x;
            }
        };
        auto issue = [&](int tl, int k_b, int slot) {
            if (tl < n_total && !(p.dbg & 1)) {
                const int mt = tl / p.n_tiles;
                const int k0 = kstart + k_b * TC_KB;
                const float *arow = p.A + (size_t)min(mt * TC_BM + t, p.M - 1) * p.lda;
                const uint32_t dst = smem_u32(raw + ((size_t)slot * TC_BM + t) * RAW_ROW);
#pragma unroll
                for (int c4 = 0; c4 < TC_KB / 4; ++c4) {
                    const int k = k0 + 4 * c4;
                    const bool in = k < p.k_end && k + 3 >= p.k_begin;   // whole float4 inside the row
                    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst + 16 * c4),
                                 "l"(arow + (in ? k : 0)), "r"(in ? 16 : 0));
                }
            }
            asm volatile("cp.async.commit_group;\n" ::: "memory");
        };
        for (int d = 0; d < RAW_DEPTH; ++d) {
            issue(tile2, kb2, d);
            advance(tile2, kb2);
        }
        uint32_t it = 0;
        while (tile < n_total) {
            asm volatile("cp.async.wait_group %0;\n" ::"n"(RAW_DEPTH - 1) : "memory");
            const float *src = raw + ((size_t)(it % RAW_SLOTS) * TC_BM + t) * RAW_ROW;
            float4 ca[TC_KB / 4];
#pragma unroll
            for (int c4 = 0; c4 < TC_KB / 4; ++c4) {
                ca[c4] = (p.dbg & 1) ? make_float4(1.f, 1.f, 1.f, 1.f) : *reinterpret_cast<const float4 *>(src + 4 * c4);
                const int k = kstart + kb * TC_KB + 4 * c4;
                if (k < p.k_begin || k + 4 > p.k_end) {   // window edges inside a float4
                    if (k + 0 < p.k_begin || k + 0 >= p.k_end) ca[c4].x = 0.f;
                    if (k + 1 < p.k_begin || k + 1 >= p.k_end) ca[c4].y = 0.f;
                    if (k + 2 < p.k_begin || k + 2 >= p.k_end) ca[c4].z = 0.f;
                    if (k + 3 < p.k_begin || k + 3 >= p.k_end) ca[c4].w = 0.f;
                }
            }
            issue(tile2, kb2, (it + RAW_DEPTH) % RAW_SLOTS);
            advance(tile2, kb2);
            const uint32_t st = it % p.stages, ph = (it / p.stages) & 1;
            mbar_wait(&S.empty[st], ph ^ 1);
            unsigned char *sa_hi = ring + (size_t)st * stage_bytes;
            unsigned char *sa_lo = sa_hi + a_bytes;
#pragma unroll
            for (int c4 = 0; c4 < TC_KB / 4; ++c4)
                if (!(p.dbg & 8)) split_store(sa_hi, sa_lo, (uint32_t)c4 * (TC_BM * 16) + (uint32_t)t * 16, ca[c4]);
            if (!(p.dbg & 16)) fence_proxy_async_smem();
            mbar_arrive(&S.full[st]);
            ++it;
            advance(tile, kb);
        }
        asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    } else if (warp == W_BLOAD) {
        // ------------------------------------------------------------ B producer (static dictionary)
        if (lane == 0) {
            uint32_t it = 0;
            for (int tile = blockIdx.x; tile < n_total; tile += gridDim.x) {
                const int nt = tile % p.n_tiles;
                const float *bt = p.Bsplit + (size_t)nt * p.nkb_total * (2 * (size_t)BN * TC_KB);
                for (int kb = 0; kb < n_kb; ++kb, ++it) {
                    const uint32_t st = it % p.stages, ph = (it / p.stages) & 1;
                    mbar_wait(&S.empty[st], ph ^ 1);
                    unsigned char *sb = ring + (size_t)st * stage_bytes + 2 * a_bytes;
                    if (p.dbg & 32) { mbar_arrive(&S.full[st]); continue; }
                    mbar_arrive_expect_tx(&S.full[st], 2 * b_bytes);
                    bulk_g2s(sb, bt + (size_t)(kb0 + kb) * (2 * (size_t)BN * TC_KB), 2 * b_bytes, &S.full[st]);
                }
            }
        }
    } else if (warp == W_MMA) {
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
                            if (p.dbg & 2) continue;
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
    } else if (warp >= W_EPI0 && warp < W_EPI0 + EPI_WARPS) {
        // ------------------------------------------------------------ epilogue
        const int ew = warp - W_EPI0;             // 0..11
        const int q = warp & 3;                   // TMEM lane quarter this warp may access
        const int cg = ew >> 2;                   // owns 32-column chunks cg, cg + 3
        const uint32_t lane_base = (uint32_t)(32 * q) << 16;
        double *xch = reinterpret_cast<double *>(smem_raw + 1024);   // [3][128] row partials
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
            {   // warm L2 with this row's epilogue operand (V or theta) while the tile accumulates
                const int prow = m0 + 32 * q + lane;
                const float *pb = p.mode == TC_RATIO ? p.V : (p.mode == TC_BACKPROJ ? p.theta : nullptr);
                if (pb && prow < p.M && !(p.dbg & 4)) {
#pragma unroll
                    for (int j = 0; j < EPI_CH; ++j) {
                        const int col = n0 + 32 * (cg + EPI_PER_Q * j);
                        if (col < p.ldc && 32 * (cg + EPI_PER_Q * j) < BN) {
                            asm volatile("prefetch.global.L2 [%0];\n" ::"l"(pb + (size_t)prow * p.ldc + col));
                            asm volatile("prefetch.global.L2 [%0];\n" ::"l"(pb + (size_t)prow * p.ldc + min(col + 31, p.ldc - 1)));
                        }
                    }
                }
            }
            for (int c = 0; c < n_chunks; ++c, ++ch_it) {
                const uint32_t slot = ch_it & 1, sph = (ch_it >> 1) & 1;
                mbar_wait(&S.pfull[slot], sph);
                tc_fence_after();
#pragma unroll
                for (int j = 0; j < EPI_CH; ++j) {
                    const int c0 = 32 * (cg + EPI_PER_Q * j);
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
                const int c0 = 32 * (cg + EPI_PER_Q * j);
                const int colb = n0 + c0;
                if (c0 >= BN || !row_ok) continue;
                const int w = min(32, BN - c0);
                if (p.dbg & 4) {
                    part += (double)acc[j][0];
                } else if (p.mode == TC_RATIO || p.mode == TC_BACKPROJ) {
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
                // three warps share each row: combine their partials in a fixed order
                const int rl = 32 * q + lane;
                xch[cg * 128 + rl] = part;
                asm volatile("bar.sync 1, %0;\n" ::"r"(EPI_WARPS * 32) : "memory");
                if (cg == 0 && row_ok)
                    p.data_part[(size_t)row * p.n_tiles + nt] = (xch[rl] + xch[128 + rl]) + xch[256 + rl];
                asm volatile("bar.sync 1, %0;\n" ::"r"(EPI_WARPS * 32) : "memory");
            }
        }
        if (bad) atomicOr(p.flags, bad);
    }

    tc_fence_before();
    __syncthreads();
    if (warp == W_MMA) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem));
    }
}

int g_num_sms = 0;

size_t stage_bytes_for(int bn) { return 2 * (size_t)TC_BM * TC_KB * 4 + 2 * (size_t)bn * TC_KB * 4; }

int stages_for(int bn) {
    const size_t budget = 227 * 1024 - RING_OFF;
    int s = (int)(budget / stage_bytes_for(bn));
    return s > 8 ? 8 : s;
}

cudaError_t launch_tc(const TcParams &p, cudaStream_t st) {
    if (g_num_sms == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
    }
    if (p.bn < 16 || p.bn > TC_MAX_BN || p.bn % 16 || p.stages < 2) return cudaErrorInvalidValue;
    const size_t smem = RING_OFF + (size_t)p.stages * stage_bytes_for(p.bn);
    static bool attr = false;
    if (!attr) {
        cudaError_t e = cudaFuncSetAttribute(tc_gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
        if (e != cudaSuccess) return e;
        attr = true;
    }
    const int n_total = ((p.M + TC_BM - 1) / TC_BM) * p.n_tiles;
    const int grid = n_total < g_num_sms ? n_total : g_num_sms;
    static int dbg = -1;
    if (dbg < 0) {
        const char *e = getenv("NFHMM_TC_DEBUG");
        dbg = e ? atoi(e) : 0;
    }
    TcParams q = p;
    q.dbg = dbg;
    tc_gemm_kernel<<<grid, TC_THREADS, smem, st>>>(q);
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

size_t tc_presplit_floats(int64_t n_rows, int64_t k_len, int bn) {
    const int64_t nt = (n_rows + bn - 1) / bn, nkb = (k_len + TC_KB - 1) / TC_KB;
    return (size_t)nt * nkb * 2 * bn * TC_KB;
}

// B[n][k] = get(n, k) for n < n_rows, k < k_len (zero elsewhere) -> dst in the shared-memory image of
// each pipeline stage: chunk (nt, kb) = [hi: c4, r, 4][lo: c4, r, 4] with r < bn, c4 < 4.
void tc_presplit_host(const float *src, int64_t ld_src, bool transposed, int64_t n_rows, int64_t k_len, int bn,
                      float *dst) {
    const int64_t nt_n = (n_rows + bn - 1) / bn, nkb = (k_len + TC_KB - 1) / TC_KB;
    for (int64_t nt = 0; nt < nt_n; ++nt)
        for (int64_t kb = 0; kb < nkb; ++kb) {
            float *chunk = dst + ((size_t)nt * nkb + kb) * 2 * bn * TC_KB;
            for (int r = 0; r < bn; ++r)
                for (int kk = 0; kk < TC_KB; ++kk) {
                    const int64_t n = nt * bn + r, k = kb * TC_KB + kk;
                    float x = 0.f;
                    if (n < n_rows && k < k_len) x = transposed ? src[(size_t)k * ld_src + n] : src[(size_t)n * ld_src + k];
                    const float hi = tf32_rn_bits(x);
                    const float lo = tf32_rn_bits(x - hi);
                    const size_t off = (size_t)(kk / 4) * (bn * 4) + (size_t)r * 4 + (kk % 4);
                    chunk[off] = hi;
                    chunk[(size_t)bn * TC_KB + off] = lo;
                }
        }
}

cudaError_t launch_recon_tc(int bn, const ReconArgs &a, cudaStream_t st) {
    TcParams p{};
    p.mode = a.R ? TC_RATIO : (a.out_src ? TC_SEPARATE : TC_STORE);
    p.M = a.M;
    p.bn = bn;
    p.n_tiles = (a.F + bn - 1) / bn;
    p.k_begin = a.k_begin;
    p.k_end = a.k_end;
    p.stages = stages_for(bn);
    p.A = a.A;
    p.lda = a.lda;
    p.Bsplit = a.Bsplit;
    p.nkb_total = a.nkb_total;
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
    p.bn = bn;
    p.n_tiles = (n_valid + bn - 1) / bn;
    p.k_begin = 0;
    p.k_end = a.Kpad;
    p.stages = stages_for(bn);
    p.A = a.A;
    p.lda = a.lda;
    p.Bsplit = a.Bsplit;
    p.nkb_total = a.nkb_total;
    p.ldc = a.ldb;
    p.theta = a.theta;
    p.n_out = a.n_out;
    return launch_tc(p, st);
}

}  // namespace nfk
