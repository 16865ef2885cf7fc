// gemm_tc.cu -- the (a) reconstruction and (b) back-projection contractions on the 5th-generation tensor
// cores (tcgen05, sm_100a) with split products, so they keep FP32 accuracy (BASELINE north_star: "SIMT FFMA
// tiles or 3xTF32 split tcgen05 with TMA-staged dictionary tiles in shared memory").  The default is the
// H16 instantiation (3xFP16: kind::f16 at twice the TF32 rate, operands scaled by powers of two, DESIGN
// "3xFP16 products"); the description below is of the 3xTF32 kernel, which H16 follows with 32-element
// stages.  PAIR instantiations run as clusters of two CTAs that share every B image by TMA multicast.
//
// C[M x N] = A[M x K] * B[N x K]^T:
//   (a) recon:    A = theta [frames][Kt_pad],  B = beta  (N = bins,     K = elements) -> V_hat   (Eq. 7)
//   (b) backproj: A = R     [frames][F_pad],   B = betaT (N = elements, K = bins)     -> R beta  (Eq. 6)
// Every FP32 operand x is split into x_hi = rn_tf32(x) and x_lo = rn_tf32(x - x_hi); the MMAs accumulate
// a_lo*b_hi + a_hi*b_lo + a_hi*b_hi (the dropped a_lo*b_lo is ~2^-22 relative; every term is non-negative,
// so there is no cancellation).  The dictionary (B) is static: it is split and re-tiled once, at
// set_model, into the exact shared-memory image of a pipeline stage, so each stage of B is ONE
// cp.async.bulk.  The per-sweep operand A arrives by TMA (one 128-row x 16-float tensor copy per stage,
// 64-byte swizzle); converter warps split it and store hi / lo into TENSOR MEMORY, from where the MMAs
// read it (TS mode) -- A never goes through shared memory twice and never through L1.
//
// Accuracy of the accumulation (DESIGN "3xTF32 on tcgen05"): the tensor core's FP32 accumulator loses
// about half an ulp per update (measured: the error grows linearly with K).  The MMAs therefore
// accumulate only CHUNK_KB k-blocks (64 k-elements, 24 updates) into a TMEM slot; the epilogue warps
// drain each slot into FP32 registers with round-to-nearest adds while the MMAs fill the other slot.
// The error is then independent of K (Kt = 800 ... 8000), and the register accumulator doubles as the
// output double-buffer: the MMAs of tile i+1 run while the epilogue of tile i computes.
//
// One persistent CTA per SM, warp-specialised (18 warps):
//   warps 0-3   converters: thread t = A row t = TMEM lane t; A slab from the stage's smem copy (swizzled,
//               conflict-free 128-bit reads) -> tf32 hi / lo -> tcgen05.st into the stage's TMEM columns;
//   warps 4-15  epilogue: three warps per TMEM lane quarter, each owning every third 32-column chunk;
//               thread = output row.  Per 32 x 16 sub-tile the epilogue operand (V or theta) is fetched
//               by TMA into private smem (64-byte swizzle) when the tile starts, and the result (R or n)
//               leaves by a TMA store of the same sub-tile: global traffic is fully coalesced, and a
//               16-column tail chunk (BN = 176, 208, ...) never touches the next column tile;
//   warp  16    TMEM allocator + single-thread tcgen05.mma issuer (M=128, N=BN, K=8 per instruction);
//   warp  17    producer: per stage one cp.async.bulk (B image) + one TMA tensor copy (A), one mbarrier.
// Epilogues: RATIO (R = V / V_hat, FP64 row partials of sum V log V_hat, zero-support flag), BACKPROJ
// (n = theta .* C) through TMA; STORE (V_hat) and SEPARATE (v_t/alpha_0 scaled V_src^(s)), which run only
// for posteriors / separation (off the sweep), write directly from registers.
#include <cuda.h>
#include <cuda_fp16.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <vector>

#include "dirichlet_math.cuh"
#include "nfhmm_internal.cuh"

namespace nfk {

namespace {

constexpr int TC_BM = 128;
constexpr int TC_KB = 16;                  // k-elements per pipeline stage (2 MMAs of K=8 per split product)
constexpr int CHUNK_KB = 16;               // default k-blocks accumulated in TMEM before the epilogue drains the slot
// Warp roles: warps 0-3 converters, 4-15 epilogue, 16 MMA issuer + TMEM allocator, 17 producer
constexpr int CONV_WARPS = 4;
constexpr int W_EPI0 = 4;
constexpr int EPI_PER_Q = 3;               // epilogue warps per TMEM lane quarter
constexpr int EPI_WARPS = 4 * EPI_PER_Q;   // 12
constexpr int W_MMA = 16;
constexpr int W_PROD = 17;
constexpr int TC_THREADS = 18 * 32;        // 576
constexpr int TC_MAX_BN = 192;             // 6 x 32-column chunks = 2 per epilogue warp (64 FP32 registers)
constexpr int EPI_CH = 2;                  // chunks per epilogue warp
constexpr int A_STAGE_COLS = 2 * TC_KB;    // TMEM columns of one A stage: [hi 16][lo 16]
// A stage smem copy: 128 x 16 floats = 8 KB (TMA, 64-byte swizzle); H16: 128 x 32 floats (128-byte swizzle)
// FP16-split variant of the reconstruction (H16, DESIGN "3xFP16 reconstruction"): 32 k-elements per stage
// (2 MMAs of K=16 per split product), the A stage's smem copy is 128 x 32 floats (128-byte swizzle) and its
// TMEM image [hi 16 | lo 16] columns of packed half pairs -- the same 32 TMEM columns and the same B-image
// bytes per stage as the TF32 kernel
constexpr int TC_KB16 = 32;
__host__ __device__ constexpr int a_tile_bytes(bool h16) { return TC_BM * (h16 ? TC_KB16 : TC_KB) * 4; }
constexpr int EPI_SUB_BYTES = 32 * 16 * 4;        // 2 KB epilogue sub-tile: 32 rows x 16 columns (TMA, 64-byte swizzle)
constexpr int EPI_TILE_BYTES = 2 * EPI_SUB_BYTES; // per 32-column chunk
constexpr int MAX_STAGES = 16;            // ring depth cap (narrow tiles: more stages in flight, see stages_for)
constexpr int A_PREFETCH = 16;             // stages ahead at which the producer pulls A tiles into L2
constexpr int XCH_OFF = 1024;                                      // [3][128] FP64 row partials
constexpr int EPI_OFF = 4096;                                      // epilogue tiles [12][4 KB]
constexpr int RING_OFF = EPI_OFF + EPI_WARPS * EPI_TILE_BYTES;   // then the stage ring (DIRICHLET: the
                                                                   // epilogue warps' dv tiles come first)
constexpr int SMEM_MAX = 227 * 1024;

// TMEM map (512 columns): accumulation slots at [0, BN) and [BN, 2 BN); A stages from a_col0(BN).
__host__ __device__ constexpr int a_col0(int bn) { return (2 * bn + 31) & ~31; }
__host__ __device__ constexpr int tmem_a_stages(int bn) { return (512 - a_col0(bn)) / A_STAGE_COLS; }
// one ring stage = [A copy 8 KB][B hi | B lo], 1 KB aligned (the A swizzle pattern is address-based)
__host__ __device__ constexpr int stage_bytes_of(int bn, bool h16 = false) {
    return (a_tile_bytes(h16) + 2 * bn * TC_KB * 4 + 1023) & ~1023;
}

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
// Same, for roles off the MMA's critical path: the thread may be suspended until the phase completes
// (hardware wake-up) instead of spinning and stealing issue slots from the MMA / converter warps.
__device__ __forceinline__ void mbar_wait_sleep(uint64_t *bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n"
        "@!P1 bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity), "r"(1000000u)
        : "memory");
}
// ring position: stage index and phase parity, advanced without divisions
struct RingPos {
    uint32_t st = 0, ph = 0;
    __device__ __forceinline__ void next(uint32_t n) {
        if (++st == n) {
            st = 0;
            ph ^= 1;
        }
    }
};
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
// 2-D TMA tensor copies: c0 = element index along the contiguous dimension, c1 = row
__device__ __forceinline__ void tma_load_2d(void *dst, const CUtensorMap *map, int c0, int c1, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(
            smem_u32(dst)),
        "l"(map), "r"(c0), "r"(c1), "r"(smem_u32(bar))
        : "memory");
}
// L2 prefetch of a tensor tile (no shared memory, no completion tracking)
__device__ __forceinline__ void tma_prefetch_2d(const CUtensorMap *map, int c0, int c1) {
    asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global [%0, {%1, %2}];\n" ::"l"(map), "r"(c0), "r"(c1) : "memory");
}
__device__ __forceinline__ void tma_store_2d(const CUtensorMap *map, int c0, int c1, const void *src) {
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];\n" ::"l"(map), "r"(c0),
                 "r"(c1), "r"(smem_u32(src))
                 : "memory");
}
// the same copy into the shared memory of every CTA in ctaMask (same CTA-relative offsets), each CTA's
// mbarrier at bar's offset receiving the complete_tx
__device__ __forceinline__ void bulk_g2s_mc(void *dst, const void *src, uint32_t bytes, uint64_t *bar, uint16_t mask) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1], %2, [%3], %4;\n" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "h"(mask)
        : "memory");
}
__device__ __forceinline__ void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read_all() { asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }

__device__ __forceinline__ void tc_commit(uint64_t *bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_u32(bar))
                 : "memory");
}

// arrive on the mbarrier at bar's offset in every CTA of ctaMask when this thread's MMAs complete
__device__ __forceinline__ void tc_commit_mc(uint64_t *bar, uint16_t mask) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n" ::"r"(
                     smem_u32(bar)),
                 "h"(mask)
                 : "memory");
}

// A from tensor memory (TS mode): a_tmem = TMEM address of the 128-lane x 8-column K-major A block.
__device__ __forceinline__ void tc_mma_tf32_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t bdesc, uint32_t idesc,
                                               uint32_t accumulate) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "setp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n"
        "}\n" ::"r"(d_tmem),
        "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

// 16 consecutive TMEM columns of this thread's lane <- v[0..15]
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&v)[16]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};\n" ::"r"(taddr),
        "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
        "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
        : "memory");
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
// Same with A/B F16 (kind::f16, K = 16 per instruction)
__host__ __device__ constexpr uint32_t idesc_f16(int n) {
    return (1u << 4) | (0u << 7) | (0u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(TC_BM >> 4) << 24);
}
__device__ __forceinline__ void tc_mma_f16_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t bdesc, uint32_t idesc,
                                              uint32_t accumulate) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "setp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n"
        "}\n" ::"r"(d_tmem),
        "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(accumulate));
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

enum TcMode : int { TC_RATIO = 0, TC_STORE = 1, TC_SEPARATE = 2, TC_BACKPROJ = 3, TC_DIRICHLET = 4, TC_PARTIAL = 5 };

struct TcParams {
    int mode;
    int M;                  // rows (frames)
    int n_tiles;            // column tiles of C
    int bn;                 // tile width (multiple of 16, <= TC_MAX_BN)
    int k_begin, k_end;     // contraction window (global element index)
    int stages;
    int chunk_kb;           // k-blocks per TMEM accumulation slot (CHUNK_KB)
    int tma_epi;            // 1: epilogue operand in / result out through TMA (RATIO without V_hat, BACKPROJ)
    const float *Bsplit;    // pre-split, pre-tiled B: chunk (nt, kb) = [hi BN x 16][lo BN x 16] UMMA images
    int nkb_total;          // k-blocks per column tile in Bsplit
    // epilogue
    int ldc;                // row length of V / R (RATIO) or theta / n (BACKPROJ); a multiple of 8
    int F;                  // true bins (V_hat / V_src column bound)
    float *Vhat;
    double *data_part;
    const float *row_scale;
    float *out_src;
    int T, S, s;
    unsigned *flags;
    // DIRICHLET (back-projection with the fused Eq. 6-8 element step): see launch_backproj_dirichlet_tc
    int ring_off;           // byte offset of the stage ring
    int max_ctas;           // cap on the persistent grid (0 = one CTA per SM)
    int K, Kt, SN, nbc, ldf;
    const double *fconst;
    double *spsT, *sps2T, *hpartT;
    float *alpha_out;
    // PARTIAL (split-K for few row tiles): every work unit is (row tile, column tile, k-split) with ONE
    // accumulation chunk of chunk_kb k-blocks; its raw sums go to part[split][M][ldp] and tc_split_reduce
    // adds the splits in chunk order (the same FP32 additions as the single-CTA drain) and applies the
    // RATIO / BACKPROJ epilogue
    int splits;             // k-splits (1: no split)
    float *part;
    int ldp;
    const float *colscale;  // H16: per output column 2^-(15 + s_l) (the B row scale and the A scale undone)
    // H16 R scaling (DESIGN "3xFP16 products"): the reconstruction writes R' = c_l R (c_l = 2^30 colscale_l, a
    // power of two ~ max_k beta_l(k)) and the largest R' of every row (float bits, atomicMax) to rowmax; the
    // H16 back-projection scales row t of R' by 2^(14 - E_t) (E_t = exponent of rowmax[t]) and undoes it
    unsigned *rowmax;
    int pair;               // 1: cluster of two CTAs sharing every B image by multicast (see the kernel)
    int a_prefetch;         // stages ahead at which the producer pulls A tiles into L2 (A_PREFETCH)
    int dbg;                // performance experiments only (NFHMM_TC_DEBUG): 1 no A loads, 2 no MMAs, 4 no epilogue
                            // I/O, 8 no A TMEM stores, 32 no B loads, 64 no drains, 128 no converter work,
                            // 256 no L2 prefetch of the epilogue operand
};

// H16 back-projection: A scale 2^(14 - E) of row `row` (E = exponent of its largest R'; 1 for empty rows)
__device__ __forceinline__ float row_a_scale(const TcParams &p, int row) {
    if (row >= p.M) return 1.f;
    const unsigned u = __ldg(p.rowmax + row);
    if (u == 0u) return 1.f;
    int e = (int)((u >> 23) & 0xFF) - 127;
    e = min(max(e, -100), 100);
    return __uint_as_float((uint32_t)(127 + 14 - e) << 23);
}

struct Smem {
    uint64_t full[MAX_STAGES], empty[MAX_STAGES], loaded[MAX_STAGES], pfull[2], pempty[2], ebar[EPI_WARPS];
    uint32_t tmem_base;
};

// One element of the RATIO epilogue, branch-free: R = V / V_hat as V times the SFU reciprocal of `den`
// (V_hat, or V_hat / c_l for the H16 R'; rcp.approx: <= 1 ulp, so R is within 2 ulp), and V log2 V_hat (SFU)
// added to the sub-tile's sum; V > 0 where V_hat = 0 raises the zero-support flag (R = 0 there).  Used by the
// tile epilogue and by the split-K reduction alike, so split and unsplit results stay bitwise equal.
__device__ __forceinline__ float ratio_elem(float v, float vh, float den, float &lsum, unsigned &bad) {
    float rc;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(rc) : "f"(den));
    const bool pos = v > 0.f, sup = vh > 0.f;
    bad |= (pos && !sup) ? (unsigned)FLAG_ZERO_SUPPORT : 0u;
    const bool use = pos && sup;
    lsum = fmaf(use ? v : 0.f, __log2f(sup ? vh : 1.f), lsum);
    return use ? v * rc : 0.f;
}

// 16-byte chunk c of row r in a TMA tile with 64-B rows, 64-byte swizzle (bits [4,5] ^= bits [7,8])
__device__ __forceinline__ uint32_t swz64(int r, int c) { return (uint32_t)r * 64u + (uint32_t)((c ^ (r >> 1)) & 3) * 16u; }

// FUSED: the DIRICHLET epilogue only (a separate instantiation keeps registers down).  H16: FP16-split
// products (RATIO / STORE / PARTIAL of the reconstruction, A = theta~ in (0, 1])
template <bool FUSED, bool H16, bool PAIR>
__global__ void __launch_bounds__(TC_THREADS, 1)
    tc_gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmIn,
                   const __grid_constant__ CUtensorMap tmOut, const __grid_constant__ CUtensorMap tmDv,
                   TcParams p) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    Smem &S = *reinterpret_cast<Smem *>(smem_raw);
    const int BN = p.bn;
    constexpr int KB = H16 ? TC_KB16 : TC_KB;               // k-elements per stage
    constexpr uint32_t A_BYTES = (uint32_t)TC_BM * KB * 4;
    const uint32_t b_bytes = (uint32_t)BN * TC_KB * 4;     // one of hi / lo (BN x 16 tf32 or BN x 32 halves)
    const uint32_t stage_bytes = (uint32_t)stage_bytes_of(BN, H16);
    unsigned char *ring = smem_raw + p.ring_off;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int n_mtiles = (p.M + TC_BM - 1) / TC_BM;
    const int splits = p.splits > 1 ? p.splits : 1;
    // PAIR (cluster of two CTAs, p.pair): the pair walks units (row-tile pair, column tile) together, rank r
    // taking row tile 2 u_m + r; each CTA fetches half of every B image and multicasts it to both, so the
    // dictionary crosses L2 -> SM once per two row tiles.  A row tile past the end computes on TMA zero
    // fill and stores nothing (the tensor maps clip), so both CTAs see the same B sequence.
    constexpr bool pair = PAIR;   // a separate instantiation: the unpaired kernels keep their code
    uint32_t crank = 0;
    if constexpr (PAIR) asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(crank));
    // first unit and stride of this CTA's walk, read at each use (as special registers: a variable held
    // across the kernel measurably added spills to the 96-register roles)
#define TC_U0 (PAIR ? (int)(blockIdx.x >> 1) : (int)blockIdx.x)
#define TC_USTRIDE (PAIR ? (int)(gridDim.x >> 1) : (int)gridDim.x)
    const int n_total = pair ? ((n_mtiles + 1) >> 1) * p.n_tiles : n_mtiles * p.n_tiles * splits;
    const int kstart = p.k_begin & ~(KB - 1);             // k-blocks on the global KB-element grid of Bsplit
    const int kb0 = kstart / KB;
    const int n_kb = (p.k_end - kstart + KB - 1) / KB;
    const int chunk_kb = p.chunk_kb;
    // work unit -> (row tile, column tile) and its k-blocks [kb_lo, kb_hi) (all of them unless split)
    auto unit_of = [&](int tile, int &mt, int &nt, int &ks, int &kb_lo, int &kb_hi) {
        if (pair) {
            const int um = tile / p.n_tiles;
            nt = tile - um * p.n_tiles;
            mt = 2 * um + (int)crank;
            ks = 0;
            kb_lo = 0;
            kb_hi = n_kb;
            return;
        }
        ks = tile % splits;
        const int t2 = tile / splits;
        mt = t2 / p.n_tiles;
        nt = t2 - mt * p.n_tiles;
        kb_lo = splits > 1 ? ks * chunk_kb : 0;
        kb_hi = splits > 1 ? min(n_kb, kb_lo + chunk_kb) : n_kb;
    };

    if (threadIdx.x == 0) {
        for (int i = 0; i < p.stages; ++i) {
            mbar_init(&S.full[i], 128);      // the converters
            mbar_init(&S.empty[i], pair ? 2 : 1);   // tcgen05.commit of the stage's MMAs (PAIR: both CTAs')
            mbar_init(&S.loaded[i], 1);      // the producer's expect_tx (A + B bytes)
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&S.pfull[i], 1);
            mbar_init(&S.pempty[i], EPI_WARPS * 32);
        }
        for (int i = 0; i < EPI_WARPS; ++i) mbar_init(&S.ebar[i], 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    if (warp == W_MMA) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(smem_u32(&S.tmem_base)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    if (warp == W_PROD && lane == 0) {
        asm volatile("prefetch.tensormap [%0];\n" ::"l"(&tmA) : "memory");
        if (p.tma_epi) {
            asm volatile("prefetch.tensormap [%0];\n" ::"l"(&tmIn) : "memory");
            asm volatile("prefetch.tensormap [%0];\n" ::"l"(&tmOut) : "memory");
        }
        if (p.mode == TC_DIRICHLET) asm volatile("prefetch.tensormap [%0];\n" ::"l"(&tmDv) : "memory");
    }
    tc_fence_before();
    __syncthreads();
    if (pair) cluster_sync();   // the peer's multicast copies and commits target these barriers
    tc_fence_after();
    const uint32_t tmem = S.tmem_base;

    if (warp < CONV_WARPS) {
        // ------------------------------------------------------------ converters (A operand -> TMEM)
        const int t = threadIdx.x;
        const uint32_t a_base = tmem + ((uint32_t)(32 * warp) << 16) + (uint32_t)a_col0(BN);
        float asc = 32768.f;   // H16: this row's A scale (set at the first k-block of each tile)
        RingPos rp;
        const uint32_t nst = (uint32_t)p.stages;
        for (int tile = TC_U0; tile < n_total; tile += TC_USTRIDE) {
            int mt_, nt_, ks_, kb_lo, kb_hi;
            unit_of(tile, mt_, nt_, ks_, kb_lo, kb_hi);
            for (int kb = kb_lo; kb < kb_hi; ++kb, rp.next(nst)) {
                const uint32_t st = rp.st;
                mbar_wait(&S.loaded[st], rp.ph);
                tc_fence_after();
                if (p.dbg & 128) {
                    mbar_arrive(&S.full[st]);
                    continue;
                }
                const unsigned char *ab = ring + (size_t)st * stage_bytes;
                if constexpr (H16) {
                    // x' = 2^15 theta~ < 2^15 (recon) or 2^(14 - E_t) R'[t] (back-projection): hi = rn_f16(x'),
                    // lo = rn_f16(x' - hi) (the difference is exact in FP32), packed in pairs (element 2c in the
                    // low half of TMEM column c)
                    if (kb == kb_lo) asc = p.mode == TC_BACKPROJ ? row_a_scale(p, mt_ * TC_BM + t) : 32768.f;
                    float x[TC_KB16];
#pragma unroll
                    for (int c4 = 0; c4 < TC_KB16 / 4; ++c4) {
                        const float4 v = (p.dbg & 1) ? make_float4(1.f, 1.f, 1.f, 1.f)
                                                     : *reinterpret_cast<const float4 *>(ab + (uint32_t)t * 128u +
                                                                                         (uint32_t)((c4 ^ (t & 7)) << 4));
                        x[4 * c4 + 0] = v.x;
                        x[4 * c4 + 1] = v.y;
                        x[4 * c4 + 2] = v.z;
                        x[4 * c4 + 3] = v.w;
                    }
                    const int k0 = kstart + kb * TC_KB16;
                    if (k0 < p.k_begin || k0 + TC_KB16 > p.k_end) {
#pragma unroll
                        for (int i = 0; i < TC_KB16; ++i)
                            if (k0 + i < p.k_begin || k0 + i >= p.k_end) x[i] = 0.f;
                    }
                    uint32_t hi[16], lo[16];
                    const uint64_t asc2 = f2c(asc);
#pragma unroll
                    for (int i = 0; i < 16; ++i) {   // packed pairs: FMUL2, F2FP, 2 cvt, FADD2, F2FP per pair
                        const uint64_t a2 = f2mul(f2pack(x[2 * i], x[2 * i + 1]), asc2);
                        float a0, a1;
                        f2unpack(a2, a0, a1);
                        const __half2 h = __floats2half2_rn(a0, a1);
                        const float2 hf = __half22float2(h);
                        float l0, l1;
                        f2unpack(f2sub(a2, f2pack(hf.x, hf.y)), l0, l1);
                        const __half2 l = __floats2half2_rn(l0, l1);
                        hi[i] = *reinterpret_cast<const uint32_t *>(&h);
                        lo[i] = *reinterpret_cast<const uint32_t *>(&l);
                    }
                    if (!(p.dbg & 8)) {
                        tmem_st16(a_base + st * A_STAGE_COLS, hi);
                        tmem_st16(a_base + st * A_STAGE_COLS + 16, lo);
                        asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
                    }
                } else {
                float x[TC_KB];
#pragma unroll
                for (int c4 = 0; c4 < TC_KB / 4; ++c4) {
                    const float4 v = (p.dbg & 1) ? make_float4(1.f, 1.f, 1.f, 1.f)
                                                 : *reinterpret_cast<const float4 *>(ab + swz64(t, c4));
                    x[4 * c4 + 0] = v.x;
                    x[4 * c4 + 1] = v.y;
                    x[4 * c4 + 2] = v.z;
                    x[4 * c4 + 3] = v.w;
                }
                const int k0 = kstart + kb * TC_KB;
                if (k0 < p.k_begin || k0 + TC_KB > p.k_end) {   // window edges inside the slab
#pragma unroll
                    for (int i = 0; i < TC_KB; ++i)
                        if (k0 + i < p.k_begin || k0 + i >= p.k_end) x[i] = 0.f;
                }
                uint32_t hi[TC_KB], lo[TC_KB];
#pragma unroll
                for (int i = 0; i < TC_KB; ++i) {
                    const float h = tf32_rn(x[i]);
                    hi[i] = __float_as_uint(h);
                    lo[i] = __float_as_uint(tf32_rn(x[i] - h));
                }
                if (!(p.dbg & 8)) {
                    tmem_st16(a_base + st * A_STAGE_COLS, hi);
                    tmem_st16(a_base + st * A_STAGE_COLS + TC_KB, lo);
                    asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
                }
                }
                tc_fence_before();
                mbar_arrive(&S.full[st]);
            }
        }
    } else if (warp == W_PROD) {
        // ------------------------------------------------------------ producer: B image + A tile per stage
        // The A rows stream from HBM on first touch: they are pulled into L2 A_PREFETCH stages ahead, so
        // the ring's own loads (which bound the bytes in flight) see L2 latency only.
        if (lane == 0) {
            RingPos rp;
            const uint32_t nst = (uint32_t)p.stages;
            int pf_tile = TC_U0, pf_kb = 0, pf_mt = 0, pf_hi = 0;
            {
                int a_, b_, c_;
                unit_of(pf_tile, pf_mt, a_, b_, pf_kb, pf_hi);
                (void)c_;
            }
            auto pf_advance = [&]() {
                if (++pf_kb == pf_hi) {
                    pf_tile += TC_USTRIDE;
                    int a_, b_;
                    if (pf_tile < n_total) unit_of(pf_tile, pf_mt, a_, b_, pf_kb, pf_hi);
                }
            };
            auto pf_issue = [&]() {
                if (pf_tile < n_total && !(p.dbg & 1))
                    tma_prefetch_2d(&tmA, kstart + pf_kb * KB, pf_mt * TC_BM);
                if (pf_tile < n_total) pf_advance();
            };
            for (int i = 0; i < p.a_prefetch; ++i) pf_issue();
            for (int tile = TC_U0; tile < n_total; tile += TC_USTRIDE) {
                int mt, nt, ks_, kb_lo, kb_hi;
                unit_of(tile, mt, nt, ks_, kb_lo, kb_hi);
                const float *bt = p.Bsplit + (size_t)nt * p.nkb_total * (2 * (size_t)BN * TC_KB);   // same floats per block
                for (int kb = kb_lo; kb < kb_hi; ++kb, rp.next(nst)) {
                    const uint32_t st = rp.st;
                    mbar_wait_sleep(&S.empty[st], rp.ph ^ 1);
                    unsigned char *sa = ring + (size_t)st * stage_bytes;
                    const uint32_t bytes = ((p.dbg & 32) ? 0u : 2 * b_bytes) + ((p.dbg & 1) ? 0u : A_BYTES);
                    if (bytes == 0) {
                        mbar_arrive(&S.loaded[st]);
                        continue;
                    }
                    mbar_arrive_expect_tx(&S.loaded[st], bytes);
                    if (!(p.dbg & 32)) {
                        const float *bsrc = bt + (size_t)(kb0 + kb) * (2 * (size_t)BN * TC_KB);
                        if (pair)   // this CTA's half ([hi] or [lo]) into both CTAs' stage
                            bulk_g2s_mc(sa + A_BYTES + crank * b_bytes, bsrc + crank * (b_bytes / 4), b_bytes,
                                        &S.loaded[st], 0x3);
                        else
                            bulk_g2s(sa + A_BYTES, bsrc, 2 * b_bytes, &S.loaded[st]);
                    }
                    if (!(p.dbg & 1)) tma_load_2d(sa, &tmA, kstart + kb * KB, mt * TC_BM, &S.loaded[st]);
                    pf_issue();
                }
            }
        }
    } else if (warp == W_MMA) {
        // ------------------------------------------------------------ MMA issuer
        const uint32_t idesc = H16 ? idesc_f16(BN) : idesc_tf32(BN);
        RingPos rp;
        const uint32_t nst = (uint32_t)p.stages;
        uint32_t ch_it = 0;
        for (int tile = TC_U0; tile < n_total; tile += TC_USTRIDE) {
            int mt_, nt_, ks_, kb_lo, kb_hi;
            unit_of(tile, mt_, nt_, ks_, kb_lo, kb_hi);
            for (int cb = kb_lo; cb < kb_hi; cb += chunk_kb, ++ch_it) {
                const uint32_t slot = ch_it & 1, sph = (ch_it >> 1) & 1;
                mbar_wait(&S.pempty[slot], sph ^ 1);
                tc_fence_after();
                const uint32_t d = tmem + slot * (uint32_t)BN;
                const int kb_end = min(kb_hi, cb + chunk_kb);
                for (int kb = cb; kb < kb_end; ++kb, rp.next(nst)) {
                    const uint32_t st = rp.st;
                    mbar_wait(&S.loaded[st], rp.ph);   // B image landed (async proxy)
                    mbar_wait(&S.full[st], rp.ph);     // A split into TMEM
                    tc_fence_after();
                    if (lane == 0) {
                        const uint32_t a_hi = tmem + (uint32_t)a_col0(BN) + st * A_STAGE_COLS;
                        const uint32_t a_lo = a_hi + A_STAGE_COLS / 2;
                        const uint32_t b_hi = smem_u32(ring + (size_t)st * stage_bytes + A_BYTES);
                        const uint32_t b_lo = b_hi + b_bytes;
#pragma unroll
                        for (int kk = 0; kk < 2; ++kk) {
                            // K = 8 (tf32) / 16 (f16) per MMA: 8 TMEM columns of A; 2 core matrices (16 B rows)
                            // along K = 2 * LBO bytes of B
                            const uint32_t bo = (uint32_t)kk * 2 * ((uint32_t)BN * 16);
                            const uint64_t dbh = umma_desc(b_hi + bo, (uint32_t)BN * 16, 128);
                            const uint64_t dbl = umma_desc(b_lo + bo, (uint32_t)BN * 16, 128);
                            const uint32_t first = (kb == cb && kk == 0) ? 0u : 1u;
                            if (p.dbg & 2) continue;
                            if constexpr (H16) {
                                tc_mma_f16_ts(d, a_lo + 8 * kk, dbh, idesc, first);   // small terms first
                                tc_mma_f16_ts(d, a_hi + 8 * kk, dbl, idesc, 1u);
                                tc_mma_f16_ts(d, a_hi + 8 * kk, dbh, idesc, 1u);
                            } else {
                                tc_mma_tf32_ts(d, a_lo + 8 * kk, dbh, idesc, first);   // small terms first
                                tc_mma_tf32_ts(d, a_hi + 8 * kk, dbl, idesc, 1u);
                                tc_mma_tf32_ts(d, a_hi + 8 * kk, dbh, idesc, 1u);
                            }
                        }
                        if (pair) tc_commit_mc(&S.empty[st], 0x3);   // the peer's B half lives here too
                        else tc_commit(&S.empty[st]);
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
        double *xch = reinterpret_cast<double *>(smem_raw + XCH_OFF);   // [3][128] row partials
        unsigned char *etile = smem_raw + EPI_OFF + (size_t)ew * EPI_TILE_BYTES;
        const bool tma_epi = p.tma_epi && !(p.dbg & 4);
        uint32_t ch_it = 0, e_ph = 0;
        unsigned bad = 0;
        // operand tiles of chunk j: sub-tiles of 16 columns that lie inside the BN-wide column tile
        auto chunk_bytes = [&](int j) {
            uint32_t b = 0;
#pragma unroll
            for (int hh = 0; hh < 2; ++hh)
                if (32 * (cg + EPI_PER_Q * j) + 16 * (hh + 1) <= BN) b += EPI_SUB_BYTES;
            return b;
        };
        // lane 0: fetch chunk j's operand sub-tiles into the warp's buffer (after earlier stores read it)
        constexpr bool fused = FUSED;
        float *dvbuf = reinterpret_cast<float *>(smem_raw + RING_OFF + (size_t)ew * p.nbc * 128);   // [nbc][32]
        auto fetch = [&](int j, int n0, int r0) {
            const uint32_t b = chunk_bytes(j);
            if (!b) return;
            bulk_wait_read_all();
            mbar_arrive_expect_tx(&S.ebar[ew], b + (fused ? (uint32_t)p.nbc * 128u : 0u));
            if (fused) tma_load_2d(dvbuf, &tmDv, r0, (n0 + 32 * (cg + EPI_PER_Q * j)) / p.K, &S.ebar[ew]);
#pragma unroll
            for (int hh = 0; hh < 2; ++hh) {
                const int c0 = 32 * (cg + EPI_PER_Q * j) + 16 * hh;
                if (c0 + 16 <= BN) tma_load_2d(etile + hh * EPI_SUB_BYTES, &tmIn, n0 + c0, r0, &S.ebar[ew]);
            }
        };
        // DIRICHLET epilogue of one 32-column chunk (Eqs. 6-8 per element, dirichlet.cu for the
        // arithmetic): alpha = theta .* C + dv(block), then psi, the new theta (in place of the operand
        // tile, leaving by the TMA store) and g~.  The columns are K-element blocks (BN % K == 0, K <= 32);
        // the chunk's block ends are a warp-uniform bit mask, so the per-element bookkeeping is
        // branch-free: a block's psi sum is stored to spsT when its last element passes (to sps2T if the
        // block started in the previous chunk, which another warp owns), and a block still open at the
        // chunk's end is stored to spsT as its first part.
        auto fused_chunk = [&](int j, int n0, int r0, int row, bool row_ok, float e0f, float(&a32)[32],
                               uint64_t &hg2) {
            const int c0 = 32 * (cg + EPI_PER_Q * j), gc = n0 + c0, K = p.K;
            const int bq = gc / K, off = gc - bq * K, lim = p.Kt - gc;
            uint32_t endm = 0;   // bit i: column gc + i closes a block
            for (int i = K - 1 - off; i < 32; i += K) endm |= 1u << i;
            const uint32_t realm = lim >= 32 ? 0xFFFFFFFFu : (lim <= 0 ? 0u : (1u << lim) - 1u);
            const bool rok = row_ok;
            const int nb_last = p.SN - 1 - bq;   // relative index of the last real block
            double *const dst0 = off ? p.sps2T : p.spsT;   // the chunk's first block
            double *const dstn = p.spsT;
            const size_t ldf = (size_t)p.ldf;
            const uint64_t e0_2 = f2c(e0f);
            const bool want_h = p.hpartT != nullptr, want_a = p.alpha_out != nullptr && row_ok;
            int rel = 0;
            double sp = 0.0;
#pragma unroll
            for (int hh = 0; hh < 2; ++hh) {
                if (c0 + 16 * hh + 16 > BN) continue;
                unsigned char *tb = etile + hh * EPI_SUB_BYTES;
#pragma unroll
                for (int i4 = 0; i4 < 4; ++i4) {
                    float4 *px = reinterpret_cast<float4 *>(tb + swz64(lane, i4));
                    const float4 x = *px;
                    const float xv[4] = {x.x, x.y, x.z, x.w};
                    float y[4], av[4];
#pragma unroll
                    for (int e = 0; e < 4; e += 2) {
                        const int cc = 16 * hh + 4 * i4 + e;   // column inside the chunk
                        const int end0 = (endm >> cc) & 1, end1 = (endm >> (cc + 1)) & 1;
                        const int relB = rel + end0;
                        const float dvA = dvbuf[rel * 32 + lane];
                        const float dvB = dvbuf[min(relB, p.nbc - 1) * 32 + lane];
                        const float a0 = __fadd_rn(__fmul_rn(xv[e], a32[cc]), dvA);
                        const float a1 = __fadd_rn(__fmul_rn(xv[e + 1], a32[cc + 1]), dvB);
                        uint64_t ps2, th2, g2;
                        elem_pair(a0, a1, e0_2, want_h, ps2, th2, g2);
                        float p0, p1, t0, t1, g0, g1;
                        f2unpack(ps2, p0, p1);
                        f2unpack(th2, t0, t1);
                        f2unpack(g2, g0, g1);
                        const bool re0 = (realm >> cc) & 1, re1 = (realm >> (cc + 1)) & 1;
                        y[e] = re0 ? t0 : xv[e];   // padding columns (>= Kt) keep their operand
                        y[e + 1] = re1 ? t1 : xv[e + 1];
                        hg2 = f2add(hg2, f2pack(re0 ? g0 : 0.f, re1 ? g1 : 0.f));
                        sp += (double)p0;
                        if (end0 && rok && rel <= nb_last) (rel == 0 ? dst0 : dstn)[(size_t)(bq + rel) * ldf + row] = sp;
                        sp = end0 ? 0.0 : sp;
                        sp += (double)p1;
                        if (end1 && rok && relB <= nb_last)
                            (relB == 0 ? dst0 : dstn)[(size_t)(bq + relB) * ldf + row] = sp;
                        sp = end1 ? 0.0 : sp;
                        rel = relB + end1;
                        av[e] = a0;
                        av[e + 1] = a1;
                    }
                    *px = make_float4(y[0], y[1], y[2], y[3]);
                    if (want_a) {   // last sweep of a call: alpha for posteriors / separation
                        const int col = gc + 16 * hh + 4 * i4;
                        float *dst = p.alpha_out + (size_t)row * p.ldc + col;
                        if (col + 4 <= p.Kt) {
                            *reinterpret_cast<float4 *>(dst) = make_float4(av[0], av[1], av[2], av[3]);
                        } else {
#pragma unroll
                            for (int e = 0; e < 4; ++e)
                                if (col + e < p.Kt) dst[e] = av[e];
                        }
                    }
                }
                fence_proxy_async_smem();
                __syncwarp();
                if (lane == 0) {
                    tma_store_2d(&tmOut, gc + 16 * hh, r0, tb);
                    bulk_commit();
                }
            }
            // a block still open at the chunk's end continues in the next chunk: this is its first part
            const int w = c0 + 32 <= BN ? 32 : 16;
            if (!((endm >> (w - 1)) & 1) && rok && rel <= nb_last) (rel == 0 ? dst0 : dstn)[(size_t)(bq + rel) * ldf + row] = sp;
        };
        for (int tile = TC_U0; tile < n_total; tile += TC_USTRIDE) {
            int mt, nt, ks, kb_lo, kb_hi;
            unit_of(tile, mt, nt, ks, kb_lo, kb_hi);
            const int m0 = mt * TC_BM, n0 = nt * BN;
            const int r0 = m0 + 32 * q;            // first row of this warp's 32-row slice
            // chunk 0's operand lands while the tile accumulates; chunk 1's is fetched after chunk 0 left
            // (one buffer per warp), so it is pulled into L2 now: its fetch then waits on L2, not on HBM
            if (tma_epi && lane == 0) {
                fetch(0, n0, r0);
#pragma unroll
                for (int j = 1; j < EPI_CH && !(p.dbg & 256); ++j)
#pragma unroll
                    for (int hh = 0; hh < 2; ++hh) {
                        const int c0 = 32 * (cg + EPI_PER_Q * j) + 16 * hh;
                        if (c0 + 16 <= BN) tma_prefetch_2d(&tmIn, n0 + c0, r0);
                    }
            }
            __syncwarp();
            float e0f = 1.f;   // DIRICHLET: e^{-psi(alpha_0)} of this thread's frame
            if (fused && r0 + lane < p.M) e0f = (float)p.fconst[4 * (size_t)(r0 + lane) + 3];
            float acc[EPI_CH][32];
#pragma unroll
            for (int j = 0; j < EPI_CH; ++j)
#pragma unroll
                for (int i = 0; i < 32; ++i) acc[j][i] = 0.f;
            for (int cb = kb_lo; cb < kb_hi; cb += chunk_kb, ++ch_it) {
                const uint32_t slot = ch_it & 1, sph = (ch_it >> 1) & 1;
                mbar_wait_sleep(&S.pfull[slot], sph);
                tc_fence_after();
#pragma unroll
                for (int j = 0; j < EPI_CH; ++j) {
                    const int c0 = 32 * (cg + EPI_PER_Q * j);
                    const uint32_t ta = tmem + slot * (uint32_t)BN + lane_base + (uint32_t)c0;
                    if (p.dbg & 64) continue;
                    if (c0 + 32 <= BN) tmem_add32(ta, acc[j]);
                    else if (c0 + 16 <= BN) tmem_add16(ta, acc[j]);
                }
                tc_fence_before();
                mbar_arrive(&S.pempty[slot]);
            }
            // the tile's full sum is in registers; the MMAs of the next tile are already running
            if (H16 && p.mode != TC_RATIO && p.mode != TC_PARTIAL) {   // undo the power-of-two operand scales (exact)
                // (RATIO / PARTIAL keep the raw sums: R' = V / (2^-30 acc) and V_hat = colscale acc per element)
                const float rf = p.mode == TC_BACKPROJ ? 1.f / row_a_scale(p, r0 + lane) * 32768.f : 1.f;
#pragma unroll
                for (int j = 0; j < EPI_CH; ++j) {
                    const int c0 = 32 * (cg + EPI_PER_Q * j);
                    if (c0 >= BN) continue;
                    const float4 *cs = reinterpret_cast<const float4 *>(p.colscale + n0 + c0);
#pragma unroll
                    for (int i4 = 0; i4 < 8; ++i4) {
                        if (c0 + 4 * i4 >= BN) break;
                        const float4 c = __ldg(cs + i4);
                        acc[j][4 * i4] *= c.x * rf;
                        acc[j][4 * i4 + 1] *= c.y * rf;
                        acc[j][4 * i4 + 2] *= c.z * rf;
                        acc[j][4 * i4 + 3] *= c.w * rf;
                    }
                }
            }
            const int row = r0 + lane;
            const bool row_ok = row < p.M;
            double part = 0.0;
            float rmax = 0.f;      // RATIO: largest R' of this thread's columns (H16 back-projection scale)
            uint64_t hg2 = 0ull;   // DIRICHLET: packed running sum of g~ over this thread's columns
            if (tma_epi) {
#pragma unroll
                for (int j = 0; j < EPI_CH; ++j) {
                    if (!chunk_bytes(j)) continue;
                    if (j > 0) {
                        if (lane == 0) fetch(j, n0, r0);
                        __syncwarp();
                    }
                    mbar_wait_sleep(&S.ebar[ew], e_ph);
                    e_ph ^= 1;
                    if constexpr (FUSED) {
                        fused_chunk(j, n0, r0, row, row_ok, e0f, acc[j], hg2);
                    } else {
#pragma unroll
                    for (int hh = 0; hh < 2; ++hh) {
                        const int c0 = 32 * (cg + EPI_PER_Q * j) + 16 * hh;
                        if (c0 + 16 > BN) continue;
                        unsigned char *tb = etile + hh * EPI_SUB_BYTES;
                        float lsum = 0.f;   // sum over the sub-tile's 16 columns of V log2 V_hat
#pragma unroll
                        for (int i4 = 0; i4 < 4; ++i4) {
                            float4 *px = reinterpret_cast<float4 *>(tb + swz64(lane, i4));
                            const float4 x = *px;
                            const float xv[4] = {x.x, x.y, x.z, x.w};
                            float y[4];
                            float4 cs4 = make_float4(1.f, 1.f, 1.f, 1.f);
                            if (H16 && p.mode == TC_RATIO) cs4 = __ldg(reinterpret_cast<const float4 *>(p.colscale + n0 + c0) + i4);
                            const float csv[4] = {cs4.x, cs4.y, cs4.z, cs4.w};
#pragma unroll
                            for (int e = 0; e < 4; ++e) {
                                const float a_ = acc[j][16 * hh + 4 * i4 + e];
                                // H16: V_hat = colscale a_ (exact); R' = c_l R = V / (2^-30 a_)
                                const float vh = (H16 && p.mode == TC_RATIO) ? a_ * csv[e] : a_;
                                if (p.mode == TC_BACKPROJ) {
                                    y[e] = xv[e] * vh;                       // n = theta .* (R beta)
                                } else {
                                    y[e] = ratio_elem(xv[e], vh, (H16 && p.mode == TC_RATIO) ? a_ * 9.31322574615478515625e-10f : vh,
                                                      lsum, bad);
                                    rmax = fmaxf(rmax, y[e]);
                                }
                            }
                            *px = make_float4(y[0], y[1], y[2], y[3]);
                        }
                        // fixed point (2^-20 nats, an integer-valued double): the per-row sums across
                        // sub-tiles, warps and column tiles are then exact, so the data term of the bound
                        // does not depend on the tile width (sharding invariance of L)
                        part += rint(0.69314718055994530942 * 1048576.0 * (double)lsum);
                        fence_proxy_async_smem();
                        __syncwarp();
                        if (lane == 0) {
                            tma_store_2d(&tmOut, n0 + c0, r0, tb);
                            bulk_commit();
                        }
                    }
                    }
                }
                if (!row_ok) part = 0.0;
                if (p.rowmax && p.mode == TC_RATIO && row_ok && rmax > 0.f) atomicMax(p.rowmax + row, __float_as_uint(rmax));
            } else if (!FUSED && !H16 && !(p.dbg & 4) && (p.mode == TC_STORE || p.mode == TC_SEPARATE)) {
                // V_hat / V_hat^(s) rows are F floats (F odd in general: no TMA map), so each 32 x 32 chunk is
                // staged in the warp's epilogue tile (XOR swizzle: conflict-free both ways) and stored row by
                // row, 32 lanes on 32 consecutive columns of one row (coalesced), instead of thread = row
                float *tile = reinterpret_cast<float *>(etile);
                size_t myoff = 0;
                float sc = 1.f;
                if (row_ok) {
                    if (p.mode == TC_SEPARATE) {
                        const int m = row / p.T, tt = row - m * p.T;
                        myoff = ((size_t)(m * p.S + p.s) * p.T + tt) * p.F;
                        sc = p.row_scale[row];
                    } else {
                        myoff = (size_t)row * p.F;
                    }
                }
                float *const out = p.mode == TC_SEPARATE ? p.out_src : p.Vhat;
                const int nrows = min(32, p.M - r0);
#pragma unroll
                for (int j = 0; j < EPI_CH; ++j) {
                    const int c0 = 32 * (cg + EPI_PER_Q * j);
                    const int colb = n0 + c0;
                    if (c0 >= BN) continue;
                    const int w = min(32, BN - c0);
                    __syncwarp();
#pragma unroll
                    for (int i = 0; i < 32; ++i) tile[lane * 32 + (i ^ lane)] = acc[j][i] * sc;
                    __syncwarp();
                    const bool col_ok = lane < w && colb + lane < p.F;
                    for (int r = 0; r < nrows; ++r) {
                        const size_t off = __shfl_sync(0xffffffffu, (unsigned long long)myoff, r);
                        if (col_ok) out[off + colb + lane] = tile[r * 32 + (lane ^ r)];
                    }
                }
            } else if (!FUSED) {
#pragma unroll
                for (int j = 0; j < EPI_CH; ++j) {
                    const int c0 = 32 * (cg + EPI_PER_Q * j);
                    const int colb = n0 + c0;
                    if (c0 >= BN || !row_ok) continue;
                    const int w = min(32, BN - c0);
                    if (p.dbg & 4) {
                        part += (double)acc[j][0];
                    } else if (p.mode == TC_PARTIAL) {   // raw split sums, row-contiguous float4 stores
                        float *dst = p.part + ((size_t)ks * p.M + row) * p.ldp + colb;
#pragma unroll
                        for (int i = 0; i < 32; i += 4)
                            if (i < w) *reinterpret_cast<float4 *>(dst + i) = make_float4(acc[j][i], acc[j][i + 1], acc[j][i + 2], acc[j][i + 3]);
                    } else if (p.mode == TC_STORE) {
#pragma unroll
                        for (int i = 0; i < 32; ++i)
                            if (i < w && colb + i < p.F) p.Vhat[(size_t)row * p.F + colb + i] = acc[j][i];
                    } else if (p.mode == TC_SEPARATE) {
                        const float sc = p.row_scale[row];
                        const int m = row / p.T, tt = row - m * p.T;
                        float *out = p.out_src + ((size_t)(m * p.S + p.s) * p.T + tt) * p.F;
#pragma unroll
                        for (int i = 0; i < 32; ++i)
                            if (i < w && colb + i < p.F) out[colb + i] = acc[j][i] * sc;
                    }
                }
            }
            if (fused && p.hpartT) {
                float h0, h1;
                f2unpack(hg2, h0, h1);
                part = row_ok ? (double)h0 + (double)h1 : 0.0;
            }
            if ((p.mode == TC_RATIO && p.data_part) || (fused && p.hpartT)) {
                // three warps share each row: combine their partials in a fixed order
                const int rl = 32 * q + lane;
                xch[cg * 128 + rl] = part;
                asm volatile("bar.sync 1, %0;\n" ::"r"(EPI_WARPS * 32) : "memory");
                if (cg == 0 && row_ok) {
                    const double v = (xch[rl] + xch[128 + rl]) + xch[256 + rl];
                    if (fused) p.hpartT[(size_t)nt * p.ldf + row] = v;
                    else p.data_part[(size_t)row * p.n_tiles + nt] = v;
                }
                asm volatile("bar.sync 1, %0;\n" ::"r"(EPI_WARPS * 32) : "memory");
            }
        }
        if (lane == 0) bulk_wait_all();
        if (bad) atomicOr(p.flags, bad);
    }

    tc_fence_before();
    __syncthreads();
    if (pair) cluster_sync();   // no multicast copy or commit may still target this CTA's shared memory
    if (warp == W_MMA) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem));
    }
}

PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;

int stages_for(int bn, int ring_off = RING_OFF, bool h16 = false) {
    // as many stages as shared memory and the TMEM A columns allow: with few row tiles the per-stage load
    // latency bounds a CTA (round 2, config 1: ~0.9k cycles per k-block at 8 stages whatever the width)
    static int cap = -1;
    if (cap < 0) {
        const char *e = getenv("NFHMM_TC_STAGES");   // A/B experiments
        cap = (e && atoi(e) >= 2 && atoi(e) <= MAX_STAGES) ? atoi(e) : MAX_STAGES;
    }
    int s = (SMEM_MAX - ring_off) / stage_bytes_of(bn, h16);
    if (s > tmem_a_stages(bn)) s = tmem_a_stages(bn);
    return s > cap ? cap : s;
}

// 2-D FP32 tensor map over rows x cols (row pitch ld floats), box box_c x box_r
cudaError_t make_map(CUtensorMap *m, const float *base, int64_t cols, int64_t rows, int64_t ld, int box_c, int box_r,
                     CUtensorMapSwizzle swz) {
    if (!g_encode) {
        cudaDriverEntryPointQueryResult q;
        void *fn = nullptr;
        cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
        if (e != cudaSuccess || q != cudaDriverEntryPointSuccess || !fn) return cudaErrorNotSupported;
        g_encode = (PFN_cuTensorMapEncodeTiled_v12000)fn;
    }
    const cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
    const cuuint64_t strides[1] = {(cuuint64_t)ld * 4};
    const cuuint32_t box[2] = {(cuuint32_t)box_c, (cuuint32_t)box_r};
    const cuuint32_t es[2] = {1, 1};
    CUresult r = g_encode(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float *>(base), dims, strides, box, es,
                          CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

// A [M][lda] (cols = lda); epilogue in / out [M][ldc]
cudaError_t launch_tc(TcParams p, const float *A, int lda, const float *ein, float *eout, cudaStream_t st,
                      const float *dvT = nullptr, bool h16 = false) {
    const int g_num_sms = device_sms();
    if (p.bn < 16 || p.bn > TC_MAX_BN || p.bn % 16 || p.stages < 2) return cudaErrorInvalidValue;
    if (p.ring_off == 0) p.ring_off = RING_OFF;
    const size_t smem = (size_t)p.ring_off + (size_t)p.stages * stage_bytes_of(p.bn, h16);
    if (smem > SMEM_MAX) return cudaErrorInvalidValue;
    const bool fused = p.mode == TC_DIRICHLET;
    if (h16 && (fused || p.mode == TC_SEPARATE || !p.colscale)) return cudaErrorInvalidValue;
    if (h16 && p.mode == TC_BACKPROJ && !p.rowmax) return cudaErrorInvalidValue;
    const int n_mt = (p.M + TC_BM - 1) / TC_BM;
    const int sms = (p.max_ctas > 0 && p.max_ctas < g_num_sms) ? p.max_ctas : g_num_sms;
    // PAIR for the sweep's many-row-tile contractions (RATIO / BACKPROJ through TMA, unsplit, >= 2 row tiles
    // per CTA); NFHMM_TC_PAIR=0 turns it off (A/B experiments)
    const char *pev = getenv("NFHMM_TC_PAIR");   // read per launch (tests switch it within one process)
    const int pair_env = pev ? atoi(pev) : -1;
    // (measured at config 3: the back-projection, 17 k-blocks per tile, 88.7 -> 85.2 ms per step; the
    // reconstruction, 25 k-blocks, unchanged; config 4 (33 / 250 k-blocks per tile) slower with it)
    const int nkb_tile = (p.k_end - (p.k_begin & ~((h16 ? TC_KB16 : TC_KB) - 1)) + (h16 ? TC_KB16 : TC_KB) - 1) /
                         (h16 ? TC_KB16 : TC_KB);
    p.pair = (pair_env > 0 || (pair_env < 0 && nkb_tile <= 24)) && p.tma_epi && p.splits <= 1 && p.mode != TC_DIRICHLET &&
             n_mt >= 2 * sms ? 1 : 0;
    auto kern = fused ? tc_gemm_kernel<true, false, false>
                : h16 ? (p.pair ? tc_gemm_kernel<false, true, true> : tc_gemm_kernel<false, true, false>)
                      : (p.pair ? tc_gemm_kernel<false, false, true> : tc_gemm_kernel<false, false, false>);
    {
        cudaError_t e = ensure_dyn_smem((const void *)kern, SMEM_MAX);
        if (e != cudaSuccess) return e;
    }
    CUtensorMap mA, mIn, mOut, mDv;
    cudaError_t e = h16 ? make_map(&mA, A, lda, p.M, lda, TC_KB16, TC_BM, CU_TENSOR_MAP_SWIZZLE_128B)
                        : make_map(&mA, A, lda, p.M, lda, TC_KB, TC_BM, CU_TENSOR_MAP_SWIZZLE_64B);
    if (e != cudaSuccess) return e;
    mIn = mA;
    mOut = mA;
    mDv = mA;
    if (p.mode == TC_DIRICHLET) {   // dvT [SN][ldf]: box = 32 frames x nbc blocks, no swizzle
        e = make_map(&mDv, dvT, p.ldf, p.SN, p.ldf, 32, p.nbc, CU_TENSOR_MAP_SWIZZLE_NONE);
        if (e != cudaSuccess) return e;
    }
    if (p.tma_epi) {
        e = make_map(&mIn, ein, p.ldc, p.M, p.ldc, 16, 32, CU_TENSOR_MAP_SWIZZLE_64B);
        if (e == cudaSuccess) e = make_map(&mOut, eout, p.ldc, p.M, p.ldc, 16, 32, CU_TENSOR_MAP_SWIZZLE_64B);
        if (e != cudaSuccess) return e;
    }
    const int n_total = p.pair ? ((n_mt + 1) / 2) * p.n_tiles : n_mt * p.n_tiles * (p.splits > 1 ? p.splits : 1);
    int grid = p.pair ? std::min(2 * n_total, sms & ~1) : (n_total < sms ? n_total : sms);
    static int dbg = -1, chunk = CHUNK_KB;
    if (dbg < 0) {
        const char *ev = getenv("NFHMM_TC_DEBUG");
        dbg = ev ? atoi(ev) : 0;
        const char *ec = getenv("NFHMM_TC_CHUNK");   // accuracy / speed experiments only
        if (ec && atoi(ec) > 0) chunk = atoi(ec);
    }
    p.dbg = dbg;
    static int apf = -1;
    if (apf < 0) {
        const char *e = getenv("NFHMM_TC_PREFETCH");   // A/B experiments
        apf = (e && atoi(e) >= 0) ? atoi(e) : A_PREFETCH;
    }
    p.a_prefetch = apf;
    p.chunk_kb = h16 ? (chunk + 1) / 2 : chunk;   // the same 256 k-elements per accumulation slot
    if (p.pair) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3((unsigned)grid);
        cfg.blockDim = dim3(TC_THREADS);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = st;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = 2;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        return cudaLaunchKernelEx(&cfg, kern, mA, mIn, mOut, mDv, p);
    }
    kern<<<grid, TC_THREADS, smem, st>>>(mA, mIn, mOut, mDv, p);
    return cudaGetLastError();
}

// Split-K epilogue: C[row][c] = ((0 + part_0) + part_1) + ... (the chunk order of the single-CTA drain,
// so C is bitwise the unsplit kernel's), then the RATIO epilogue (R = V / C, 0 where V = 0, zero-support
// flag, the data term of the bound per 16-column sub-tile in the same fixed point) or BACKPROJ
// (n = theta .* C; supported, not used: see nfhmm_abi.cu).  One thread per (row, 16-column sub-tile).
__global__ void __launch_bounds__(256) tc_split_reduce_kernel(int mode, int splits, const float *__restrict__ part,
                                                              int ldp, int M, int ldc, const float *__restrict__ ein,
                                                              float *__restrict__ eout, double *data_part, int n_sub,
                                                              unsigned *flags, const float *__restrict__ colscale,
                                                              unsigned *rowmax) {
    const long long id = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    const int row = (int)(id / n_sub), sub = (int)(id - (long long)row * n_sub);
    if (row >= M) return;
    const int c0 = 16 * sub;
    float acc[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) acc[i] = 0.f;
    for (int s = 0; s < splits; ++s) {
        const float4 *src = reinterpret_cast<const float4 *>(part + ((size_t)s * M + row) * ldp + c0);
#pragma unroll
        for (int i4 = 0; i4 < 4; ++i4) {
            const float4 v = src[i4];
            acc[4 * i4] += v.x;
            acc[4 * i4 + 1] += v.y;
            acc[4 * i4 + 2] += v.z;
            acc[4 * i4 + 3] += v.w;
        }
    }
    const float *x = ein + (size_t)row * ldc + c0;
    float *y = eout + (size_t)row * ldc + c0;
    const int w = min(16, ldc - c0);   // ldc is a multiple of 8
    if (mode == TC_BACKPROJ) {
#pragma unroll
        for (int i4 = 0; i4 < 4; ++i4) {
            if (4 * i4 >= w) break;
            const float4 t = reinterpret_cast<const float4 *>(x)[i4];
            reinterpret_cast<float4 *>(y)[i4] =
                make_float4(t.x * acc[4 * i4], t.y * acc[4 * i4 + 1], t.z * acc[4 * i4 + 2], t.w * acc[4 * i4 + 3]);
        }
        return;
    }
    float lsum = 0.f, rmax = 0.f;
    unsigned bad = 0;
#pragma unroll
    for (int i4 = 0; i4 < 4; ++i4) {
        if (4 * i4 >= w) break;
        const float4 v4 = reinterpret_cast<const float4 *>(x)[i4];
        const float xv[4] = {v4.x, v4.y, v4.z, v4.w};
        const float4 cs4 = colscale ? __ldg(reinterpret_cast<const float4 *>(colscale + c0) + i4) : make_float4(1.f, 1.f, 1.f, 1.f);
        const float csv[4] = {cs4.x, cs4.y, cs4.z, cs4.w};
        float r[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            // H16 sums are raw: V_hat = colscale acc, R' = c_l R = V / (2^-30 acc) (as the tile epilogue)
            const float vh = colscale ? acc[4 * i4 + e] * csv[e] : acc[4 * i4 + e];
            r[e] = ratio_elem(xv[e], vh, colscale ? acc[4 * i4 + e] * 9.31322574615478515625e-10f : vh, lsum, bad);
            rmax = fmaxf(rmax, r[e]);
        }
        reinterpret_cast<float4 *>(y)[i4] = make_float4(r[0], r[1], r[2], r[3]);
    }
    if (rowmax && rmax > 0.f) atomicMax(rowmax + row, __float_as_uint(rmax));
    if (data_part) data_part[(size_t)row * n_sub + sub] = rint(0.69314718055994530942 * 1048576.0 * (double)lsum);
    if (bad) atomicOr(flags, bad);
}

cudaError_t launch_split(TcParams p, const float *A, int lda, const float *ein, float *eout, int ldc, double *data_part,
                         cudaStream_t st, bool h16 = false) {
    const int mode = p.mode;
    p.mode = TC_PARTIAL;
    p.tma_epi = 0;
    cudaError_t e = launch_tc(p, A, lda, nullptr, nullptr, st, nullptr, h16);
    if (e != cudaSuccess) return e;
    const int n_sub = (ldc + 15) / 16;
    const long long threads = (long long)p.M * n_sub;
    tc_split_reduce_kernel<<<(unsigned)((threads + 255) / 256), 256, 0, st>>>(mode, p.splits, p.part, p.ldp, p.M, ldc,
                                                                            ein, eout, data_part, n_sub, p.flags,
                                                                            h16 ? p.colscale : nullptr, p.rowmax);
    return cudaGetLastError();
}

}  // namespace

int tc_pick_bn(int64_t n, int mult, int64_t rows, int sms) {
    int best = 0;
    int64_t best_cost = INT64_MAX;
    const int64_t mt = (rows + TC_BM - 1) / TC_BM;
    // time ~ waves of the persistent grid x per-tile work, the latter ~ padded width plus a per-tile cost
    // (each column tile re-reads the A rows from L2; 24 columns' worth).  For large row counts this is the
    // padded width plus 24 per tile; for few row tiles (single mixtures: 8-16 row tiles) narrower tiles
    // put more of the 148 SMs to work.
    for (int bn = mult; bn <= TC_MAX_BN; bn += mult) {
        const int64_t nt = (n + bn - 1) / bn;
        const int64_t waves = (mt * nt + sms - 1) / sms;
        const int64_t cost = rows > 0 ? waves * (bn + 24) : nt * (bn + 24);
        if (cost < best_cost || (cost == best_cost && bn > best)) {
            best_cost = cost;
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
// each pipeline stage: chunk (nt, kb) = [hi: c4, r, 4][lo: c4, r, 4] with r < bn, c4 < 4.  The chunks of a
// column tile are laid out for k_pad >= k_len (the contraction length the kernel walks, nkb_total =
// ceil(k_pad / 16)), so tile nt starts at chunk nt * nkb_total.
void tc_presplit_host(const float *src, int64_t ld_src, bool transposed, int64_t n_rows, int64_t k_len, int bn,
                      float *dst, int64_t k_pad, const float *kscale) {
    if (k_pad < k_len) k_pad = k_len;
    const int64_t nt_n = (n_rows + bn - 1) / bn, nkb = (k_pad + TC_KB - 1) / TC_KB;
    for (int64_t nt = 0; nt < nt_n; ++nt)
        for (int64_t kb = 0; kb < nkb; ++kb) {
            float *chunk = dst + ((size_t)nt * nkb + kb) * 2 * bn * TC_KB;
            for (int r = 0; r < bn; ++r)
                for (int kk = 0; kk < TC_KB; ++kk) {
                    const int64_t n = nt * bn + r, k = kb * TC_KB + kk;
                    float x = 0.f;
                    if (n < n_rows && k < k_len) x = transposed ? src[(size_t)k * ld_src + n] : src[(size_t)n * ld_src + k];
                    if (kscale && n < n_rows && k < k_len) x *= kscale[k];   // power of two: exact
                    const float hi = tf32_rn_bits(x);
                    const float lo = tf32_rn_bits(x - hi);
                    const size_t off = (size_t)(kk / 4) * (bn * 4) + (size_t)r * 4 + (kk % 4);
                    chunk[off] = hi;
                    chunk[(size_t)bn * TC_KB + off] = lo;
                }
        }
}

size_t tc_presplit16_floats(int64_t n_rows, int64_t k_len, int bn) {
    const int64_t nt = (n_rows + bn - 1) / bn, nkb = (k_len + TC_KB16 - 1) / TC_KB16;
    return (size_t)nt * nkb * bn * TC_KB16;   // 2 x bn x 32 halves per chunk
}

// FP16 image of B[n][k] for the H16 reconstruction: row n scaled by 2^s_n so that its maximum lies in
// [2^14, 2^15), then hi = rn_f16(x'), lo = rn_f16(x' - hi); chunk (nt, kb) = [hi: c8, r, 8][lo: c8, r, 8]
// (c8 < 4: 8-element core-matrix rows of 16 bytes).  colscale[n] = 2^-(15 + s_n) undoes the B scale and
// the converters' 2^15 scale of A; it is written for nt_n * bn columns (1 past n_rows).
void tc_presplit16_host(const float *src, int64_t ld_src, bool transposed, int64_t n_rows, int64_t k_len, int bn,
                        float *dst, float *colscale, int64_t k_pad, const float *kscale) {
    if (k_pad < k_len) k_pad = k_len;
    const int64_t nt_n = (n_rows + bn - 1) / bn, nkb = (k_pad + TC_KB16 - 1) / TC_KB16;
    auto get = [&](int64_t n, int64_t k) {
        if (n >= n_rows || k >= k_len) return 0.f;
        const float x = transposed ? src[(size_t)k * ld_src + n] : src[(size_t)n * ld_src + k];
        return kscale ? x * kscale[k] : x;
    };
    std::vector<float> sc((size_t)nt_n * bn, 1.f);
    for (int64_t n = 0; n < nt_n * bn; ++n) {
        float mx = 0.f;
        for (int64_t k = 0; k < k_len && n < n_rows; ++k) mx = fmaxf(mx, get(n, k));
        int e = 0;
        if (mx > 0.f) {
            frexpf(mx, &e);   // mx = f 2^e, f in [0.5, 1): scaled max 2^(15-e) mx in [2^14, 2^15)
            e = 15 - e;
        }
        sc[n] = ldexpf(1.f, e);
        colscale[n] = ldexpf(1.f, -(e + 15));
    }
    __half *h = reinterpret_cast<__half *>(dst);
    for (int64_t nt = 0; nt < nt_n; ++nt)
        for (int64_t kb = 0; kb < nkb; ++kb) {
            __half *chunk = h + ((size_t)nt * nkb + kb) * 2 * bn * TC_KB16;
            for (int r = 0; r < bn; ++r)
                for (int kk = 0; kk < TC_KB16; ++kk) {
                    const int64_t n = nt * bn + r, k = kb * TC_KB16 + kk;
                    const float x = get(n, k) * sc[n];
                    const __half hi = __float2half_rn(x);
                    const __half lo = __float2half_rn(x - __half2float(hi));
                    const size_t off = (size_t)(kk / 8) * (bn * 8) + (size_t)r * 8 + (kk % 8);
                    chunk[off] = hi;
                    chunk[(size_t)bn * TC_KB16 + off] = lo;
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
    p.tma_epi = (p.mode == TC_RATIO && !a.Vhat) ? 1 : 0;
    p.Bsplit = a.Bsplit;
    p.nkb_total = a.nkb_total;
    p.ldc = a.ldv;
    p.F = a.F;
    p.Vhat = a.Vhat;
    p.data_part = a.data_part;
    p.row_scale = a.row_scale;
    p.out_src = a.out_src;
    p.T = a.T;
    p.S = a.S;
    p.s = a.s;
    p.flags = a.flags;
    p.max_ctas = a.max_ctas;
    const bool h16 = a.colscale != nullptr && p.mode != TC_SEPARATE;
    p.colscale = a.colscale;
    p.rowmax = p.mode == TC_RATIO ? a.rowmax : nullptr;
    p.stages = stages_for(bn, RING_OFF, h16);
    if (p.mode == TC_RATIO && a.Vhat) return cudaErrorInvalidValue;   // RATIO always goes through TMA
    return launch_tc(p, a.A, a.lda, a.V, a.R, st, nullptr, h16);
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
    p.tma_epi = 1;
    p.Bsplit = a.Bsplit;
    p.nkb_total = a.nkb_total;
    p.ldc = a.ldb;
    p.max_ctas = a.max_ctas;
    const bool h16 = a.colscale != nullptr;   // 3xFP16 products on R' (rows scaled by 2^(14 - E_t))
    p.colscale = a.colscale;
    p.rowmax = h16 ? const_cast<unsigned *>(a.rowmax) : nullptr;
    if (h16) p.stages = stages_for(bn, RING_OFF, true);
    return launch_tc(p, a.A, a.lda, a.theta, a.n_out, st, nullptr, h16);
}

int tc_split_count(int64_t k_len) {
    const int n_kb = (int)((k_len + TC_KB - 1) / TC_KB);
    return (n_kb + CHUNK_KB - 1) / CHUNK_KB;
}

int tc_pick_bn_split(int64_t n, int64_t rows, int splits, int sms) {
    if (const char *e = getenv("NFHMM_SPLIT_BN")) {   // A/B experiments: one width for both contractions
        const int b = atoi(e);
        if (b >= 16 && b <= TC_MAX_BN && b % 16 == 0) return b;
    }
    // split-K units all carry one accumulation chunk: time ~ waves of units (the per-k-block step time
    // measured ~0.6 us from BN = 32 to 176), then the widest tile
    const int64_t mt = (rows + TC_BM - 1) / TC_BM;
    int best = 16;
    int64_t best_waves = INT64_MAX;
    for (int bn = 16; bn <= TC_MAX_BN; bn += 16) {
        const int64_t nt = (n + bn - 1) / bn;
        const int64_t waves = (mt * nt * splits + sms - 1) / sms;
        if (waves < best_waves || (waves == best_waves && bn < best)) {
            best_waves = waves;
            best = bn;
        }
    }
    return best;
}

cudaError_t launch_recon_tc_split(int bn, const ReconArgs &a, float *part, cudaStream_t st) {
    TcParams p{};
    p.mode = TC_RATIO;
    p.M = a.M;
    p.bn = bn;
    p.n_tiles = (a.F + bn - 1) / bn;
    p.k_begin = a.k_begin;
    p.k_end = a.k_end;
    p.stages = stages_for(bn);
    p.Bsplit = a.Bsplit;
    p.nkb_total = a.nkb_total;
    p.ldc = a.ldv;
    p.F = a.F;
    p.flags = a.flags;
    p.max_ctas = a.max_ctas;
    const bool h16 = a.colscale != nullptr;
    p.colscale = a.colscale;
    p.rowmax = a.rowmax;
    p.stages = stages_for(bn, RING_OFF, h16);
    // ceil(k / 256) accumulation chunks either way (16 k-blocks of 16 or 8 of 32)
    p.splits = tc_split_count(a.k_end - (a.k_begin & ~((h16 ? TC_KB16 : TC_KB) - 1)));
    p.part = part;
    p.ldp = p.n_tiles * bn;
    if (!a.R || a.Vhat || p.ldp < a.ldv) return cudaErrorInvalidValue;
    return launch_split(p, a.A, a.lda, a.V, a.R, a.ldv, a.data_part, st, h16);
}

int tc_fused_blocks_per_chunk(int K) { return (2 * K - 2 + 32) / K; }

cudaError_t launch_backproj_dirichlet_tc(int bn, int n_valid, const BackprojArgs &a, const FusedDirichletArgs &d,
                                         cudaStream_t st) {
    if (bn % d.K || d.K > 32 || d.ldf % 4 || a.ldb % 4) return cudaErrorInvalidValue;
    TcParams p{};
    p.mode = TC_DIRICHLET;
    p.M = a.M;
    p.bn = bn;
    p.n_tiles = (n_valid + bn - 1) / bn;
    p.k_begin = 0;
    p.k_end = a.Kpad;
    p.nbc = tc_fused_blocks_per_chunk(d.K);
    p.ring_off = (RING_OFF + EPI_WARPS * p.nbc * 128 + 1023) & ~1023;
    p.stages = stages_for(bn, p.ring_off);
    p.tma_epi = 1;
    p.Bsplit = a.Bsplit;
    p.nkb_total = a.nkb_total;
    p.ldc = a.ldb;
    p.K = d.K;
    p.Kt = d.Kt;
    p.SN = d.SN;
    p.ldf = d.ldf;
    p.fconst = d.fconst;
    p.spsT = d.spsT;
    p.sps2T = d.sps2T;
    p.hpartT = d.hpartT;
    p.alpha_out = d.alpha_out;
    return launch_tc(p, a.A, a.lda, a.theta, const_cast<float *>(a.theta), st, d.dvT);
}

}  // namespace nfk
