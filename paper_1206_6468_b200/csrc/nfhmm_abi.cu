// nfhmm_abi.cu -- host runtime behind the C-ABI of include/nfhmm.h: handle, workspace carving, argument
// validation, the per-sweep launch sequence and the copies in/out.  Every step of the path runs in the
// kernels of gemm_simt.cu, dirichlet.cu, fb.cu and misc.cu; there is no CPU fallback.
#include <cuda_runtime.h>
#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <string.h>

#include <string>
#include <vector>

#include "nfhmm_internal.cuh"

using namespace nfk;

struct nfhmm {
    int64_t F = 0, T = 0, M = 0, frames = 0;
    int S = 0, N = 0, K = 0, Kt = 0;
    int Fa = 0, Kb = 0, bn_a = 0, bn_b = 0, nt_a = 0;
    int math = NFHMM_MATH_TC, bn_tc_a = 0, bn_tc_b = 0, nt_tc_a = 0;
    double gamma = 1.0;
    int device = 0, max_iters = 1024, free_energy = 1;
    cudaStream_t st = nullptr;

    void *ws = nullptr;
    size_t ws_bytes = 0;
    bool ws_owned = false;

    float *betaT = nullptr, *beta = nullptr, *trans = nullptr, *prior = nullptr;
    float *V = nullptr, *R = nullptr, *theta = nullptr, *alpha = nullptr;
    float *bwd = nullptr, *ec = nullptr, *fwd = nullptr;   // FB messages b, u (q(D) = u .* b / sum), emissions
    float *vt = nullptr, *scale = nullptr, *vsrc = nullptr;
    float *bs_a = nullptr, *bs_b = nullptr;   // tensor-core path: pre-split beta for (a) and betaT for (b)
    float *bs_a16 = nullptr, *csa = nullptr;  // 3xFP16 reconstruction: FP16 image of beta and its column scales
    bool h16 = false;
    // 3xFP16 back-projection (needs h16: the reconstruction then writes R' = c_l R and the per-row maxima)
    float *bs_b16 = nullptr, *csb = nullptr;
    unsigned *rowmax = nullptr;
    bool h16b = false;
    double *eoff = nullptr, *logZ = nullptr, *data_part = nullptr, *hdir = nullptr, *fe = nullptr;
    double *fconst = nullptr;   // per-frame alpha_0, psi(alpha_0), bound constant (set_observations)
    double *elbo_part = nullptr;   // [M][ELBO_MAX_BLOCKS] bound partial sums
    unsigned *elbo_ctr = nullptr;  // [M] per-mixture block counters of the bound kernel
    // Dirichlet step fused into the back-projection epilogue (tensor-core engine, K <= 32): block-major
    // pseudo-counts, Eq. 8 block sums and g~ partials, frame pitch ldf
    bool fused = false;
    int dir_variant = 0;   // Dirichlet kernel variant (NFHMM_DIRICHLET=tile: frame-tile kernel)
    int fb_wide = 1;       // N > 64: multi-warp forward-backward (NFHMM_FB_WIDE=0: one warp per direction)
    // forward-backward overlapped with the reconstruction GEMM: the GEMM's persistent grid leaves
    // `overlap_sms` SMs to the latency-bound recursion, which runs on a side stream (fork / join events)
    int overlap_sms = 0, num_sms = 0;
    // the next sweep's back-projection (b) joins the reconstruction in the forward-backward's shadow: (b) of
    // sweep i+1 needs only R (from (a) of sweep i) and theta~, so the side-stream recursion overlaps (a) and
    // (b); n_ready = n for the coming sweep already sits in the alpha buffer (never after a call's last sweep)
    bool defer = false, n_ready = false;
    bool fb_first = false;   // launch the recursion before the GEMM (few chains: the recursion is the longer branch)
    cudaStream_t fbst = nullptr;
    cudaStream_t pst = nullptr;    // NFHMM_PRIO=1 (experiment): the contractions of the overlapped sweep on a high-priority stream
    cudaEvent_t pev = nullptr;
    int prio = -1;
    cudaEvent_t fev[2] = {nullptr, nullptr};
    int ldf = 0, nt_tc_b = 0;
    // split-K reconstruction for few row tiles (single mixtures): units of one accumulation chunk + reduce
    int split = 0;
    float *tcpart = nullptr;
    float *dvT = nullptr;
    double *spsT = nullptr, *sps2T = nullptr, *hpartT = nullptr;
    // parallel-in-time forward-backward (few chains): chunks, their transfer matrices and start messages
    int fb_nchunk = 0, fb_len = 0;
    int fb_multi = 1;   // chains per warp: 1 FFMA2 multi-chain (default), 2 tensor-core kernel, 0 one (NFHMM_FB_MULTI)
    float *fbP = nullptr, *fbPT = nullptr, *fbF = nullptr, *fbB = nullptr;
    int *fbE = nullptr;
    // CUDA graphs of one sweep (mid: alpha not stored; last: alpha stored), replayed on an internal stream
    // bridged to the caller's stream with events (the legacy default stream cannot be captured)
    bool graphs = true;
    cudaStream_t gst = nullptr;
    cudaEvent_t gev[2] = {nullptr, nullptr};
    cudaGraphExec_t gx[2] = {nullptr, nullptr};
    int64_t g_kernels = 0;      // kernels per captured sweep
    int eager_sweeps = 0;       // sweeps run eagerly by this handle (capture only after one)
    unsigned *flags = nullptr;
    // guard zones (NFHMM_GUARD=<bytes>, a bounds checker in place of compute-sanitizer): every workspace
    // piece is followed (and the first preceded) by a zone filled with kGuardByte at set_workspace, from
    // the piece's exact end; nfhmm_guard_check counts the zone bytes a kernel overwrote
    size_t guard = 0;
    struct Zone { size_t off, len; int piece; };
    std::vector<Zone> zones;

    bool have_model = false, have_obs = false, R_valid = false;
    int iters_done = 0;
    int64_t launches = 0;
    double c_prior_T = 0.0;
    std::string err;
    // per-kernel-class profiling (events bracketing each launch)
    bool prof = false;
    struct Rec { int cls; cudaEvent_t a, b; };
    std::vector<Rec> recs;
    std::vector<cudaEvent_t> pool;
    size_t pool_used = 0;
};

namespace {

const int kReconBN[] = {40, 64, 88, 104, 128};
const int kBackBN[] = {24, 64, 80, 120, 128, 160};

int pick_bn(int64_t n, const int *c, int nc) {
    int best = -1;
    int64_t best_pad = INT64_MAX;
    for (int i = 0; i < nc; ++i) {
        const int64_t pad = (n + c[i] - 1) / c[i] * c[i];
        if (pad < best_pad || (pad == best_pad && c[i] > best)) {
            best_pad = pad;
            best = c[i];
        }
    }
    return best;
}

int fail(nfhmm_t *h, int code, const char *fmt, ...) {
    if (h) {
        char buf[512];
        va_list ap;
        va_start(ap, fmt);
        vsnprintf(buf, sizeof buf, fmt, ap);
        va_end(ap);
        h->err = buf;
    }
    return code;
}

#define CU(h, call)                                                                            \
    do {                                                                                       \
        cudaError_t e_ = (call);                                                               \
        if (e_ != cudaSuccess) return fail(h, NFHMM_ECUDA, "%s: %s", #call, cudaGetErrorString(e_)); \
    } while (0)

cudaEvent_t prof_event(nfhmm_t *h) {
    if (h->pool_used == h->pool.size()) {
        cudaEvent_t e;
        if (cudaEventCreate(&e) != cudaSuccess) return nullptr;
        h->pool.push_back(e);
    }
    return h->pool[h->pool_used++];
}

#define LAUNCH(h, cls, call)                                                   \
    do {                                                                       \
        cudaEvent_t ea_ = nullptr, eb_ = nullptr;                              \
        if ((h)->prof) {                                                       \
            ea_ = prof_event(h);                                               \
            eb_ = prof_event(h);                                               \
            if (ea_) cudaEventRecord(ea_, (h)->st);                            \
        }                                                                      \
        CU(h, call);                                                           \
        (h)->launches++;                                                       \
        if (ea_ && eb_) {                                                      \
            cudaEventRecord(eb_, (h)->st);                                     \
            (h)->recs.push_back({cls, ea_, eb_});                              \
        }                                                                      \
    } while (0)

bool is_device_ptr(const void *p) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

size_t al(size_t b) { return (b + 255) & ~size_t(255); }

const int kGuardByte = 0xA5;

// Carve (or just size) the workspace.  Order is fixed; sizes in bytes.
size_t carve(nfhmm_t *h, char *base) {
    const size_t fr = (size_t)h->frames, Fa = h->Fa, Kb = h->Kb;
    const size_t chainTN = (size_t)h->M * h->S * h->T * h->N, chainT = (size_t)h->M * h->S * h->T;
    const size_t g = al(h->guard);
    size_t o = g;
    int piece = 0;
    h->zones.clear();
    if (g) h->zones.push_back({0, g, -1});
    auto take = [&](size_t bytes) {
        char *p = base ? base + o : nullptr;
        if (g) h->zones.push_back({o + bytes, al(bytes) - bytes + g, piece});
        o += al(bytes) + g;
        ++piece;
        return p;
    };
    char *p;
    p = take(Kb * Fa * 4);                       h->betaT = (float *)p;
    p = take(Fa * Kb * 4);                       h->beta = (float *)p;
    p = take((size_t)h->S * h->N * h->N * 4);    h->trans = (float *)p;
    p = take((size_t)h->S * h->N * 4);           h->prior = (float *)p;
    p = take(fr * Fa * 4);                       h->V = (float *)p;
    p = take(fr * Fa * 4);                       h->R = (float *)p;
    p = take(fr * Kb * 4);                       h->theta = (float *)p;
    p = take(fr * Kb * 4);                       h->alpha = (float *)p;
    p = take(chainTN * 4);                       h->bwd = (float *)p;
    p = take(chainTN * 4);                       h->ec = (float *)p;
    p = take(chainTN * 4);                       h->fwd = (float *)p;
    p = take(chainT * 8);                        h->eoff = (double *)p;
    p = take((size_t)h->M * h->S * 8);           h->logZ = (double *)p;
    {
        size_t nt = (size_t)(h->nt_a > h->nt_tc_a ? h->nt_a : h->nt_tc_a);
        if (h->split && (size_t)(h->Fa + 15) / 16 > nt) nt = (size_t)(h->Fa + 15) / 16;   // split: 16-col sub-tiles
        p = take(fr * nt * 8);                   h->data_part = (double *)p;
    }
    p = take(fr * 8);                            h->hdir = (double *)p;
    p = take(fr * 4 * 8);                        h->fconst = (double *)p;
    p = take((size_t)h->M * ELBO_MAX_BLOCKS * 8); h->elbo_part = (double *)p;
    p = take((size_t)h->M * 4);                  h->elbo_ctr = (unsigned *)p;
    {   // parallel-in-time FB scratch (NMAX <= 64 on that path)
        const size_t units = (size_t)h->M * h->S * (size_t)h->fb_nchunk;
        p = take(units * 64 * 64 * 4);           h->fbP = (float *)p;
        p = take(units * 64 * 64 * 4);           h->fbPT = (float *)p;
        p = take(units * 64 * 4);                h->fbF = (float *)p;
        p = take(units * 64 * 4);                h->fbB = (float *)p;
        p = take(units * 64 * 4);                h->fbE = (int *)p;
    }
    p = take((size_t)h->M * h->max_iters * 8);   h->fe = (double *)p;
    p = take(fr * 4);                            h->vt = (float *)p;
    p = take(fr * 4);                            h->scale = (float *)p;
    p = take((size_t)h->M * h->S * h->T * h->F * 4); h->vsrc = (float *)p;
    p = take(tc_presplit_floats(h->F, h->Kt, h->bn_tc_a) * 4); h->bs_a = (float *)p;
    p = take(tc_presplit_floats(h->Kt, h->Fa, h->bn_tc_b) * 4); h->bs_b = (float *)p;
    if (h->h16) {
        p = take(tc_presplit16_floats(h->F, h->Kt, h->bn_tc_a) * 4);  h->bs_a16 = (float *)p;
        p = take((size_t)h->nt_tc_a * h->bn_tc_a * 4);               h->csa = (float *)p;
        p = take(fr * 4);                                            h->rowmax = (unsigned *)p;
    }
    if (h->h16b) {
        p = take(tc_presplit16_floats(h->Kt, h->Fa, h->bn_tc_b) * 4); h->bs_b16 = (float *)p;
        p = take((size_t)h->nt_tc_b * h->bn_tc_b * 4);               h->csb = (float *)p;
    }
    if (h->fused) {
        const size_t sn = (size_t)h->S * h->N, ldf = (size_t)h->ldf;
        p = take(sn * ldf * 4);                  h->dvT = (float *)p;
        p = take(sn * ldf * 8);                  h->spsT = (double *)p;
        p = take(sn * ldf * 8);                  h->sps2T = (double *)p;
        p = take((size_t)h->nt_tc_b * ldf * 8);  h->hpartT = (double *)p;
    }
    if (h->split) {   // split-K partial sums (the larger of the two contractions)
        const size_t pa = (size_t)tc_split_count(h->Kt) * fr * (size_t)h->nt_tc_a * h->bn_tc_a;
        p = take(pa * 4);                        h->tcpart = (float *)p;
    }
    p = take(256);                               h->flags = (unsigned *)p;
    return o;
}

// Bytes the workspace needs (sized on a copy so the live handle's pointers are untouched).
size_t ws_need(const nfhmm_t *h) {
    nfhmm tmp = *h;
    return carve(&tmp, nullptr);
}

int check_flags(nfhmm_t *h) {
    unsigned f = 0;
    CU(h, cudaMemcpyAsync(&f, h->flags, sizeof f, cudaMemcpyDeviceToHost, h->st));
    CU(h, cudaStreamSynchronize(h->st));
    if (f & FLAG_BAD_INPUT) return fail(h, NFHMM_EINVAL, "observations contain negative or non-finite values");
    if (f & FLAG_ZERO_SUPPORT) return fail(h, NFHMM_EZEROSUPPORT, "V > 0 where V_hat = 0 (zero support, S:278)");
    if (f & FLAG_NONFINITE) return fail(h, NFHMM_ENUMERIC, "non-finite alpha, phi or log Z");
    return NFHMM_OK;
}

// (a) / (f) reconstruction GEMM on the selected engine: sets the operand layout the engine expects.
int run_recon(nfhmm_t *h, int cls, ReconArgs a) {
    if (h->math == NFHMM_MATH_TC) {
        a.B = h->beta;      // [F_pad][Kt_pad], K-major rows
        a.Bsplit = h->bs_a;
        a.nkb_total = (h->Kt + 15) / 16;
        if (h->h16 && !a.out_src) {   // A = theta~: the 3xFP16 products (DESIGN "3xFP16 products")
            a.Bsplit = h->bs_a16;
            a.nkb_total = (h->Kt + 31) / 32;
            a.colscale = h->csa;
            if (a.R && h->h16b) a.rowmax = h->rowmax;   // per-row maxima of R' (3xFP16 back-projection;
                                                          // zeroed by recon_ratio's caller)
        }
        a.ldb = h->Kb;
        a.n_tiles = h->nt_tc_a;
        if (h->split && a.R && !a.Vhat) {
            LAUNCH(h, cls, launch_recon_tc_split(h->bn_tc_a, a, h->tcpart, h->st));
        } else {
            LAUNCH(h, cls, launch_recon_tc(h->bn_tc_a, a, h->st));
        }
    } else {
        a.B = h->betaT;     // [Kt_pad][F_pad]
        a.ldb = h->Fa;
        a.n_tiles = h->nt_a;
        LAUNCH(h, cls, launch_recon(h->bn_a, a, h->st));
    }
    return NFHMM_OK;
}

int data_tiles(const nfhmm_t *h) {
    if (h->math == NFHMM_MATH_TC) return h->split ? (int)((h->Fa + 15) / 16) : h->nt_tc_a;
    return h->nt_a;
}

// zero: clear the per-row maxima of R' first (the overlapped sweep clears them before its fork, so that no
// memset kernel sits between the fork and the capped GEMM grid: the recursion's CTAs would take the SMs first)
int recon_ratio(nfhmm_t *h, int max_ctas = 0, bool zero = true) {
    if (zero && h->h16b) CU(h, cudaMemsetAsync(h->rowmax, 0, (size_t)h->frames * 4, h->st));
    ReconArgs a{};
    a.max_ctas = max_ctas;
    a.M = (int)h->frames;
    a.k_begin = 0;
    a.k_end = h->Kt;
    a.A = h->theta;
    a.lda = h->Kb;
    a.B = h->betaT;
    a.ldb = h->Fa;
    a.F = (int)h->F;
    a.V = h->V;
    a.ldv = h->Fa;
    a.R = h->R;
    a.data_part = h->data_part;
    a.flags = h->flags;
    return run_recon(h, NFHMM_K_RECON, a);
}

DirichletArgs dirichlet_args(nfhmm_t *h, bool write_alpha);

// (b) n = theta .* (R beta): the Eq. 6 data term  sum_l V_lt z_{t,l,k}; fused engine: (b) with the
// element step of (c)+(d) in its epilogue (theta updated in place, alpha stored on the last sweep)
int step_backproj(nfhmm_t *h, bool last = true, int max_ctas = 0) {
    BackprojArgs b{};
    b.max_ctas = max_ctas;
    b.M = (int)h->frames;
    b.Kpad = h->Fa;
    b.A = h->R;
    b.lda = h->Fa;
    b.B = h->beta;
    b.ldb = h->Kb;
    b.theta = h->theta;
    b.n_out = h->alpha;
    if (h->math == NFHMM_MATH_TC) {
        b.B = h->betaT;     // [Kt_pad][F_pad], K-major rows
        b.Bsplit = h->bs_b;
        b.nkb_total = (h->Fa + 15) / 16;
        if (h->fused) {
            FusedDirichletArgs d{};
            d.K = h->K;
            d.Kt = h->Kt;
            d.SN = h->S * h->N;
            d.ldf = h->ldf;
            d.dvT = h->dvT;
            d.fconst = h->fconst;
            d.spsT = h->spsT;
            d.sps2T = h->sps2T;
            d.hpartT = h->free_energy ? h->hpartT : nullptr;
            d.alpha_out = last ? h->alpha : nullptr;
            LAUNCH(h, NFHMM_K_BACKPROJ, launch_backproj_dirichlet_tc(h->bn_tc_b, h->Kt, b, d, h->st));
            return NFHMM_OK;
        }
        if (h->h16b) {   // A = R' (rows scaled by 2^(14 - E_t)), B = beta^T / c_l in FP16
            b.Bsplit = h->bs_b16;
            b.nkb_total = (h->Fa + 31) / 32;
            b.colscale = h->csb;
            b.rowmax = h->rowmax;
        }
        LAUNCH(h, NFHMM_K_BACKPROJ, launch_backproj_tc(h->bn_tc_b, h->Kt, b, h->st));
    } else {
        LAUNCH(h, NFHMM_K_BACKPROJ, launch_backproj(h->bn_b, b, h->st));
    }
    return NFHMM_OK;
}

// (c)+(d) Eq. 6, digamma/exp, Eq. 8
DirichletArgs dirichlet_args(nfhmm_t *h, bool write_alpha) {
    DirichletArgs d{};
    d.frames = (int)h->frames;
    d.T = (int)h->T;
    d.S = h->S;
    d.N = h->N;
    d.K = h->K;
    d.Kt = h->Kt;
    d.ld = h->Kb;
    d.gamma = (float)h->gamma;
    d.n_in = h->alpha;
    d.alpha = h->alpha;
    d.theta = h->theta;
    d.u_fwd = h->fwd;
    d.b_bwd = h->bwd;
    d.ec = h->ec;
    d.eoff = h->eoff;
    d.fconst = h->fconst;
    d.write_alpha = write_alpha ? 1 : 0;
    d.hdir = h->free_energy ? h->hdir : nullptr;
    d.flags = h->flags;
    d.ldf = h->ldf;
    d.variant = h->dir_variant;
    return d;
}

int step_dirichlet(nfhmm_t *h, bool write_alpha) {
    const DirichletArgs d = dirichlet_args(h, write_alpha);
    LAUNCH(h, NFHMM_K_DIRICHLET, launch_dirichlet(d, h->st));
    return NFHMM_OK;
}

// fused engine: pseudo-counts gamma d + 1 before (b), Eq. 8 emissions and H_t after it
int step_dv(nfhmm_t *h) {
    const DirichletArgs d = dirichlet_args(h, false);
    LAUNCH(h, NFHMM_K_DIRICHLET, launch_dv(d, h->dvT, h->st));
    return NFHMM_OK;
}
int step_eq8(nfhmm_t *h) {
    const DirichletArgs d = dirichlet_args(h, false);
    LAUNCH(h, NFHMM_K_DIRICHLET, launch_eq8(d, h->spsT, h->sps2T, h->hpartT, h->nt_tc_b, h->bn_tc_b, h->st));
    return NFHMM_OK;
}

// (e) forward-backward per source
int step_fb(nfhmm_t *h) {
    // NFHMM_SKIP_FB=1: timing experiment only (what the sweep costs without the recursion; the posteriors
    // are then wrong) -- used to measure how much of the forward-backward the overlap hides
    static const int skip_fb = getenv("NFHMM_SKIP_FB") ? atoi(getenv("NFHMM_SKIP_FB")) : 0;
    if (skip_fb) return NFHMM_OK;
    FBArgs f{};
    f.M = (int)h->M;
    f.S = h->S;
    f.T = (int)h->T;
    f.N = h->N;
    f.ec = h->ec;
    f.eoff = h->eoff;
    f.trans = h->trans;
    f.prior = h->prior;
    f.fwd = h->fwd;
    f.bwd = h->bwd;
    f.nchunk = h->fb_nchunk;
    f.chunk_len = h->fb_len;
    f.P = h->fbP;
    f.PT = h->fbPT;
    f.PE = h->fbE;
    f.fstart = h->fbF;
    f.bstart = h->fbB;
    f.logZ = h->logZ;
    f.flags = h->flags;
    f.wide = h->fb_wide;
    f.multi = h->fb_multi;
    LAUNCH(h, NFHMM_K_FB, launch_fb(f, h->st));
    return NFHMM_OK;
}

// One VB sweep.  `last`: the final sweep of this call, which also stores alpha (posteriors, separation).
int sweep(nfhmm_t *h, bool last) {
    if (!h->R_valid) {
        int r = recon_ratio(h);
        if (r) return r;
        h->R_valid = true;
    }
    int r = NFHMM_OK;
    if (h->fused) {
        r = step_dv(h);
        if (!r) r = step_backproj(h, last);
        if (!r) r = step_eq8(h);
    } else {
        if (!h->n_ready) r = step_backproj(h);
        h->n_ready = false;
        if (!r) r = step_dirichlet(h, last);
    }
    if (r) return r;
    if (h->overlap_sms > 0 && !h->prof) {   // (per-launch profiling times every kernel on its own)
        // (a) and (e) are independent given the new alpha: the reconstruction GEMM (launched first, on
        // num_sms - overlap_sms SMs) and the forward-backward (side stream, the remaining SMs) overlap;
        // the bound waits for both
        if (!h->fbst) {
            CU(h, cudaStreamCreateWithFlags(&h->fbst, cudaStreamNonBlocking));
            CU(h, cudaEventCreateWithFlags(&h->fev[0], cudaEventDisableTiming));
            CU(h, cudaEventCreateWithFlags(&h->fev[1], cudaEventDisableTiming));
        }
        if (h->prio < 0) {
            const char *ep = getenv("NFHMM_PRIO");
            h->prio = (ep && atoi(ep) != 0 && !h->graphs) ? 1 : 0;
            if (h->prio) {
                int lo = 0, hi = 0;
                CU(h, cudaDeviceGetStreamPriorityRange(&lo, &hi));
                CU(h, cudaStreamCreateWithPriority(&h->pst, cudaStreamNonBlocking, hi));
                CU(h, cudaEventCreateWithFlags(&h->pev, cudaEventDisableTiming));
            }
        }
        if (h->h16b) CU(h, cudaMemsetAsync(h->rowmax, 0, (size_t)h->frames * 4, h->st));
        CU(h, cudaEventRecord(h->fev[0], h->st));
        CU(h, cudaStreamWaitEvent(h->fbst, h->fev[0], 0));
        // launch order decides who takes the SMs first: the GEMM for many chains (its capped grid, the
        // recursion in the rest), the recursion for few chains (there the recursion is the longer branch)
        cudaStream_t main_st = h->st;
        if (h->fb_first) {
            h->st = h->fbst;
            r = step_fb(h);
            h->st = main_st;
            if (r) return r;
        }
        if (h->prio) {   // pending recursion CTAs must not take the SMs (a) frees ahead of (b)'s CTAs
            CU(h, cudaStreamWaitEvent(h->pst, h->fev[0], 0));
            h->st = h->pst;
        }
        r = recon_ratio(h, h->num_sms - h->overlap_sms, false);
        h->st = main_st;
        if (r) return r;
        if (!h->fb_first) {
            h->st = h->fbst;
            r = step_fb(h);
            h->st = main_st;
            if (r) return r;
        }
        if (h->defer && !last && !h->fused) {   // (b) of sweep i+1, still beside the recursion
            if (h->prio) h->st = h->pst;
            r = step_backproj(h, true, h->num_sms - h->overlap_sms);
            h->st = main_st;
            if (r) return r;
            h->n_ready = true;
        }
        if (h->prio) {
            CU(h, cudaEventRecord(h->pev, h->pst));
            CU(h, cudaStreamWaitEvent(h->st, h->pev, 0));
        }
        CU(h, cudaEventRecord(h->fev[1], h->fbst));
        CU(h, cudaStreamWaitEvent(h->st, h->fev[1], 0));
    } else {
        r = step_fb(h);
        if (r) return r;
        // (a) z-step of the new alpha: R for the next sweep and the data term of L_i
        r = recon_ratio(h);
        if (r) return r;
    }
    // (g) L_i (row iters_done of fe; the kernel keeps the index in a device counter)
    if (h->free_energy) {
        ElboArgs e{};
        e.M = (int)h->M;
        e.T = (int)h->T;
        e.n_tiles = data_tiles(h);
        e.S = h->S;
        e.iter_ctr = reinterpret_cast<int *>(h->flags + 1);
        e.done_ctr = h->flags + 2;
        e.part = h->elbo_part;
        e.mix_ctr = h->elbo_ctr;
        e.max_iters = h->max_iters;
        e.c_prior_T = h->c_prior_T;
        e.data_part = h->data_part;
        e.hdir = h->hdir;
        e.logZ = h->logZ;
        e.fe = h->fe;
        LAUNCH(h, NFHMM_K_ELBO, launch_elbo(e, h->st));
    }
    h->iters_done++;
    return NFHMM_OK;
}

void drop_graphs(nfhmm_t *h) {
    for (int i = 0; i < 2; ++i)
        if (h->gx[i]) {
            cudaGraphExecDestroy(h->gx[i]);
            h->gx[i] = nullptr;
        }
}

// Capture one sweep (last = store alpha) into h->gx[last] on the internal stream.
int capture_sweep(nfhmm_t *h, bool last) {
    if (!h->gst) {
        CU(h, cudaStreamCreateWithFlags(&h->gst, cudaStreamNonBlocking));
        CU(h, cudaEventCreateWithFlags(&h->gev[0], cudaEventDisableTiming));
        CU(h, cudaEventCreateWithFlags(&h->gev[1], cudaEventDisableTiming));
    }
    cudaStream_t user = h->st;
    const int64_t l0 = h->launches;
    const int done = h->iters_done;
    const bool ready = h->n_ready;
    h->st = h->gst;
    cudaGraph_t g = nullptr;
    cudaError_t e = cudaStreamBeginCapture(h->gst, cudaStreamCaptureModeThreadLocal);
    int r = e == cudaSuccess ? sweep(h, last) : NFHMM_ECUDA;
    cudaError_t e2 = cudaStreamEndCapture(h->gst, &g);
    h->st = user;
    h->iters_done = done;
    h->n_ready = ready;
    const int64_t k = h->launches - l0;
    h->launches = l0;
    if (r) return r;
    if (e != cudaSuccess || e2 != cudaSuccess) {
        if (g) cudaGraphDestroy(g);
        return fail(h, NFHMM_ECUDA, "graph capture: %s", cudaGetErrorString(e != cudaSuccess ? e : e2));
    }
    e = cudaGraphInstantiate(&h->gx[last ? 1 : 0], g, 0);
    cudaGraphDestroy(g);
    if (e != cudaSuccess) return fail(h, NFHMM_ECUDA, "graph instantiate: %s", cudaGetErrorString(e));
    h->g_kernels = k;
    return NFHMM_OK;
}

int enter(nfhmm_t *h) {
    if (!h) return NFHMM_EINVAL;
    h->err.clear();
    CU(h, cudaSetDevice(h->device));
    return NFHMM_OK;
}

}  // namespace

extern "C" {

void nfhmm_default_options(nfhmm_options *o) {
    if (!o) return;
    memset(o, 0, sizeof *o);
    o->n_mix = 1;
    o->gamma = 1.0;
    o->device = 0;
    o->max_iters = 1024;
    o->free_energy = 1;
    o->math = NFHMM_MATH_TC;
    o->stream = nullptr;
}

int nfhmm_create(int64_t F, int64_t T, int32_t S, int32_t N, int32_t K, const nfhmm_options *opt, nfhmm_t **out) {
    if (!out) return NFHMM_EINVAL;
    *out = nullptr;
    nfhmm_options o;
    nfhmm_default_options(&o);
    if (opt) o = *opt;
    if (F < 1 || T < 1 || S < 1 || N < 1 || K < 1 || o.n_mix < 1 || !(o.gamma >= 0.0) || !isfinite(o.gamma) ||
        o.max_iters < 1 || (o.math != NFHMM_MATH_TC && o.math != NFHMM_MATH_SIMT))
        return NFHMM_EINVAL;
    if (N > 128) return NFHMM_EINVAL;  // forward-backward keeps <= 4 states per lane
    const char *eg = getenv("NFHMM_GUARD");
    const long long guard = eg ? atoll(eg) : 0;
    if (guard < 0 || guard > (1LL << 30)) return NFHMM_EINVAL;
    const int64_t Kt = (int64_t)S * N * K;
    const int64_t frames = o.n_mix * T;
    if (Kt > (1 << 24) || F > (1 << 24) || frames > (int64_t)1 << 30) return NFHMM_EINVAL;
    nfhmm_t *h = new (std::nothrow) nfhmm;
    if (!h) return NFHMM_ENOMEM;
    h->guard = (size_t)guard;
    h->F = F;
    h->T = T;
    h->S = S;
    h->N = N;
    h->K = K;
    h->Kt = (int)Kt;
    h->M = o.n_mix;
    h->frames = frames;
    h->gamma = o.gamma;
    h->device = o.device;
    h->max_iters = o.max_iters;
    h->free_energy = o.free_energy ? 1 : 0;
    h->st = (cudaStream_t)o.stream;
    h->bn_a = pick_bn(F, kReconBN, sizeof kReconBN / sizeof *kReconBN);
    h->bn_b = pick_bn(Kt, kBackBN, sizeof kBackBN / sizeof *kBackBN);
    h->Fa = (int)((F + h->bn_a - 1) / h->bn_a * h->bn_a);
    h->Kb = (int)((Kt + h->bn_b - 1) / h->bn_b * h->bn_b);
    h->nt_a = h->Fa / h->bn_a;
    h->math = o.math == NFHMM_MATH_SIMT ? NFHMM_MATH_SIMT : NFHMM_MATH_TC;
    {   // CUDA-graph replay of the sweeps for launch-bound (small) problems: measured +23 % at config 0,
        // +7 % at config 1, -1 % at config 3 (512k frames, where launch gaps are negligible).
        // NFHMM_GRAPHS=0 / 1 forces it off / on.
        const char *e = getenv("NFHMM_GRAPHS");
        h->graphs = e ? atoi(e) != 0 : frames <= 65536;
    }
    {   // parallel-in-time forward-backward for few chains (NFHMM_FB_PARALLEL=0 disables)
        const char *e = getenv("NFHMM_FB_PARALLEL");
        int L = 0;
        const int nc = (e && atoi(e) == 0) ? 0 : fb_pick_chunks(h->M * h->S, h->T, h->N, &L);
        h->fb_nchunk = nc > 1 ? nc : 0;
        h->fb_len = nc > 1 ? L : 0;
    }
    h->bn_tc_a = tc_pick_bn(F, 16, frames);
    {   // Dirichlet element step fused into the back-projection epilogue (opt-in, NFHMM_FUSED=1): correct
        // but measured slower (DESIGN "Fused Dirichlet epilogue"): the element work competes with the
        // GEMM's own epilogue / converter issue slots and stalls the MMAs.  Column tiles of whole K-blocks.
        const char *e = getenv("NFHMM_FUSED");
        int l = 16;
        while (l % K) l += 16;   // lcm(16, K)
        const int64_t SN = (int64_t)S * N;
        h->fused = h->math == NFHMM_MATH_TC && K <= 32 && l <= 192 && SN * 33 * 8 <= 200 * 1024 &&
                   e && atoi(e) != 0;
        h->bn_tc_b = h->fused ? tc_pick_bn(Kt, l, frames) : tc_pick_bn(Kt, 16, frames);
        h->nt_tc_b = (int)((Kt + h->bn_tc_b - 1) / h->bn_tc_b);
        h->ldf = (int)((frames + 31) / 32 * 32);
        const char *ed = getenv("NFHMM_DIRICHLET");
        h->dir_variant = (ed && strcmp(ed, "tile") == 0) ? 1 : (ed && strcmp(ed, "pipe") == 0) ? 2 : 0;
        const char *ew = getenv("NFHMM_FB_WIDE");
        h->fb_wide = (ew && atoi(ew) == 0) ? 0 : 1;
        const char *em = getenv("NFHMM_FB_MULTI");
        // (the tensor-core kernel, NFHMM_FB_MULTI=2, measured 68 vs 90 ms per step alone but needs >= 16 SMs
        // beside the reconstruction GEMM and measured no faster there: 77.9 vs 80.1 M frame-iterations/s)
        // (up to 64 chains the one-chain kernel, whose step is shorter, wins: at 32 mixtures of config 3 --
        // the per-GPU share on 8 GPUs -- 68.6 -> 94.3 M frame-iterations/s; at 64 mixtures the multi-chain
        // kernel, 103.6 vs 97.5 M)
        h->fb_multi = em ? atoi(em) : (h->M * h->S > 64 ? 1 : 0);
        if (h->fb_multi < 0 || h->fb_multi > 2) h->fb_multi = 1;
        // Sequential forward-backward: the reconstruction GEMM leaves 32 SMs to the forward-backward running
        // beside it (measured at config 3: 16 / 24 / 32 / 40 / 48 / 64
        // reserved SMs -> -5 / -6 / +1.9 / +1.6 / -0.2 / -4.7 %).  NFHMM_OVERLAP=n overrides (0 = off).
        const char *eo = getenv("NFHMM_OVERLAP");
        // (with the multi-chain forward-backward, round 2: 0 / 20 / 24 / 32 / 40 SMs -> 72.8 / 78.8 / 82.6 /
        // 81.8 / 79.9 M frame-iterations/s; the one-chain kernel keeps 32)
        // (any batch size with the sequential recursion, round 2: at 32 mixtures -- the per-GPU share of
        // config 3 on 8 GPUs, 64,000 frames -- the step is the recursion's latency and the overlap measured
        // 49.5 -> 68.6 M frame-iterations/s; 8 to 24 SMs within 1 %)
        h->overlap_sms = (h->math == NFHMM_MATH_TC && h->fb_nchunk == 0) ? ((h->fb_multi == 2 && fb_mma_supported(h->N, h->M, 0)) ? 16 : (h->fb_multi && fb_multi_supported(h->N, h->M, 0)) ? 24 : 32) : 0;
        // few chains (parallel-in-time forward-backward, single mixtures): the three phases of the
        // recursion run beside (a) and (b) as well (their persistent grids keep 148 - 32 CTAs)
        if (h->math == NFHMM_MATH_TC && h->fb_nchunk > 0) h->overlap_sms = 32;
        if (eo) h->overlap_sms = h->math == NFHMM_MATH_TC ? atoi(eo) : 0;
        if (h->overlap_sms < 0 || h->overlap_sms > 96) h->overlap_sms = 0;
        const char *ed2 = getenv("NFHMM_DEFER");   // 0: the next sweep's (b) waits for the recursion
        h->defer = h->overlap_sms > 0 && !h->fused && !(ed2 && atoi(ed2) == 0);
        // with the deferred (b) the multi-chain recursion hides behind (a) + (b): 16 SMs suffice (measured at
        // config 3: 12 / 16 / 24 / 32 SMs -> 80.7 / 87.9 / 85.7 / 83.2 M; 24 without the deferral: 87.3 M)
        if (!eo && h->defer && h->fb_nchunk == 0 && h->overlap_sms == 24) h->overlap_sms = 16;
        const char *ef = getenv("NFHMM_FB_FIRST");
        h->fb_first = ef ? atoi(ef) != 0 : h->fb_nchunk > 0;
    }
    {   // split-K for few row tiles: measured per k-block step ~0.6 us whatever the tile width, so
        // single-mixture contractions (8-16 row tiles, 50-75 k-blocks per CTA) are latency-bound; units of
        // one accumulation chunk cut the k-blocks per CTA 3-5x.  NFHMM_SPLITK=0 / 1 forces it off / on.
        const char *e = getenv("NFHMM_SPLITK");
        const int64_t mt = (frames + 127) / 128;
        // Measured (round 2, ms per 100 sweeps, split / unsplit): config 1 reconstruction 2.93 / 3.47,
        // back-projection 2.77 / 2.51; config 2 4.41 / 4.60 and 4.66 / 2.72 -- the back-projection's
        // contraction (F_pad = 520: chunks of 16, 16 and 1 k-blocks) splits unevenly and its unsplit narrow
        // tiles already fill the SMs, so only the reconstruction (Kt = 800 / 1200) is split.
        const bool want = h->math == NFHMM_MATH_TC && !h->fused && mt <= 16 && tc_split_count(Kt) >= 3;
        h->split = e ? (atoi(e) != 0 && h->math == NFHMM_MATH_TC && !h->fused) : want;
        if (h->split) h->bn_tc_a = tc_pick_bn_split(F, frames, tc_split_count(Kt));
    }
    h->nt_tc_a = (int)((F + h->bn_tc_a - 1) / h->bn_tc_a);
    {   // 3xFP16 reconstruction (tensor-core engine): NFHMM_RECON=tf32 selects the 3xTF32 products
        const char *e = getenv("NFHMM_RECON");
        h->h16 = h->math == NFHMM_MATH_TC && !(e && strcmp(e, "tf32") == 0);
        const char *eb = getenv("NFHMM_BACKPROJ");   // tf32: the 3xTF32 back-projection (on R')
        h->h16b = h->h16 && !h->fused && !(eb && strcmp(eb, "tf32") == 0);
    }
    // c_prior = lnGamma(Kt + gamma S K) - S K lnGamma(1 + gamma)  (Eq. 1 normaliser, DESIGN R8)
    h->c_prior_T = (double)T * (lgamma((double)Kt + o.gamma * S * K) - (double)S * K * lgamma(1.0 + o.gamma));
    // no CUDA call here: dims/layout/workspace queries work without a device; the first call that
    // touches the device (set_workspace) selects it.
    *out = h;
    return NFHMM_OK;
}

int nfhmm_workspace_size(const nfhmm_t *h, size_t *bytes) {
    if (!h || !bytes) return NFHMM_EINVAL;
    *bytes = ws_need(h);
    return NFHMM_OK;
}

int nfhmm_set_workspace(nfhmm_t *h, void *dptr, size_t bytes) {
    int r = enter(h);
    if (r) return r;
    if (!h->num_sms) CU(h, cudaDeviceGetAttribute(&h->num_sms, cudaDevAttrMultiProcessorCount, h->device));
    const size_t need = ws_need(h);
    if (h->ws_owned && h->ws) {
        cudaFree(h->ws);
        h->ws = nullptr;
        h->ws_owned = false;
    }
    if (!dptr) {
        CU(h, cudaMalloc(&h->ws, need));
        h->ws_owned = true;
        h->ws_bytes = need;
    } else {
        if (bytes < need) return fail(h, NFHMM_ENOMEM, "workspace %zu < required %zu bytes", bytes, need);
        if (((uintptr_t)dptr & 255) != 0) return fail(h, NFHMM_EINVAL, "workspace must be 256-byte aligned");
        if (!is_device_ptr(dptr)) return fail(h, NFHMM_EINVAL, "workspace must be device memory");
        h->ws = dptr;
        h->ws_bytes = bytes;
    }
    carve(h, (char *)h->ws);
    drop_graphs(h);   // the captured sweeps hold workspace pointers
    // zero everything once: all padding (bins >= F, elements >= Kt) stays zero for the handle's life
    CU(h, cudaMemsetAsync(h->ws, 0, need, h->st));
    for (const auto &z : h->zones)
        CU(h, cudaMemsetAsync((char *)h->ws + z.off, kGuardByte, z.len, h->st));
    h->have_model = h->have_obs = h->R_valid = h->n_ready = false;
    h->iters_done = 0;
    return NFHMM_OK;
}

int nfhmm_set_model(nfhmm_t *h, const float *dict, const float *trans, const float *prior) {
    int r = enter(h);
    if (r) return r;
    if (!h->ws) return fail(h, NFHMM_ESTATE, "set_workspace must precede set_model");
    if (!dict || !trans || !prior) return fail(h, NFHMM_EINVAL, "NULL model array");
    const size_t nd = (size_t)h->Kt * h->F, nt = (size_t)h->S * h->N * h->N, np = (size_t)h->S * h->N;
    std::vector<float> hd(nd), ht(nt), hp(np);
    CU(h, cudaMemcpy(hd.data(), dict, nd * 4, cudaMemcpyDefault));
    CU(h, cudaMemcpy(ht.data(), trans, nt * 4, cudaMemcpyDefault));
    CU(h, cudaMemcpy(hp.data(), prior, np * 4, cudaMemcpyDefault));
    for (int k = 0; k < h->Kt; ++k) {
        double s = 0.0;
        for (int64_t l = 0; l < h->F; ++l) {
            const float v = hd[(size_t)k * h->F + l];
            if (!(v >= 0.f) || !isfinite(v)) return fail(h, NFHMM_EINVAL, "dictionary element %d has a negative/non-finite entry", k);
            s += v;
        }
        if (fabs(s - 1.0) > 1e-4) return fail(h, NFHMM_EINVAL, "dictionary element %d sums to %.8g, not 1", k, s);
    }
    for (int s = 0; s < h->S; ++s) {
        for (int i = 0; i < h->N; ++i) {
            double acc = 0.0;
            for (int j = 0; j < h->N; ++j) {
                const float v = ht[((size_t)s * h->N + i) * h->N + j];
                if (!(v >= 0.f) || !isfinite(v)) return fail(h, NFHMM_EINVAL, "transition (%d,%d,%d) invalid", s, i, j);
                acc += v;
            }
            if (fabs(acc - 1.0) > 1e-4) return fail(h, NFHMM_EINVAL, "transition row (%d,%d) sums to %.8g", s, i, acc);
        }
        double acc = 0.0;
        for (int i = 0; i < h->N; ++i) {
            const float v = hp[(size_t)s * h->N + i];
            if (!(v >= 0.f) || !isfinite(v)) return fail(h, NFHMM_EINVAL, "prior (%d,%d) invalid", s, i);
            acc += v;
        }
        if (fabs(acc - 1.0) > 1e-4) return fail(h, NFHMM_EINVAL, "prior of source %d sums to %.8g", s, acc);
    }
    // betaT [Kb][Fa] (rows k, padded with zeros), beta [Fa][Kb] its transpose
    CU(h, cudaMemsetAsync(h->betaT, 0, (size_t)h->Kb * h->Fa * 4, h->st));
    CU(h, cudaMemsetAsync(h->beta, 0, (size_t)h->Fa * h->Kb * 4, h->st));
    CU(h, cudaMemcpy2DAsync(h->betaT, (size_t)h->Fa * 4, hd.data(), (size_t)h->F * 4, (size_t)h->F * 4, h->Kt,
                            cudaMemcpyHostToDevice, h->st));
    LAUNCH(h, NFHMM_K_OTHER, launch_transpose(h->betaT, h->Kt, (int)h->F, h->Fa, h->beta, h->Kb, h->st));
    {   // tensor-core operand images of the static dictionary (split once, bulk-copied every stage)
        std::vector<float> bsa(tc_presplit_floats(h->F, h->Kt, h->bn_tc_a));
        std::vector<float> bsb(tc_presplit_floats(h->Kt, h->Fa, h->bn_tc_b));
        tc_presplit_host(hd.data(), h->F, /*transposed=*/true, h->F, h->Kt, h->bn_tc_a, bsa.data());    // B[n=l][k]
        std::vector<float> kinv;   // H16: 1 / c_l per bin (R' = c_l R, so the back-projection contracts beta / c_l)
        if (h->h16) {
            std::vector<float> b16(tc_presplit16_floats(h->F, h->Kt, h->bn_tc_a));
            std::vector<float> cs((size_t)h->nt_tc_a * h->bn_tc_a);
            tc_presplit16_host(hd.data(), h->F, /*transposed=*/true, h->F, h->Kt, h->bn_tc_a, b16.data(), cs.data());
            kinv.resize((size_t)h->F);
            for (int64_t l = 0; l < h->F; ++l) kinv[l] = ldexpf(1.f, -30) / cs[l];   // exact (powers of two)
            CU(h, cudaMemcpyAsync(h->bs_a16, b16.data(), b16.size() * 4, cudaMemcpyHostToDevice, h->st));
            CU(h, cudaMemcpyAsync(h->csa, cs.data(), cs.size() * 4, cudaMemcpyHostToDevice, h->st));
            CU(h, cudaStreamSynchronize(h->st));
        }
        if (h->h16b) {
            std::vector<float> b16(tc_presplit16_floats(h->Kt, h->Fa, h->bn_tc_b));
            std::vector<float> cs((size_t)h->nt_tc_b * h->bn_tc_b);
            tc_presplit16_host(hd.data(), h->F, /*transposed=*/false, h->Kt, h->F, h->bn_tc_b, b16.data(), cs.data(), h->Fa,
                               kinv.data());
            CU(h, cudaMemcpyAsync(h->bs_b16, b16.data(), b16.size() * 4, cudaMemcpyHostToDevice, h->st));
            CU(h, cudaMemcpyAsync(h->csb, cs.data(), cs.size() * 4, cudaMemcpyHostToDevice, h->st));
            CU(h, cudaStreamSynchronize(h->st));
        }
        // B[n=k][l]: bins l < F, chunks laid out for the padded contraction Fa the kernel walks
        tc_presplit_host(hd.data(), h->F, /*transposed=*/false, h->Kt, h->F, h->bn_tc_b, bsb.data(), h->Fa,
                         h->h16 ? kinv.data() : nullptr);
        CU(h, cudaMemcpyAsync(h->bs_a, bsa.data(), bsa.size() * 4, cudaMemcpyHostToDevice, h->st));
        CU(h, cudaMemcpyAsync(h->bs_b, bsb.data(), bsb.size() * 4, cudaMemcpyHostToDevice, h->st));
        CU(h, cudaStreamSynchronize(h->st));
    }
    CU(h, cudaMemcpyAsync(h->trans, ht.data(), nt * 4, cudaMemcpyHostToDevice, h->st));
    CU(h, cudaMemcpyAsync(h->prior, hp.data(), np * 4, cudaMemcpyHostToDevice, h->st));
    CU(h, cudaStreamSynchronize(h->st));   // host vectors go out of scope
    h->have_model = true;
    h->R_valid = h->n_ready = false;
    return NFHMM_OK;
}

int nfhmm_reset(nfhmm_t *h) {
    int r = enter(h);
    if (r) return r;
    if (!h->have_model || !h->have_obs) return fail(h, NFHMM_ESTATE, "set_model and set_observations must precede reset");
    // DESIGN R5: alpha = 1 + gamma/N, d = 1/N, theta~ uniform (init_state_kernel)
    const double a0 = 1.0 + h->gamma / h->N;
    LAUNCH(h, NFHMM_K_OTHER, launch_init_state((int)h->frames, h->Kb, h->Kt, a0, h->alpha, h->theta, h->fwd, h->bwd,
                                (long long)h->M * h->S * h->T * h->N, h->st));
    CU(h, cudaMemsetAsync(h->fe, 0, (size_t)h->M * h->max_iters * 8, h->st));
    CU(h, cudaMemsetAsync(h->flags + 1, 0, 2 * sizeof(unsigned), h->st));   // sweep counter, ELBO block count
    CU(h, cudaMemsetAsync(h->elbo_ctr, 0, (size_t)h->M * sizeof(unsigned), h->st));
    h->R_valid = false;
    h->n_ready = false;
    r = recon_ratio(h);
    if (r) return r;
    h->R_valid = true;
    h->iters_done = 0;
    return NFHMM_OK;
}

int nfhmm_set_observations(nfhmm_t *h, const float *V) {
    int r = enter(h);
    if (r) return r;
    if (!h->have_model) return fail(h, NFHMM_ESTATE, "set_model must precede set_observations");
    if (!V) return fail(h, NFHMM_EINVAL, "NULL observations");
    CU(h, cudaMemsetAsync(h->flags, 0, sizeof(unsigned), h->st));   // new data: clear sticky flags
    CU(h, cudaMemcpy2DAsync(h->V, (size_t)h->Fa * 4, V, (size_t)h->F * 4, (size_t)h->F * 4, (size_t)h->frames,
                            cudaMemcpyDefault, h->st));
    LAUNCH(h, NFHMM_K_OTHER, launch_obs_stats(h->V, (int)h->frames, (int)h->F, h->Fa, h->vt, h->flags, h->st));
    LAUNCH(h, NFHMM_K_OTHER, launch_frame_consts(h->vt, (int)h->frames, h->Kt, h->gamma, h->S, h->K, h->fconst, h->st));
    h->have_obs = true;
    return nfhmm_reset(h);
}

int nfhmm_vb_iterate_async(nfhmm_t *h, int32_t n_iters) {
    int r = enter(h);
    if (r) return r;
    if (n_iters < 0) return fail(h, NFHMM_EINVAL, "n_iters < 0");
    if (!h->have_model || !h->have_obs) return fail(h, NFHMM_ESTATE, "model and observations required");
    int i = 0;
    // eager sweeps: profiling (per-launch events), short calls, and the first sweep of the handle
    const bool use_graphs = h->graphs && !h->prof && h->R_valid;
    // (with the deferred back-projection the graphs start from n_ready: the call's first sweep runs eagerly)
    for (; i < n_iters && (!use_graphs || h->eager_sweeps == 0 || n_iters - i < 2 || (h->defer && !h->n_ready)); ++i) {
        r = sweep(h, i == n_iters - 1);
        if (r) return r;
        h->eager_sweeps++;
    }
    if (i < n_iters) {
        // the remaining sweeps as CUDA-graph replays (launch-bound small problems lose their launch gaps)
        for (int k = 0; k < 2; ++k)
            if (!h->gx[k]) {
                r = capture_sweep(h, k == 1);
                if (r) return r;
            }
        CU(h, cudaEventRecord(h->gev[0], h->st));
        CU(h, cudaStreamWaitEvent(h->gst, h->gev[0], 0));
        for (; i < n_iters; ++i) {
            CU(h, cudaGraphLaunch(h->gx[i == n_iters - 1 ? 1 : 0], h->gst));
            h->launches += h->g_kernels;
            h->iters_done++;
        }
        // the replays end with the call's last sweep, which defers nothing: the next call's first sweep
        // must form n itself (capture_sweep restores the host flag it had before capturing)
        h->n_ready = false;
        CU(h, cudaEventRecord(h->gev[1], h->gst));
        CU(h, cudaStreamWaitEvent(h->st, h->gev[1], 0));
    }
    return NFHMM_OK;
}

int nfhmm_sync(nfhmm_t *h) {
    int r = enter(h);
    if (r) return r;
    return check_flags(h);
}

int nfhmm_vb_iterate(nfhmm_t *h, int32_t n_iters) {
    int r = nfhmm_vb_iterate_async(h, n_iters);
    if (r) return r;
    return check_flags(h);
}

int nfhmm_posteriors(nfhmm_t *h, float *d_hat, float *alpha_hat, float *V_hat, double *free_energy,
                     int32_t *iters_done) {
    int r = enter(h);
    if (r) return r;
    if (!h->have_model || !h->have_obs) return fail(h, NFHMM_ESTATE, "model and observations required");
    const size_t chainTN = (size_t)h->M * h->S * h->T * h->N;
    if (d_hat) {   // the FB keeps its messages u, b: marginals u .* b / sum per (m, s, t) on the way out
        const bool dev = is_device_ptr(d_hat);
        LAUNCH(h, NFHMM_K_OTHER, launch_marginals(h->fwd, h->bwd, dev ? d_hat : h->ec, (long long)h->M * h->S * h->T, h->N, h->st));
        if (!dev) CU(h, cudaMemcpyAsync(d_hat, h->ec, chainTN * 4, cudaMemcpyDeviceToHost, h->st));
    }
    if (alpha_hat)
        CU(h, cudaMemcpy2DAsync(alpha_hat, (size_t)h->Kt * 4, h->alpha, (size_t)h->Kb * 4, (size_t)h->Kt * 4,
                                (size_t)h->frames, cudaMemcpyDefault, h->st));
    if (V_hat) {
        const bool dev = is_device_ptr(V_hat);
        ReconArgs a{};
        a.M = (int)h->frames;
        a.k_begin = 0;
        a.k_end = h->Kt;
        a.A = h->theta;
        a.lda = h->Kb;
        a.B = h->betaT;
        a.ldb = h->Fa;
        a.F = (int)h->F;
        a.Vhat = dev ? V_hat : h->vsrc;
        a.flags = h->flags;
        r = run_recon(h, NFHMM_K_OTHER, a);
        if (r) return r;
        if (!dev) CU(h, cudaMemcpyAsync(V_hat, h->vsrc, (size_t)h->frames * h->F * 4, cudaMemcpyDeviceToHost, h->st));
    }
    if (free_energy)
        CU(h, cudaMemcpyAsync(free_energy, h->fe, (size_t)h->M * h->max_iters * 8, cudaMemcpyDefault, h->st));
    if (iters_done) *iters_done = h->iters_done;
    return check_flags(h);
}

int nfhmm_separate(nfhmm_t *h, float *V_star, float *V_src) {
    int r = nfhmm_separate_async(h, V_star, V_src);
    if (r) return r;
    return check_flags(h);
}

int nfhmm_separate_async(nfhmm_t *h, float *V_star, float *V_src) {
    int r = enter(h);
    if (r) return r;
    if (!h->have_model || !h->have_obs) return fail(h, NFHMM_ESTATE, "model and observations required");
    if (!V_star) return fail(h, NFHMM_EINVAL, "V_star is required");
    LAUNCH(h, NFHMM_K_SEPARATE, launch_sep_scale(h->alpha, (int)h->frames, h->Kt, h->Kb, h->vt, h->scale, h->st));
    const int NK = h->N * h->K;
    for (int s = 0; s < h->S; ++s) {
        ReconArgs a{};
        a.M = (int)h->frames;
        a.k_begin = s * NK;
        a.k_end = (s + 1) * NK;
        a.A = h->alpha;
        a.lda = h->Kb;
        a.B = h->betaT;
        a.ldb = h->Fa;
        a.F = (int)h->F;
        a.n_tiles = h->nt_a;
        a.row_scale = h->scale;
        a.out_src = h->vsrc;
        a.T = (int)h->T;
        a.S = h->S;
        a.s = s;
        a.flags = h->flags;
        r = run_recon(h, NFHMM_K_SEPARATE, a);
        if (r) return r;
    }
    const size_t n = (size_t)h->M * h->S * h->T * h->F;
    if (V_src) CU(h, cudaMemcpyAsync(V_src, h->vsrc, n * 4, cudaMemcpyDefault, h->st));
    const bool dev = is_device_ptr(V_star);
    LAUNCH(h, NFHMM_K_SEPARATE, launch_wiener(h->V, h->Fa, h->vsrc, dev ? V_star : h->vsrc, (int)h->M, h->S, (int)h->T, (int)h->F, h->st));
    if (!dev) CU(h, cudaMemcpyAsync(V_star, h->vsrc, n * 4, cudaMemcpyDeviceToHost, h->st));
    return NFHMM_OK;
}

int nfhmm_profile_enable(nfhmm_t *h, int on) {
    int r = enter(h);
    if (r) return r;
    CU(h, cudaStreamSynchronize(h->st));
    h->recs.clear();
    h->pool_used = 0;
    h->prof = on != 0;
    return NFHMM_OK;
}

int nfhmm_profile_read(nfhmm_t *h, double *ms, int64_t *launches) {
    int r = enter(h);
    if (r) return r;
    CU(h, cudaStreamSynchronize(h->st));
    double acc[NFHMM_NUM_KERNEL_CLASSES] = {0};
    int64_t cnt[NFHMM_NUM_KERNEL_CLASSES] = {0};
    for (const auto &rec : h->recs) {
        float t = 0.f;
        CU(h, cudaEventElapsedTime(&t, rec.a, rec.b));
        acc[rec.cls] += t;
        cnt[rec.cls] += 1;
    }
    for (int i = 0; i < NFHMM_NUM_KERNEL_CLASSES; ++i) {
        if (ms) ms[i] = acc[i];
        if (launches) launches[i] = cnt[i];
    }
    return NFHMM_OK;
}

int nfhmm_bench_kernel(nfhmm_t *h, int cls, int32_t reps, double *ms_per_launch) {
    int r = enter(h);
    if (r) return r;
    if (!h->have_model || !h->have_obs) return fail(h, NFHMM_ESTATE, "model and observations required");
    if (reps < 1 || !ms_per_launch) return fail(h, NFHMM_EINVAL, "reps >= 1 and ms_per_launch required");
    if (cls < NFHMM_K_RECON || cls > NFHMM_K_FB) return fail(h, NFHMM_EINVAL, "cls must be RECON..FB");
    cudaEvent_t a = prof_event(h), b = prof_event(h);
    if (!a || !b) return fail(h, NFHMM_ECUDA, "event creation failed");
    const bool prof = h->prof;
    h->prof = false;
    CU(h, cudaEventRecord(a, h->st));
    for (int i = 0; i < reps && !r; ++i) {
        switch (cls) {
            case NFHMM_K_RECON: r = recon_ratio(h); break;
            case NFHMM_K_BACKPROJ: r = step_backproj(h); break;
            case NFHMM_K_DIRICHLET:
                if (h->fused) {
                    r = step_dv(h);
                    if (!r) r = step_eq8(h);
                } else {
                    r = step_dirichlet(h, true);
                }
                break;
            default: r = step_fb(h); break;
        }
    }
    CU(h, cudaEventRecord(b, h->st));
    h->prof = prof;
    if (r) return r;
    CU(h, cudaEventSynchronize(b));
    float t = 0.f;
    CU(h, cudaEventElapsedTime(&t, a, b));
    *ms_per_launch = (double)t / reps;
    // the repeated step left the state inconsistent: force a reset before the next sweep
    h->R_valid = false;
    h->iters_done = 0;
    CU(h, cudaMemsetAsync(h->flags, 0, sizeof(unsigned), h->st));
    return nfhmm_reset(h);
}

int nfhmm_destroy(nfhmm_t *h) {
    if (!h) return NFHMM_OK;
    cudaSetDevice(h->device);
    for (cudaEvent_t e : h->pool) cudaEventDestroy(e);
    drop_graphs(h);
    for (cudaEvent_t e : h->gev)
        if (e) cudaEventDestroy(e);
    if (h->gst) cudaStreamDestroy(h->gst);
    for (cudaEvent_t e : h->fev)
        if (e) cudaEventDestroy(e);
    if (h->fbst) cudaStreamDestroy(h->fbst);
    if (h->pst) cudaStreamDestroy(h->pst);
    if (h->pev) cudaEventDestroy(h->pev);
    if (h->ws_owned && h->ws) cudaFree(h->ws);
    delete h;
    return NFHMM_OK;
}

const char *nfhmm_strerror(int s) {
    switch (s) {
        case NFHMM_OK: return "ok";
        case NFHMM_EINVAL: return "invalid argument";
        case NFHMM_ESTATE: return "call order violated";
        case NFHMM_ECUDA: return "CUDA error";
        case NFHMM_ENOMEM: return "out of memory / workspace too small";
        case NFHMM_EZEROSUPPORT: return "zero support: V > 0 where V_hat = 0";
        case NFHMM_ENUMERIC: return "non-finite value in alpha, phi or log Z";
        default: return "unknown status";
    }
}

const char *nfhmm_last_error(const nfhmm_t *h) { return h ? h->err.c_str() : ""; }

int nfhmm_kernel_launches(const nfhmm_t *h, int64_t *count) {
    if (!h || !count) return NFHMM_EINVAL;
    *count = h->launches;
    return NFHMM_OK;
}

int nfhmm_products(const nfhmm_t *h, int32_t *recon, int32_t *backproj) {
    if (!h) return NFHMM_EINVAL;
    const bool tc = h->math == NFHMM_MATH_TC;
    if (recon) *recon = !tc ? NFHMM_PRODUCTS_FFMA : h->h16 ? NFHMM_PRODUCTS_3XFP16 : NFHMM_PRODUCTS_3XTF32;
    if (backproj) *backproj = !tc ? NFHMM_PRODUCTS_FFMA : h->h16b ? NFHMM_PRODUCTS_3XFP16 : NFHMM_PRODUCTS_3XTF32;
    return NFHMM_OK;
}

int nfhmm_guard_check(nfhmm_t *h, int64_t *checked_bytes, int64_t *bad_bytes) {
    int r = enter(h);
    if (r) return r;
    if (!checked_bytes || !bad_bytes) return fail(h, NFHMM_EINVAL, "null output pointer");
    *checked_bytes = *bad_bytes = 0;
    if (!h->ws) return fail(h, NFHMM_ESTATE, "no workspace");
    CU(h, cudaStreamSynchronize(h->st));
    if (h->fbst) CU(h, cudaStreamSynchronize(h->fbst));
    if (h->pst) CU(h, cudaStreamSynchronize(h->pst));
    if (h->gst) CU(h, cudaStreamSynchronize(h->gst));
    std::vector<unsigned char> buf;
    int first = -2;
    for (const auto &z : h->zones) {
        buf.resize(z.len);
        CU(h, cudaMemcpy(buf.data(), (const char *)h->ws + z.off, z.len, cudaMemcpyDeviceToHost));
        int64_t bad = 0;
        for (unsigned char c : buf) bad += c != (unsigned char)kGuardByte;
        if (bad && first == -2) first = z.piece;
        *checked_bytes += (int64_t)z.len;
        *bad_bytes += bad;
    }
    if (*bad_bytes) return fail(h, NFHMM_ECUDA, "%lld guard bytes overwritten (first after workspace piece %d)",
                                (long long)*bad_bytes, first);
    return NFHMM_OK;
}

int nfhmm_layout(const nfhmm_t *h, int64_t *F_pad, int64_t *Kt_pad, int32_t *bn_recon, int32_t *bn_backproj) {
    if (!h) return NFHMM_EINVAL;
    if (F_pad) *F_pad = h->Fa;
    if (Kt_pad) *Kt_pad = h->Kb;
    if (bn_recon) *bn_recon = h->bn_a;
    if (bn_backproj) *bn_backproj = h->bn_b;
    return NFHMM_OK;
}

}  // extern "C"
