// fic_api.cu -- the C ABI of include/fic.h: contexts, pools, the per-level driver and the
// quadtree loop (§2 line 40).
#include <cuda_runtime.h>
#include <quadmath.h>

#include <cmath>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include <nccl.h>

#include "fic_internal.cuh"

using fic::Buf;
using fic::Pool;

struct fic_pool {
    Pool P;
};

struct fic_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    int num_sms = 148;
    std::string err;
    int timing = 0;
    int64_t lut[4097];
    int64_t *d_delta = nullptr;  // delta[t] = lut[t+1] - lut[t], t < 4096
    Pool levels[fic::kMaxLevels];
    Buf b_blocksum, b_counts, b_rng[2], b_rec, b_acc, b_child, b_part, b_t2f, b_img, b_out,
        b_scounts;
    unsigned long long *h_counts = nullptr;  // pinned [64]
    std::vector<fic_level_stats> stats;
    cudaEvent_t ev[fic::kMaxLevels][5] = {};  // pool start, search start, search end, finalize end, pool end
    int64_t launches = 0;                      // libfic kernels enqueued (fic_level_stats.kernel_launches)
    cudaStream_t side = nullptr;                 // pool builds of levels >= 1 overlap the searches
    cudaStream_t crit = nullptr;                 // the encode's critical path (highest priority)
    bool child_clean = false;                    // b_child is all zero (see encode_body)
    cudaEvent_t fork_ev = nullptr, join_ev = nullptr;
    int overlap_pools = 1;                       // env FIC_OVERLAP_POOLS=0: every pool on the main stream
    cudaEvent_t pool_ready[fic::kMaxLevels] = {};
    cudaEvent_t level_done[fic::kMaxLevels] = {};  // finalize of level l done (records ready)
    Buf b_blocksum2;  // compaction scratch of the side-stream record gathering
    Buf b_code;       // FIC1 writer scratch (fic_serialize)
    cudaEvent_t main_ready = nullptr;
    Buf b_d2;                       // the decimated image, shared by the levels' pools (fic_encode)
    cudaEvent_t d2_ready = nullptr;
    cudaEvent_t top_ready = nullptr;  // the top-level range list, selected on the side stream
    int b2_window = 1;    // env FIC_B2_WINDOW=0: B = 2 full scan instead of the C windows
    int top_side = 1;     // env FIC_TOP_SIDE=0: top-level range selection on the critical stream
    int counts_kernel = 1;  // env FIC_COUNTS_KERNEL=0: the counters by cudaMemcpyAsync (A/B)
    Buf b_u, b_gthr, b_rop, b_dec, b_nccl;
    ncclComm_t comm = nullptr;  // fic_ctx_create_nccl: one rank per GPU
    int32_t nranks = 1, rank = 0;
};

namespace fic {
bool pdl_enabled() {
    static const bool on = [] {
        const char *v = getenv("FIC_PDL");
        return !(v && strcmp(v, "0") == 0);
    }();
    return on;
}
}  // namespace fic

namespace {

// ---------------------------------------------------------------------------- host helpers
fic_status cuda_fail(fic_ctx *ctx, cudaError_t e, const char *what, int line) {
    if (ctx) {
        char buf[512];
        snprintf(buf, sizeof buf, "CUDA error %d (%s) at fic_api.cu:%d in %s", (int)e,
                 cudaGetErrorString(e), line, what);
        ctx->err = buf;
    }
    return e == cudaErrorMemoryAllocation ? FIC_ERR_NOMEM : FIC_ERR_CUDA;
}
fic_status fail(fic_ctx *ctx, fic_status st, const std::string &msg) {
    if (ctx) ctx->err = msg;
    return st;
}
#define CK(x)                                                               \
    do {                                                                    \
        cudaError_t e_ = (x);                                               \
        if (e_ != cudaSuccess) return cuda_fail(ctx, e_, #x, __LINE__);     \
    } while (0)
#define CKS(x)                                   \
    do {                                         \
        fic_status s_ = (x);                     \
        if (s_ != FIC_OK) return s_;             \
    } while (0)

cudaError_t grow(fic_ctx *ctx, Buf &b, size_t bytes) {
    if (bytes == 0) bytes = 16;
    if (b.cap >= bytes) return cudaSuccess;
    if (b.p) {
        if (ctx) cudaStreamSynchronize(ctx->stream);
        cudaFree(b.p);
        b.p = nullptr;
        b.cap = 0;
    }
    const size_t nb = bytes + bytes / 4 + 256;
    cudaError_t e = cudaMalloc(&b.p, nb);
    if (e != cudaSuccess) return e;
    b.cap = nb;
    return cudaSuccess;
}
template <class T>
T *ptr(Buf &b) {
    return reinterpret_cast<T *>(b.p);
}

void free_buf(Buf &b) {
    if (b.p) cudaFree(b.p);
    b.p = nullptr;
    b.cap = 0;
}
void free_pool(Pool &P) {
    free_buf(P.b_keys); free_buf(P.b_keep); free_buf(P.b_kept);
    free_buf(P.b_SDf); free_buf(P.b_SD); free_buf(P.b_C); free_buf(P.b_misc);
    free_buf(P.b_Dtc); free_buf(P.b_D2); free_buf(P.b_F2); free_buf(P.b_blocksum); free_buf(P.b_topk); free_buf(P.b_t2f);
}

bool pow2(int32_t v) { return v > 0 && (v & (v - 1)) == 0; }

// round-half-even(c log2(c) 2^32) in binary128, via the natural log (reading R6)
void make_lut(int64_t *lut, int32_t mmax) {
    const __float128 inv_ln2 = 1 / logq((__float128)2);
    for (int32_t c = 0; c <= mmax; ++c) {
        if (c < 2) {
            lut[c] = 0;
            continue;
        }
        const __float128 v = (__float128)c * logq((__float128)c) * inv_ln2 * (__float128)4294967296.0;
        lut[c] = (int64_t)nearbyintq(v);
    }
}

// T = floor(((tau log2(e)) m) 2^32), binary64 left to right (readings R5, R6)
int64_t entropy_threshold(double tau, int32_t m) {
    volatile double t = tau * 1.4426950408889634;
    t = t * (double)m;
    t = t * 4294967296.0;
    return (int64_t)std::floor(t);
}

// ------------------------------------------------------------------------- pool building
// d2_shared: the decimated image of img built once for every level (fic_encode; d2_ready is
// recorded after it), else the pool decimates into its own buffer
fic_status pool_enqueue(fic_ctx *ctx, Pool &P, const uint8_t *img, int32_t N, int32_t B,
                        int32_t L, double tau, int64_t topk, cudaStream_t st,
                        unsigned long long *d_kept_mirror = nullptr, const uint16_t *d2_shared = nullptr,
                        cudaEvent_t d2_ready = nullptr) {
    P.device = ctx->device;
    P.N = N; P.B = B; P.L = L; P.n = B * B;
    P.A = (N - 2 * B) / L + 1;
    P.n_c = (int64_t)P.A * P.A;
    const int64_t tiles_max = (P.n_c + fic::kTileD - 1) / fic::kTileD;
    const int64_t slots = tiles_max * fic::kTileD;
    CK(grow(ctx, P.b_keys, sizeof(int64_t) * P.n_c));
    CK(grow(ctx, P.b_keep, P.n_c + 16));
    CK(grow(ctx, P.b_kept, sizeof(int32_t) * P.n_c));
    P.mode = B == 2 ? 3 : 0;  // B = 2: closed form on CUDA cores (fic_b2.cu); else tcgen05 (fic_tc.cu)
    if (P.mode == 0) CK(grow(ctx, P.b_Dtc, fic::tc_pool_bytes(B, tiles_max)));
    const bool own_d2 = P.mode == 0 && fic::tc_pool_d2_bytes(B, N, L) && !d2_shared;
    if (own_d2) CK(grow(ctx, P.b_D2, fic::tc_pool_d2_bytes(B, N, L)));
    if (P.mode == 3) CK(grow(ctx, P.b_F2, fic::b2_pool_bytes(slots)));
    CK(grow(ctx, P.b_SDf, sizeof(float) * slots));
    CK(grow(ctx, P.b_SD, sizeof(int32_t) * slots));
    CK(grow(ctx, P.b_C, sizeof(int64_t) * slots));
    CK(grow(ctx, P.b_misc, 4 * sizeof(unsigned long long)));
    CK(grow(ctx, P.b_blocksum, sizeof(int64_t) * fic::select_blocksum_len(P.n_c)));
    P.n_tiles_max = tiles_max;
    P.keys = ptr<int64_t>(P.b_keys); P.keep = ptr<uint8_t>(P.b_keep);
    P.kept = ptr<int32_t>(P.b_kept); P.SDf = ptr<float>(P.b_SDf);
    P.Dtc = P.mode == 0 ? ptr<uint8_t>(P.b_Dtc) : nullptr;
    P.SD = ptr<int32_t>(P.b_SD); P.C = ptr<int64_t>(P.b_C);
    P.d_misc = ptr<unsigned long long>(P.b_misc);
    CK(cudaMemsetAsync(P.d_misc, 0, 4 * sizeof(unsigned long long), st));
    const int32_t m = 4 * B * B;
    const int use_tau = tau >= 0.0;
    const int64_t T = use_tau ? entropy_threshold(tau, m) : 0;
    CK(fic::launch_entropy_keys(img, N, B, L, P.A, ctx->d_delta, ctx->lut[m], T, use_tau, P.keys,
                                P.keep, st));
    if (topk > 0) {  // pool size K instead of the threshold (reading R27)
        CK(grow(ctx, P.b_topk, fic::topk_scratch_bytes(P.n_c)));
        CK(fic::launch_topk_select(P.keys, P.n_c, topk, P.b_topk.p, P.keep, st));
        ctx->launches += 2;
    }
    CK(fic::launch_select_index(P.keep, P.n_c, ptr<int64_t>(P.b_blocksum), P.kept, &P.d_misc[0], st,
                                d_kept_mirror));
    if (P.mode == 0) {
        const uint16_t *D2 = nullptr;
        if (own_d2) {
            CK(fic::launch_decimate(img, N, L, ptr<uint16_t>(P.b_D2), st));
            D2 = ptr<uint16_t>(P.b_D2);
        } else if (fic::tc_pool_d2_bytes(B, N, L)) {
            if (d2_ready) CK(cudaStreamWaitEvent(st, d2_ready, 0));
            D2 = d2_shared;
        }
        CK(fic::launch_pool_tc(img, N, B, L, P.A, P.kept, &P.d_misc[0], tiles_max, P.Dtc, P.SD, P.SDf, P.C,
                               &P.d_misc[1], D2, st));
    }
    else
        CK(fic::launch_b2_pool(img, N, L, P.A, P.kept, &P.d_misc[0], slots, P.b_F2.p, &P.b2, P.SD, P.SDf, P.C,
                               &P.d_misc[1], st));
    const bool fused = P.mode == 3 || fic::tc_pool_has_moments(B);
    if (!fused)
        CK(fic::launch_pool_moments(img, N, B, L, P.A, P.kept, &P.d_misc[0], slots, P.SD, P.SDf, P.C,
                                    &P.d_misc[1], st));
    // entropy, select x3, gather, moments (+ the decimated image of the QR pools)
    // (B = 2: + the coarse C index of the sorted pool)
    ctx->launches += 6 + (P.mode == 3 ? 2 : 0) - (fused ? 1 : 0) + (own_d2 ? 1 : 0);
    return FIC_OK;
}

// after a stream sync: copy the pool's counters into the host struct
void pool_take_counts(Pool &P, const unsigned long long *h) {
    P.n_k = (int64_t)h[0];
    P.cmax = (int64_t)h[1];
    {
        const unsigned int bits = (unsigned int)(h[2] & 0xffffffffu);
        float f;
        memcpy(&f, &bits, 4);
        P.dnmax = (double)f;
    }
    P.n_tiles = (P.n_k + fic::kTileD - 1) / fic::kTileD;
}

fic_status check_level(fic_ctx *ctx, int32_t N, int32_t B, int32_t L) {
    if (!pow2(B) || B < 2) return fail(ctx, FIC_ERR_ARG, "B must be a power of two >= 2");
    if (B > 32) return fail(ctx, FIC_ERR_ARG, "B must be <= 32");
    if (L < 1) return fail(ctx, FIC_ERR_ARG, "L must be >= 1");
    if (N < 1 || 2 * B > N) return fail(ctx, FIC_ERR_SHAPE, "2B > N: no domain block fits");
    return FIC_OK;
}

fic_status check_s(fic_ctx *ctx, const double *h_s, int32_t n_s) {
    if (!h_s || n_s < 1 || n_s > fic::kMaxS)
        return fail(ctx, FIC_ERR_ARG, "need 1 <= n_s <= 32 contrast values");
    for (int j = 0; j < n_s; ++j)
        if (!(h_s[j] >= 0.0 && h_s[j] <= 1.0))
            return fail(ctx, FIC_ERR_ARG, "contrast values s must lie in [0,1]");
    return FIC_OK;
}

// --------------------------------------------------------------------------- one level
// ranges: device int2 [n_r]; the range count is *d_nr (device), n_r_max a host upper bound that
// sizes grids and buffers.  Writes rec [n_r], acc [n_r_max] (0 past n_r) and child marks.
// The level's fp32 filter table (t2f_kernel) from the pool's C and the level's s set, enqueued on
// the pool's stream right after the pool (off the quadtree's critical path); tcgen05 / direct only.
fic_status t2f_enqueue(fic_ctx *ctx, Pool &P, const double *h_s, int32_t n_s, cudaStream_t st) {
    P.t2f_ready = 0;
    if (P.mode != 0) return FIC_OK;
    fic::SList sl;
    memset(&sl, 0, sizeof sl);
    int nsp = 0;
    for (int j = 0; j < n_s; ++j)
        if (h_s[j] != 0.0) sl.s[nsp++] = h_s[j];
    const int64_t slots = P.n_tiles_max * fic::kTileD;
    const fic::SGrid grid = fic::detect_sgrid(sl.s, nsp);
    CK(grow(ctx, P.b_t2f, sizeof(float) * (size_t)slots * (nsp ? nsp : 1)));
    CK(fic::launch_t2f(P.C, &P.d_misc[0], slots, sl, nsp, reinterpret_cast<float *>(P.b_t2f.p),
                       nsp > 2 ? (grid.on ? 2 : 1) : 0, fic::tc_t2_fold(P.B, nsp), st, grid.h));
    if (nsp > 0 && slots > 0) ctx->launches += 1;
    P.t2f_ready = 1;
    return FIC_OK;
}

fic_status level_enqueue(fic_ctx *ctx, const Pool &P, const uint8_t *img, const int2 *ranges,
                         const unsigned long long *d_nr, int64_t n_r_max, const double *h_s, int32_t n_s,
                         double rms_tol, int is_min, fic_record *rec, uint8_t *acc, uint8_t *child,
                         int level_slot, int32_t *d_err, fic_record *out_direct = nullptr,
                         const unsigned long long *d_base = nullptr, int64_t capacity = 0,
                         unsigned long long *d_level_count = nullptr, cudaEvent_t before_finalize = nullptr,
                         int prep_done = 0) {
    cudaStream_t st = ctx->stream;
    if (n_r_max == 0) return FIC_OK;
    fic::SearchParams sp;
    memset(&sp, 0, sizeof sp);
    sp.img = img;
    sp.N = P.N;
    sp.ranges = ranges;
    sp.n_r = (int32_t)n_r_max;
    sp.d_nr = d_nr;
    sp.d_misc = P.d_misc;
    sp.SDf = P.SDf; sp.SD = P.SD; sp.C = P.C;
    const int64_t tiles = P.n_tiles_max;
    sp.n_k = (int32_t)(tiles * fic::kTileD);
    sp.n_tiles = (int32_t)tiles;
    const int64_t slots = tiles * fic::kTileD;
    sp.slot_stride = slots;
    sp.has_zero = 0;
    sp.j_zero = 0;
    sp.smax = 0.0;
    for (int j = 0; j < n_s; ++j) {
        if (h_s[j] == 0.0) {
            if (!sp.has_zero) { sp.has_zero = 1; sp.j_zero = j; }
        } else {
            sp.spos[sp.nsp] = h_s[j];
            sp.jpos[sp.nsp] = j;
            ++sp.nsp;
        }
        if (h_s[j] > sp.smax) sp.smax = h_s[j];
    }
    sp.prep_done = prep_done;
    if (P.mode == 0)
        sp.nsplit = fic::tc_nsplit_hint(P.B, n_r_max, tiles, ctx->num_sms);
    else
        sp.nsplit = fic::b2_nsplit_hint(n_r_max, tiles, ctx->num_sms);
    if (sp.nsplit < 1) sp.nsplit = 1;
    sp.tiles_per_split = (int32_t)((tiles + sp.nsplit - 1) / sp.nsplit);
    // both search kernels (tcgen05, B = 2) choose their split count on the device, up to ns_cap
    const bool dyn = true;
    sp.grid = fic::detect_sgrid(sp.spos, sp.nsp);
    sp.b2_window = ctx->b2_window;
    sp.num_sms = ctx->num_sms;
    sp.L = P.L;
    sp.Acnt = P.A;
    sp.kept = P.kept;
    sp.ns_cap = dyn ? (int32_t)std::min<int64_t>(4 * (int64_t)sp.nsplit, std::max<int64_t>(1, tiles)) : sp.nsplit;
    sp.d_ns = ptr<unsigned long long>(ctx->b_counts) + 56 + level_slot;
    if (!dyn) CK(fic::launch_set_u64(sp.d_ns, (unsigned long long)sp.nsplit, st));
    const bool t2f_pre = P.t2f_ready && P.mode == 0;  // enqueued with the pool
    if (!t2f_pre) CK(grow(ctx, ctx->b_t2f, sizeof(float) * (size_t)slots * (sp.nsp ? sp.nsp : 1)));
    CK(grow(ctx, ctx->b_part, sizeof(fic::Partial) * (size_t)n_r_max * sp.ns_cap));
    sp.t2f = t2f_pre ? reinterpret_cast<float *>(P.b_t2f.p) : ptr<float>(ctx->b_t2f);
    sp.part = ptr<fic::Partial>(ctx->b_part);
    sp.exact_count = ptr<unsigned long long>(ctx->b_counts) + 8 + level_slot;
    fic::SList sl;
    memcpy(sl.s, sp.spos, sizeof sl.s);
    if (P.mode == 0) {
        if (!t2f_pre) {
            CK(fic::launch_t2f(P.C, &P.d_misc[0], slots, sl, sp.nsp, ptr<float>(ctx->b_t2f),
                               sp.nsp > 2 ? (sp.grid.on ? 2 : 1) : 0, fic::tc_t2_fold(P.B, sp.nsp), st, sp.grid.h));
            if (sp.nsp > 0 && slots > 0) ctx->launches += 1;
        }
        if (ctx->timing) CK(cudaEventRecord(ctx->ev[level_slot][1], st));
        if (sp.nsp > 0) {
            CK(grow(ctx, ctx->b_rop, fic::tc_range_bytes(P.B, n_r_max)));
            CK(fic::launch_tc_search(P.B, sp, P.Dtc, slots, ptr<uint8_t>(ctx->b_rop), st));
            ctx->launches += 2;  // range preparation (operand + moments, one launch) + search
        }
    } else {
        CK(grow(ctx, ctx->b_u, sizeof(float) * (size_t)slots * fic::b2_t2_width(sp.nsp)));
        if (ctx->timing) CK(cudaEventRecord(ctx->ev[level_slot][1], st));
        CK(grow(ctx, ctx->b_gthr, fic::b2_scratch_bytes(n_r_max, sp.ns_cap)));
        CK(fic::launch_b2_search(sp, P.b2, ptr<float>(ctx->b_u), P.kept, P.L, P.A, ctx->b_gthr.p,
                                 ptr<unsigned long long>(ctx->b_counts) + 40 + level_slot, st));
        // t2 table, pass 1 scan, pass 2 exact -- or the single window kernel
        const bool win = (sp.b2_window && !sp.has_zero && sp.nsp <= 2) || fic::b2_wink_applies(sp);
        ctx->launches += sp.nsp > 0 && n_r_max > 0 ? (win ? 1 : 3) : 0;
    }
    if (ctx->timing) CK(cudaEventRecord(ctx->ev[level_slot][2], st));
    fic::FinalizeParams fp;
    memset(&fp, 0, sizeof fp);
    fp.img = img; fp.N = P.N; fp.B = P.B; fp.L = P.L; fp.A = P.A;
    fp.ranges = ranges;
    fp.n_r = (int32_t)n_r_max;
    fp.d_nr = d_nr;
    fp.d_misc = P.d_misc;
    fp.d_err = d_err;
    fp.nsplit = sp.nsp > 0 ? sp.ns_cap : 0;
    fp.d_ns = sp.d_ns;
    fp.part = sp.part;
    fp.SD = P.SD; fp.kept = P.kept;
    for (int j = 0; j < n_s; ++j) fp.s[j] = h_s[j];
    fp.n_s = n_s; fp.has_zero = sp.has_zero; fp.j_zero = sp.j_zero;
    fp.fix_kj = 0;
    for (int j = 0; j < n_s; ++j)
        if (h_s[j] > 0.0 && h_s[j] < fic::kSLicensed) fp.fix_kj = 1;
    fp.rms_tol = rms_tol; fp.is_min = is_min;
    fp.rec = rec; fp.accepted = acc; fp.child = child;
    fp.out_direct = out_direct; fp.d_base = d_base; fp.capacity = capacity; fp.d_level_count = d_level_count;
    if (acc && !out_direct) CK(cudaMemsetAsync(acc, 0, (size_t)n_r_max, st));
    if (before_finalize) CK(cudaStreamWaitEvent(st, before_finalize, 0));
    CK(fic::launch_finalize(fp, st));
    ctx->launches += 1;
    if (ctx->timing >= 2) CK(cudaEventRecord(ctx->ev[level_slot][3], st));
    return FIC_OK;
}

fic_status ctx_check(fic_ctx *ctx) {
    if (!ctx) return FIC_ERR_ARG;
    ctx->err.clear();
    CK(cudaSetDevice(ctx->device));
    return FIC_OK;
}

}  // namespace

// =============================================================================== C ABI
extern "C" {

// ------------------------------------------------------------------------- decoding, PSNR
fic_status fic_decode(fic_ctx *ctx, const fic_record *rec, int64_t n_rec, int32_t N, int32_t B_max,
                      int32_t n_levels, const double *h_s, const int32_t *h_n_s, int32_t iterations,
                      const uint8_t *init, uint8_t *out) {
    CKS(ctx_check(ctx));
    if ((!rec && n_rec) || n_rec < 0 || !h_s || !h_n_s || !out || iterations < 0)
        return fail(ctx, FIC_ERR_ARG, "null or negative argument");
    if (N < 1 || !pow2(B_max) || n_levels < 1 || n_levels > fic::kMaxLevels || (B_max >> (n_levels - 1)) < 1)
        return fail(ctx, FIC_ERR_ARG, "bad N, B_max or level count");
    fic::DecSList sl;
    memset(&sl, 0, sizeof sl);
    int32_t off = 0;
    for (int l = 0; l < n_levels; ++l) {
        CKS(check_s(ctx, h_s + off, h_n_s[l]));
        sl.off[l] = off;
        sl.n_s[l] = h_n_s[l];
        for (int j = 0; j < h_n_s[l]; ++j) sl.s[off + j] = h_s[off + j];
        off += h_n_s[l];
    }
    cudaStream_t st = ctx->stream;
    CK(grow(ctx, ctx->b_dec, fic::decode_scratch_bytes(N, n_rec)));
    unsigned long long *d_counts = ptr<unsigned long long>(ctx->b_counts);
    int32_t *d_bad = reinterpret_cast<int32_t *>(d_counts + 62);
    CK(cudaMemsetAsync(d_bad, 0, sizeof(int32_t), st));
    CK(fic::launch_decode(rec, n_rec, N, B_max, n_levels, sl, iterations, init, out, ctx->b_dec.p, d_bad, st));
    int32_t bad = 0;
    CK(cudaMemcpyAsync(&bad, d_bad, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (bad) return fail(ctx, FIC_ERR_ARG, "a record is out of bounds or names an unknown level / s index");
    return FIC_OK;
}

fic_status fic_psnr(fic_ctx *ctx, const uint8_t *a, const uint8_t *b, int64_t n, double *h_psnr) {
    CKS(ctx_check(ctx));
    if (!a || !b || !h_psnr || n < 1) return fail(ctx, FIC_ERR_ARG, "null argument or empty image");
    cudaStream_t st = ctx->stream;
    unsigned long long *d_sse = ptr<unsigned long long>(ctx->b_counts) + 63;
    CK(fic::launch_sse(a, b, n, d_sse, st));
    unsigned long long sse = 0;
    CK(cudaMemcpyAsync(&sse, d_sse, sizeof sse, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    // reading R26: 10 log10(255^2 / MSE), MSE = SSE / n; +inf for identical images
    *h_psnr = sse == 0 ? INFINITY : 10.0 * std::log10(65025.0 / ((double)sse / (double)n));
    return FIC_OK;
}

// ------------------------------------------------------------------------- NCCL (multi-GPU)
fic_status fic_serialize(fic_ctx *ctx, const fic_record *rec, int64_t n_rec, int32_t N, int32_t B_max,
                         int32_t B_min, int32_t L, const int32_t *h_n_s, int32_t s_mode, double s_max,
                         uint8_t *out, int64_t capacity, int64_t *h_nbytes) {
    CKS(ctx_check(ctx));
    if (h_nbytes) *h_nbytes = 0;
    if (!h_n_s || !h_nbytes || (!rec && n_rec > 0) || n_rec < 0 || (!out && capacity > 0) || capacity < 0)
        return fail(ctx, FIC_ERR_ARG, "null argument");
    if (!pow2(B_max) || !pow2(B_min) || B_min < 2 || B_min > B_max || N < 1 || N % B_max || N > 65535 ||
        B_max > 255 || L < 1 || L > 65535 || s_mode < 0 || s_mode > 255 || !(s_max >= 0.0 && s_max <= 6.5535))
        return fail(ctx, FIC_ERR_ARG, "bad code parameters");
    int nl = 0;
    for (int32_t B = B_max; B >= B_min; B /= 2) ++nl;
    if (nl > fic::kMaxLevels) return fail(ctx, FIC_ERR_ARG, "too many levels");
    fic::CodeParams P;
    memset(&P, 0, sizeof P);
    P.N = N; P.B_max = B_max; P.B_min = B_min; P.L = L;
    auto nbits = [](int64_t c) { int b = 0; while ((int64_t{1} << b) < c) ++b; return b; };
    std::vector<uint8_t> head = {'F', 'I', 'C', '1', (uint8_t)(N >> 8), (uint8_t)N, (uint8_t)(N >> 8), (uint8_t)N,
                                 (uint8_t)B_max, (uint8_t)B_min, (uint8_t)s_mode};
    const int sm = (int)std::lround(s_max * 10000.0);
    head.push_back((uint8_t)(sm >> 8)); head.push_back((uint8_t)sm);
    head.push_back((uint8_t)(L >> 8)); head.push_back((uint8_t)L);
    for (int l = 0; l < nl; ++l) {
        const int32_t B = B_max >> l;
        if (h_n_s[l] < 1 || h_n_s[l] > 255) return fail(ctx, FIC_ERR_ARG, "s count out of range");
        head.push_back((uint8_t)h_n_s[l]);
        P.sbits[l] = nbits(h_n_s[l]);
        P.n_s[l] = h_n_s[l];
        P.posbits[l] = N >= 2 * B ? nbits((N - 2 * B) / L + 1) : 0;
    }
    const int64_t hb = (int64_t)head.size();
    cudaStream_t st = ctx->stream;
    // body bound: per leaf <= log2(B_max / B_min) + 1 + 2 * 16 + 3 + 8 + 8 bits
    const int64_t max_words = (n_rec * 64 + 31) / 32 + 2;
    CK(grow(ctx, ctx->b_code, fic::code_scratch_bytes(n_rec) + sizeof(unsigned) * (size_t)max_words + 256));
    unsigned *words = reinterpret_cast<unsigned *>(static_cast<char *>(ctx->b_code.p) + fic::code_scratch_bytes(n_rec));
    unsigned long long *d_total = ptr<unsigned long long>(ctx->b_counts) + 63;
    int32_t *d_bad = reinterpret_cast<int32_t *>(ptr<unsigned long long>(ctx->b_counts) + 62);
    CK(cudaMemsetAsync(words, 0, sizeof(unsigned) * (size_t)max_words, st));
    CK(cudaMemsetAsync(d_bad, 0, sizeof(int32_t), st));
    CK(fic::launch_code_body(rec, n_rec, P, ctx->b_code.p, words, d_total, d_bad, st));
    unsigned long long bits = 0;
    int32_t bad = 0;
    CK(cudaMemcpyAsync(&bits, d_total, sizeof bits, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(&bad, d_bad, sizeof bad, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (bad) return fail(ctx, FIC_ERR_ARG, "a record cannot be coded (out of bounds, unknown level, s index or isometry)");
    const int64_t nbytes = hb + (int64_t)((bits + 7) / 8);
    *h_nbytes = nbytes;
    if (nbytes > capacity) return fail(ctx, FIC_ERR_CAPACITY, "output capacity too small for the stream");
    CK(cudaMemcpyAsync(out, head.data(), (size_t)hb, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(out + hb, words, (size_t)(nbytes - hb), cudaMemcpyDeviceToDevice, st));
    CK(cudaStreamSynchronize(st));
    return FIC_OK;
}

fic_status fic_nccl_unique_id(uint8_t *h_id128) {
    if (!h_id128) return FIC_ERR_ARG;
    static_assert(sizeof(ncclUniqueId) == 128, "NCCL unique id is 128 bytes");
    ncclUniqueId id;
    if (ncclGetUniqueId(&id) != ncclSuccess) return FIC_ERR_NCCL;
    memcpy(h_id128, &id, sizeof id);
    return FIC_OK;
}

fic_status fic_ctx_create_nccl(int32_t device, void *cuda_stream, const uint8_t *h_id128, int32_t nranks,
                               int32_t rank, fic_ctx **out) {
    if (!out || !h_id128 || nranks < 1 || rank < 0 || rank >= nranks) return FIC_ERR_ARG;
    fic_status st = fic_ctx_create(device, cuda_stream, out);
    if (st != FIC_OK) return st;
    fic_ctx *ctx = *out;
    ncclUniqueId id;
    memcpy(&id, h_id128, sizeof id);
    const ncclResult_t r = ncclCommInitRank(&ctx->comm, nranks, id, rank);
    if (r != ncclSuccess) {
        ctx->comm = nullptr;
        fic_ctx_destroy(ctx);
        *out = nullptr;
        return FIC_ERR_NCCL;
    }
    ctx->nranks = nranks;
    ctx->rank = rank;
    return FIC_OK;
}

#define CKN(x)                                                                              \
    do {                                                                                    \
        const ncclResult_t r_ = (x);                                                        \
        if (r_ != ncclSuccess) return fail(ctx, FIC_ERR_NCCL, std::string("NCCL: ") + ncclGetErrorString(r_)); \
    } while (0)

static fic_status encode_impl(fic_ctx *ctx, const uint8_t *img, int32_t N, int32_t B_max, int32_t B_min,
                              int32_t L, const double *h_tau, const int64_t *h_topk, const double *h_s,
                              const int32_t *h_n_s, const double *h_rms_tol, int32_t shard, int32_t n_shards,
                              fic_record *out, int64_t capacity, int64_t *h_n_out);

// Rank r encodes the top-level blocks t % nranks == r (no exchange on the data path), then one
// all-gather of the counts and one of the records (padded to the largest shard) over the
// communicator, and the canonical merge (B desc, ry, rx) on every rank.  A rank whose local encode
// fails still takes part in the count all-gather, sending -status in place of its count, so
// every rank sees the failure and returns the same status (that of the lowest failing rank)
// instead of waiting in a collective the failed rank never reaches.
static fic_status encode_nccl_impl(fic_ctx *ctx, const uint8_t *img, int32_t N, int32_t B_max, int32_t B_min,
                                   int32_t L, const double *h_tau, const int64_t *h_topk, const double *h_s,
                                   const int32_t *h_n_s, const double *h_rms_tol, fic_record *out, int64_t capacity,
                                   int64_t *h_n_out) {
    CKS(ctx_check(ctx));
    if (h_n_out) *h_n_out = 0;
    if (!ctx->comm) return fail(ctx, FIC_ERR_ARG, "context has no NCCL communicator (fic_ctx_create_nccl)");
    if (!h_n_out || (!out && capacity > 0) || capacity < 0) return fail(ctx, FIC_ERR_ARG, "null argument");
    if (B_min < 1 || N < 1) return fail(ctx, FIC_ERR_ARG, "bad sizes");
    const int W = ctx->nranks;
    const int64_t cap_local = (int64_t)(N / B_min) * (N / B_min);
    // layout of b_nccl: local records [cap_local] | gathered [W][cap_local] | counts [W] | my count
    const size_t rec_bytes = sizeof(fic_record) * (size_t)cap_local;
    CK(grow(ctx, ctx->b_nccl, rec_bytes * (size_t)(W + 1) + sizeof(int64_t) * (size_t)(W + 1)));
    char *base = static_cast<char *>(ctx->b_nccl.p);
    fic_record *local = reinterpret_cast<fic_record *>(base);
    fic_record *gathered = reinterpret_cast<fic_record *>(base + rec_bytes);
    int64_t *d_counts = reinterpret_cast<int64_t *>(base + rec_bytes * (size_t)(W + 1));
    int64_t *d_mine = d_counts + W;
    int64_t n_local = 0;
    const fic_status st_local = encode_impl(ctx, img, N, B_max, B_min, L, h_tau, h_topk, h_s, h_n_s, h_rms_tol,
                                            ctx->rank, W, local, cap_local, &n_local);
    const std::string err_local = ctx->err;
    const int64_t mine = st_local == FIC_OK ? n_local : -(int64_t)st_local;
    cudaStream_t st = ctx->stream;
    CK(cudaMemcpyAsync(d_mine, &mine, sizeof(int64_t), cudaMemcpyHostToDevice, st));
    CKN(ncclAllGather(d_mine, d_counts, 1, ncclInt64, ctx->comm, st));
    std::vector<int64_t> counts(W);
    CK(cudaMemcpyAsync(counts.data(), d_counts, sizeof(int64_t) * W, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    for (int i = 0; i < W; ++i)
        if (counts[i] < 0) {
            const fic_status bad = (fic_status)(-counts[i]);
            if (i == ctx->rank) return fail(ctx, bad, err_local);
            return fail(ctx, bad, "rank " + std::to_string(i) + " failed its shard of the encode (status " +
                                      std::to_string((int)bad) + ")");
        }
    int64_t stride = 1, total = 0;
    for (int i = 0; i < W; ++i) {
        stride = std::max(stride, counts[i]);
        total += counts[i];
    }
    // every rank sends `stride` records (entries past its count are not read by the merge)
    CKN(ncclAllGather(local, gathered, sizeof(fic_record) * (size_t)stride, ncclUint8, ctx->comm, st));
    *h_n_out = total;
    if (total > capacity) {
        CK(cudaStreamSynchronize(st));
        return fail(ctx, FIC_ERR_CAPACITY, "output capacity too small");
    }
    // gathered is [W][stride] contiguous: merge with stride `stride`
    CK(fic::launch_merge_shards(gathered, d_counts, W, stride, stride, out, st));
    CK(cudaStreamSynchronize(st));
    return FIC_OK;
}

fic_status fic_encode_nccl(fic_ctx *ctx, const uint8_t *img, int32_t N, int32_t B_max, int32_t B_min, int32_t L,
                           const double *h_tau, const double *h_s, const int32_t *h_n_s, const double *h_rms_tol,
                           fic_record *out, int64_t capacity, int64_t *h_n_out) {
    return encode_nccl_impl(ctx, img, N, B_max, B_min, L, h_tau, nullptr, h_s, h_n_s, h_rms_tol, out, capacity,
                            h_n_out);
}

fic_status fic_encode_nccl_topk(fic_ctx *ctx, const uint8_t *img, int32_t N, int32_t B_max, int32_t B_min,
                                int32_t L, const int64_t *h_K, const double *h_s, const int32_t *h_n_s,
                                const double *h_rms_tol, fic_record *out, int64_t capacity, int64_t *h_n_out) {
    if (!h_K) {
        if (h_n_out) *h_n_out = 0;
        return ctx ? fail(ctx, FIC_ERR_ARG, "null pool sizes") : FIC_ERR_ARG;
    }
    return encode_nccl_impl(ctx, img, N, B_max, B_min, L, nullptr, h_K, h_s, h_n_s, h_rms_tol, out, capacity,
                            h_n_out);
}

const char *fic_version(void) { return "fic-b200 0.1 (sm_100a; fp32-exact CUDA-core search)"; }

fic_status fic_entropy_lut(int64_t *h_lut, int32_t mmax) {
    if (!h_lut || mmax < 0 || mmax > (1 << 20)) return FIC_ERR_ARG;
    make_lut(h_lut, mmax);
    return FIC_OK;
}

fic_status fic_ctx_create(int32_t device, void *cuda_stream, fic_ctx **out) {
    if (!out) return FIC_ERR_ARG;
    *out = nullptr;
    fic_ctx *ctx = new (std::nothrow) fic_ctx();
    if (!ctx) return FIC_ERR_NOMEM;
    ctx->device = device;
    ctx->stream = (cudaStream_t)cuda_stream;
    cudaError_t e = cudaSetDevice(device);
    if (e != cudaSuccess) {
        delete ctx;
        return FIC_ERR_CUDA;
    }
    cudaDeviceGetAttribute(&ctx->num_sms, cudaDevAttrMultiProcessorCount, device);
    make_lut(ctx->lut, 4096);
    std::vector<int64_t> delta(4096);
    for (int t = 0; t < 4096; ++t) delta[t] = ctx->lut[t + 1] - ctx->lut[t];
    e = cudaMalloc(&ctx->d_delta, sizeof(int64_t) * 4096);
    if (e == cudaSuccess)
        e = cudaMemcpy(ctx->d_delta, delta.data(), sizeof(int64_t) * 4096, cudaMemcpyHostToDevice);
    if (e == cudaSuccess)  // (mapped: the counters' kernel writes it, FIC_COUNTS_KERNEL)
        e = cudaHostAlloc(reinterpret_cast<void **>(&ctx->h_counts), 64 * sizeof(unsigned long long),
                          cudaHostAllocPortable | cudaHostAllocMapped);
    if (e == cudaSuccess) e = grow(nullptr, ctx->b_counts, 64 * sizeof(unsigned long long));
    {
        const char *bw = getenv("FIC_B2_WINDOW");
        ctx->b2_window = bw && strcmp(bw, "0") == 0 ? 0 : 1;
        const char *tsd = getenv("FIC_TOP_SIDE");
        ctx->top_side = tsd && strcmp(tsd, "0") == 0 ? 0 : 1;
        const char *ov = getenv("FIC_OVERLAP_POOLS");
        ctx->overlap_pools = ov ? atoi(ov) != 0 : 1;
        const char *ck = getenv("FIC_COUNTS_KERNEL");
        ctx->counts_kernel = ck && strcmp(ck, "0") == 0 ? 0 : 1;
        // the counters' kernel writes the pinned host buffer through UVA (device-accessible)
        int uva = 0;
        if (e == cudaSuccess) e = cudaDeviceGetAttribute(&uva, cudaDevAttrUnifiedAddressing, device);
        if (!uva) ctx->counts_kernel = 0;
    }
    for (int l = 0; l < fic::kMaxLevels && e == cudaSuccess; ++l)
        for (int q = 0; q < 5 && e == cudaSuccess; ++q) e = cudaEventCreate(&ctx->ev[l][q]);
    // the quadtree's critical path runs on a highest-priority stream, the overlapped pool builds
    // and record gathering on a lowest-priority one: when both have blocks waiting, the critical
    // path's small kernels are scheduled first
    int prio_lo = 0, prio_hi = 0;
    if (e == cudaSuccess) e = cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi);
    {
        const char *sp = getenv("FIC_SIDE_PRIO");  // (A/B experiments: "hi" = the critical path's priority)
        if (sp && strcmp(sp, "hi") == 0) prio_lo = prio_hi;
    }
    if (e == cudaSuccess) e = cudaStreamCreateWithPriority(&ctx->side, cudaStreamNonBlocking, prio_lo);
    if (e == cudaSuccess) e = cudaStreamCreateWithPriority(&ctx->crit, cudaStreamNonBlocking, prio_hi);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ctx->fork_ev, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ctx->join_ev, cudaEventDisableTiming);
    for (int l = 0; l < fic::kMaxLevels && e == cudaSuccess; ++l)
        e = cudaEventCreateWithFlags(&ctx->pool_ready[l], cudaEventDisableTiming);
    for (int l = 0; l < fic::kMaxLevels && e == cudaSuccess; ++l)
        e = cudaEventCreateWithFlags(&ctx->level_done[l], cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ctx->main_ready, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ctx->d2_ready, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ctx->top_ready, cudaEventDisableTiming);
    if (e != cudaSuccess) {
        fic_ctx_destroy(ctx);
        return FIC_ERR_CUDA;
    }
    *out = ctx;
    return FIC_OK;
}

fic_status fic_ctx_set_stream(fic_ctx *ctx, void *cuda_stream) {
    if (!ctx) return FIC_ERR_ARG;
    ctx->stream = (cudaStream_t)cuda_stream;
    return FIC_OK;
}

fic_status fic_ctx_set_timing(fic_ctx *ctx, int32_t enable) {
    if (!ctx) return FIC_ERR_ARG;
    ctx->timing = enable < 0 ? 0 : (enable > 2 ? 2 : enable);
    return FIC_OK;
}

fic_status fic_ctx_destroy(fic_ctx *ctx) {
    if (!ctx) return FIC_ERR_ARG;
    cudaSetDevice(ctx->device);
    if (ctx->stream) cudaStreamSynchronize(ctx->stream);
    for (auto &P : ctx->levels) free_pool(P);
    Buf *bufs[] = {&ctx->b_blocksum, &ctx->b_counts, &ctx->b_rng[0], &ctx->b_rng[1], &ctx->b_rec,
                   &ctx->b_acc, &ctx->b_child, &ctx->b_part, &ctx->b_t2f, &ctx->b_img, &ctx->b_out,
                   &ctx->b_scounts, &ctx->b_u, &ctx->b_gthr, &ctx->b_rop, &ctx->b_dec, &ctx->b_nccl};
    if (ctx->comm) ncclCommDestroy(ctx->comm);
    for (Buf *b : bufs) free_buf(*b);
    if (ctx->d_delta) cudaFree(ctx->d_delta);
    if (ctx->h_counts) cudaFreeHost(ctx->h_counts);
    for (auto &row : ctx->ev)
        for (auto &e : row)
            if (e) cudaEventDestroy(e);
    for (auto &e : ctx->pool_ready)
        if (e) cudaEventDestroy(e);
    for (auto &e : ctx->level_done)
        if (e) cudaEventDestroy(e);
    free_buf(ctx->b_blocksum2);
    free_buf(ctx->b_d2);
    free_buf(ctx->b_code);
    if (ctx->main_ready) cudaEventDestroy(ctx->main_ready);
    if (ctx->d2_ready) cudaEventDestroy(ctx->d2_ready);
    if (ctx->top_ready) cudaEventDestroy(ctx->top_ready);
    if (ctx->side) {
        cudaStreamSynchronize(ctx->side);
        cudaStreamDestroy(ctx->side);
    }
    if (ctx->crit) {
        cudaStreamSynchronize(ctx->crit);
        cudaStreamDestroy(ctx->crit);
    }
    if (ctx->fork_ev) cudaEventDestroy(ctx->fork_ev);
    if (ctx->join_ev) cudaEventDestroy(ctx->join_ev);
    delete ctx;
    return FIC_OK;
}

const char *fic_last_error(const fic_ctx *ctx) { return ctx ? ctx->err.c_str() : "null context"; }

fic_status fic_get_stats(const fic_ctx *ctx, fic_level_stats *h_out, int32_t max_levels,
                         int32_t *h_n_levels) {
    if (!ctx) return FIC_ERR_ARG;
    const int32_t n = (int32_t)ctx->stats.size();
    if (h_n_levels) *h_n_levels = n;
    for (int32_t i = 0; i < n && i < max_levels && h_out; ++i) h_out[i] = ctx->stats[i];
    return FIC_OK;
}

static fic_status build_pool(fic_ctx *ctx, const uint8_t *img, int32_t N, int32_t B, int32_t L, double tau_nats,
                             int64_t topk, fic_pool **out) {
    CKS(ctx_check(ctx));
    if (!img || !out) return fail(ctx, FIC_ERR_ARG, "null argument");
    *out = nullptr;
    CKS(check_level(ctx, N, B, L));
    fic_pool *pool = new (std::nothrow) fic_pool();
    if (!pool) return fail(ctx, FIC_ERR_NOMEM, "host allocation failed");
    fic_status st = pool_enqueue(ctx, pool->P, img, N, B, L, tau_nats, topk, ctx->stream);
    if (st == FIC_OK) {
        cudaError_t e = cudaMemcpyAsync(ctx->h_counts, pool->P.d_misc, 3 * sizeof(unsigned long long),
                                        cudaMemcpyDeviceToHost, ctx->stream);
        if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
        if (e != cudaSuccess) st = cuda_fail(ctx, e, "pool counts", __LINE__);
    }
    if (st != FIC_OK) {
        free_pool(pool->P);
        delete pool;
        return st;
    }
    pool_take_counts(pool->P, ctx->h_counts);
    *out = pool;
    if (pool->P.n_k == 0) return fail(ctx, FIC_ERR_EMPTY_POOL, "no domain block passed the entropy filter");
    return FIC_OK;
}

fic_status fic_build_domain_pool(fic_ctx *ctx, const uint8_t *img, int32_t N, int32_t B, int32_t L,
                                 double tau_nats, fic_pool **out) {
    return build_pool(ctx, img, N, B, L, tau_nats, 0, out);
}

fic_status fic_build_domain_pool_topk(fic_ctx *ctx, const uint8_t *img, int32_t N, int32_t B, int32_t L,
                                      int64_t K, fic_pool **out) {
    if (K < 1) {
        if (out) *out = nullptr;
        return ctx ? fail(ctx, FIC_ERR_ARG, "pool size K must be >= 1") : FIC_ERR_ARG;
    }
    return build_pool(ctx, img, N, B, L, -1.0, K, out);
}

fic_status fic_pool_info(const fic_pool *pool, int64_t *h_n_candidates, int64_t *h_n_kept,
                         const uint8_t **keep_mask, const int32_t **kept, const int64_t **keys) {
    if (!pool) return FIC_ERR_ARG;
    if (h_n_candidates) *h_n_candidates = pool->P.n_c;
    if (h_n_kept) *h_n_kept = pool->P.n_k;
    if (keep_mask) *keep_mask = pool->P.keep;
    if (kept) *kept = pool->P.kept;
    if (keys) *keys = pool->P.keys;
    return FIC_OK;
}

fic_status fic_pool_destroy(fic_pool *pool) {
    if (!pool) return FIC_ERR_ARG;
    cudaSetDevice(pool->P.device);
    cudaDeviceSynchronize();
    free_pool(pool->P);
    delete pool;
    return FIC_OK;
}

fic_status fic_encode_level(fic_ctx *ctx, const uint8_t *img, int32_t N, const fic_pool *pool,
                            const int32_t *ranges, int64_t n_r, const double *h_s, int32_t n_s,
                            double rms_tol, int32_t is_min_level, fic_record *out) {
    CKS(ctx_check(ctx));
    if (!img || !pool || (!ranges && n_r) || (!out && n_r) || n_r < 0)
        return fail(ctx, FIC_ERR_ARG, "null argument");
    if (pool->P.N != N) return fail(ctx, FIC_ERR_SHAPE, "pool was built for another N");
    if (n_r > (int64_t)1 << 30) return fail(ctx, FIC_ERR_ARG, "too many ranges");
    CKS(check_s(ctx, h_s, n_s));
    if (pool->P.n_k < 1) return fail(ctx, FIC_ERR_EMPTY_POOL, "empty domain pool");
    if (reinterpret_cast<uintptr_t>(ranges) & 7) return fail(ctx, FIC_ERR_ARG, "ranges must be 8-byte aligned");
    CK(grow(ctx, ctx->b_acc, n_r + 16));
    ctx->stats.clear();
    fic_level_stats ls;
    memset(&ls, 0, sizeof ls);
    unsigned long long *d_counts = ptr<unsigned long long>(ctx->b_counts);
    // device range count for the level kernels (slot 20), exact-path counter (slot 8)
    CK(fic::launch_set_u64(d_counts + 20, (unsigned long long)n_r, ctx->stream));
    CK(cudaMemsetAsync(d_counts + 8, 0, sizeof(unsigned long long), ctx->stream));
    CK(cudaMemsetAsync(d_counts + 30, 0, sizeof(unsigned long long), ctx->stream));
    if (ctx->timing) CK(cudaEventRecord(ctx->ev[0][0], ctx->stream));
    CKS(level_enqueue(ctx, pool->P, img, reinterpret_cast<const int2 *>(ranges), d_counts + 20, n_r, h_s, n_s,
                      rms_tol, is_min_level, out, ptr<uint8_t>(ctx->b_acc), nullptr, 0,
                      reinterpret_cast<int32_t *>(d_counts + 30)));
    ls.B = pool->P.B; ls.n_candidates = pool->P.n_c; ls.n_kept = pool->P.n_k; ls.n_ranges = n_r;
    ls.pairs = n_r * pool->P.n_k * 8;
    ls.pairs_scanned = n_r * pool->P.n_k;  // not read back here (stream-asynchronous call)
    ctx->stats.push_back(ls);
    return FIC_OK;
}

// Device counters (b_counts, 64 x u64):
//   [0] running output total  [1] level accepted count  [2] next-level range count (scratch)
//   [8 + l] exact evaluations of level l   [16 + l] accepted at level l   [24..] error flag (int)
//   [32 + l] range count of level l
static fic_status encode_body(fic_ctx *ctx, const uint8_t *img, int32_t N, int32_t B_max, int32_t B_min,
                              int32_t L, const double *h_tau, const int64_t *h_topk, const double *h_s,
                              const int32_t *h_n_s, const double *h_rms_tol, int32_t shard, int32_t n_shards,
                              fic_record *out, int64_t capacity, int64_t *h_n_out);

// The encode runs on ctx->crit, forked from the caller's stream (the image is ready in its order)
// and joined back into it; ctx->stream is pointed at ctx->crit for the duration of the call.
static fic_status encode_impl(fic_ctx *ctx, const uint8_t *img, int32_t N, int32_t B_max, int32_t B_min,
                              int32_t L, const double *h_tau, const int64_t *h_topk, const double *h_s,
                              const int32_t *h_n_s, const double *h_rms_tol, int32_t shard, int32_t n_shards,
                              fic_record *out, int64_t capacity, int64_t *h_n_out) {
    CKS(ctx_check(ctx));
    cudaStream_t user = ctx->stream;
    CK(cudaEventRecord(ctx->fork_ev, user));
    CK(cudaStreamWaitEvent(ctx->crit, ctx->fork_ev, 0));
    ctx->stream = ctx->crit;
    const fic_status r = encode_body(ctx, img, N, B_max, B_min, L, h_tau, h_topk, h_s, h_n_s, h_rms_tol, shard,
                                     n_shards, out, capacity, h_n_out);
    ctx->stream = user;
    cudaEventRecord(ctx->join_ev, ctx->crit);
    cudaStreamWaitEvent(user, ctx->join_ev, 0);
    return r;
}

static fic_status encode_body(fic_ctx *ctx, const uint8_t *img, int32_t N, int32_t B_max, int32_t B_min,
                              int32_t L, const double *h_tau, const int64_t *h_topk, const double *h_s,
                              const int32_t *h_n_s, const double *h_rms_tol, int32_t shard, int32_t n_shards,
                              fic_record *out, int64_t capacity, int64_t *h_n_out) {
    if (h_n_out) *h_n_out = 0;
    if (!img || !(h_tau || h_topk) || !h_s || !h_n_s || !h_rms_tol || !h_n_out || (!out && capacity > 0) ||
        capacity < 0)
        return fail(ctx, FIC_ERR_ARG, "null argument");
    if (!pow2(B_max) || !pow2(B_min) || B_min < 2 || B_min > B_max)
        return fail(ctx, FIC_ERR_ARG, "B_max, B_min must be powers of two with 2 <= B_min <= B_max");
    if (n_shards < 1 || shard < 0 || shard >= n_shards) return fail(ctx, FIC_ERR_ARG, "bad shard");
    if (N < 1 || N % B_max) return fail(ctx, FIC_ERR_SHAPE, "N must be a multiple of B_max");
    int nl = 0;
    for (int32_t B = B_max; B >= B_min; B /= 2) ++nl;
    if (nl > fic::kMaxLevels) return fail(ctx, FIC_ERR_ARG, "too many levels");
    std::vector<int64_t> s_off(nl + 1, 0);
    for (int l = 0; l < nl; ++l) {
        CKS(check_level(ctx, N, B_max >> l, L));
        CKS(check_s(ctx, h_s + s_off[l], h_n_s[l]));
        if (h_topk && h_topk[l] < 1) return fail(ctx, FIC_ERR_ARG, "pool size K must be >= 1");
        s_off[l + 1] = s_off[l] + h_n_s[l];
    }
    cudaStream_t st = ctx->stream;
    ctx->stats.assign(nl, fic_level_stats{});
    unsigned long long *d_counts = ptr<unsigned long long>(ctx->b_counts);
    int32_t *d_err = reinterpret_cast<int32_t *>(d_counts + 24);
    CK(cudaMemsetAsync(d_counts, 0, 64 * sizeof(unsigned long long), st));

    const int64_t G = N / B_max;
    const int64_t Gmin = N / B_min;
    // the child bitmap is all zero between encodes: finalize marks it, select_grid clears what it
    // consumes; a fresh buffer or an encode that stopped half way is cleared here once
    {
        void *before = ctx->b_child.p;
        CK(grow(ctx, ctx->b_child, (size_t)(Gmin * Gmin) + 16));
        if (ctx->b_child.p != before || !ctx->child_clean)
            CK(cudaMemsetAsync(ctx->b_child.p, 0, ctx->b_child.cap, st));
        ctx->child_clean = false;
    }
    CK(grow(ctx, ctx->b_rng[0], sizeof(int2) * (size_t)(Gmin * Gmin)));
    CK(grow(ctx, ctx->b_rng[1], sizeof(int2) * (size_t)(Gmin * Gmin)));
    // range-count upper bounds of every level, and per-level slices of the record / accepted
    // buffers: the records of level l are gathered into `out` on the side stream while the main
    // stream already searches level l + 1, so levels must not share these buffers
    std::vector<int64_t> nr_bound(nl + 1, 0), rec_off(nl + 1, 0);
    {
        int64_t nb = G * G > shard ? (G * G - shard + n_shards - 1) / n_shards : 0;
        for (int l = 0; l < nl; ++l) {
            nr_bound[l] = nb;
            rec_off[l + 1] = rec_off[l] + nb + 16;
            const int64_t Gc = N / std::max<int32_t>((B_max >> l) / 2, 1);
            nb = std::min<int64_t>(4 * nb, Gc * Gc);
        }
    }
    CK(grow(ctx, ctx->b_rec, sizeof(fic_record) * (size_t)rec_off[nl]));
    CK(grow(ctx, ctx->b_acc, (size_t)rec_off[nl] + 16));
    CK(grow(ctx, ctx->b_blocksum, sizeof(int64_t) * fic::select_blocksum_len(Gmin * Gmin)));
    CK(grow(ctx, ctx->b_blocksum2, sizeof(int64_t) * fic::select_blocksum_len(Gmin * Gmin)));
    // 1. pools: level 0 on the main stream; levels >= 1 on the side stream, overlapping the
    //    level-0 search (pools depend only on the image)
    CK(cudaEventRecord(ctx->main_ready, st));  // the image is ready (caller's stream order)
    CK(cudaStreamWaitEvent(ctx->side, ctx->main_ready, 0));
    // 2. top-level ranges of this shard (row-major), selected on the side stream while the
    //    level-0 pool builds on the critical one (the level-0 search waits for top_ready)
    uint8_t *child = ptr<uint8_t>(ctx->b_child);
    const bool top_side = ctx->top_side;
    {
        cudaStream_t ts = top_side ? ctx->side : st;
        CK(fic::launch_top_flags(child, G, shard, n_shards, ts));
        CK(fic::launch_select_grid(child, G, B_max, ptr<int64_t>(ctx->b_blocksum), ptr<int2>(ctx->b_rng[0]),
                                   d_counts + 32, ts));
        // and the level-0 range preparation (operand + moments: image and ranges only), off the
        // critical stream too -- the level-0 search then follows its pool directly
        if (top_side && B_max >= 4) {
            const int64_t nr0 = G * G > shard ? (G * G - shard + n_shards - 1) / n_shards : 0;
            CK(grow(ctx, ctx->b_rop, fic::tc_range_bytes(B_max, nr0)));
            CK(fic::launch_tc_prep(B_max, img, N, ptr<int2>(ctx->b_rng[0]), d_counts + 32, nr0,
                                   ptr<uint8_t>(ctx->b_rop), ts));
        }
        if (top_side) CK(cudaEventRecord(ctx->top_ready, ts));
    }
    // the decimated image, once for every level, on the side stream: it overlaps the level-0
    // entropy filter (the level-0 pool waits for d2_ready; the side-stream pools follow it)
    const size_t d2_bytes = fic::tc_pool_d2_bytes(16, N, L);
    const uint16_t *d2 = nullptr;
    if (d2_bytes && B_max >= 4) {
        CK(grow(ctx, ctx->b_d2, d2_bytes));
        d2 = ptr<uint16_t>(ctx->b_d2);
        CK(fic::launch_decimate(img, N, L, ptr<uint16_t>(ctx->b_d2), ctx->side));
        CK(cudaEventRecord(ctx->d2_ready, ctx->side));
    }
    for (int l = 0; l < nl; ++l) {
        cudaStream_t ps = (l == 0 || !ctx->overlap_pools) ? st : ctx->side;
        ctx->launches = l == 0 && d2 ? 1 : 0;
        if (ctx->timing >= 2) CK(cudaEventRecord(ctx->ev[l][0], ps));
        // (n_kept is also written next to the other counters: one device -> host copy at the end)
        CKS(pool_enqueue(ctx, ctx->levels[l], img, N, B_max >> l, L, h_topk ? -1.0 : h_tau[l],
                         h_topk ? h_topk[l] : 0, ps, d_counts + 48 + l, d2, ps == ctx->side ? nullptr : ctx->d2_ready));
        CKS(t2f_enqueue(ctx, ctx->levels[l], h_s + s_off[l], h_n_s[l], ps));
        if (ctx->timing >= 2) CK(cudaEventRecord(ctx->ev[l][4], ps));
        if (l > 0) CK(cudaEventRecord(ctx->pool_ready[l], ps));
        ctx->stats[l].kernel_launches = ctx->launches;
    }
    ctx->launches = 4;  // top flags + select x3 (step 2)
    int64_t n_r_max = G * G > shard ? (G * G - shard + n_shards - 1) / n_shards : 0;
    std::vector<int64_t> bound(nl, 0);

    // 3. the quadtree, one level at a time, sizes carried on the device
    int cur = 0;
    int last_direct = -1;  // level whose records finalize wrote straight into `out`
    for (int l = 0; l < nl && n_r_max > 0; ++l) {
        const int32_t B = B_max >> l;
        const Pool &P = ctx->levels[l];
        const bool last = (l == nl - 1);
        const int64_t Gc = N / (B / 2 > 0 ? B / 2 : 1);
        bound[l] = n_r_max;
        if (l > 0) CK(cudaStreamWaitEvent(st, ctx->pool_ready[l], 0));
        if (l == 0 && top_side) CK(cudaStreamWaitEvent(st, ctx->top_ready, 0));
        fic_record *rec_l = ptr<fic_record>(ctx->b_rec) + rec_off[l];
        uint8_t *acc_l = ptr<uint8_t>(ctx->b_acc) + rec_off[l];
        if (last) {
            // every range of the last level is accepted: finalize writes the records straight
            // into `out` after those the side stream gathered for the earlier levels
            // (finalize waits for that gathering; the search overlaps it)
            CK(cudaEventRecord(ctx->main_ready, ctx->side));
            CKS(level_enqueue(ctx, P, img, ptr<int2>(ctx->b_rng[cur]), d_counts + 32 + l, n_r_max,
                              h_s + s_off[l], h_n_s[l], h_rms_tol[l], 1, rec_l, acc_l, nullptr, l, d_err, out,
                              d_counts + 0, capacity, d_counts + 16 + l, ctx->main_ready,
                              (l == 0 && top_side && B >= 4) ? 1 : 0));
            last_direct = l;  // (the host adds this level's count to the total after the copy)
        } else {
            CKS(level_enqueue(ctx, P, img, ptr<int2>(ctx->b_rng[cur]), d_counts + 32 + l, n_r_max,
                              h_s + s_off[l], h_n_s[l], h_rms_tol[l], 0, rec_l, acc_l, child, l, d_err,
                              nullptr, nullptr, 0, nullptr, nullptr, (l == 0 && top_side && B >= 4) ? 1 : 0));
            // the accepted records of this level go to `out` on the side stream (in level order,
            // after the pools there), off the critical path of the next level's search
            CK(cudaEventRecord(ctx->level_done[l], st));
            CK(cudaStreamWaitEvent(ctx->side, ctx->level_done[l], 0));
            CK(fic::launch_select_records(acc_l, n_r_max, ptr<int64_t>(ctx->b_blocksum2), rec_l, out,
                                          d_counts + 0, capacity, d_counts + 16 + l, ctx->side));
            CK(fic::launch_accumulate(d_counts + 0, d_counts + 16 + l, ctx->side));
            ctx->launches += 2;
        }
        ctx->levels[l].t2f_ready = 0;
        if (!last) {
            CK(fic::launch_select_grid(child, Gc, B / 2, ptr<int64_t>(ctx->b_blocksum),
                                       ptr<int2>(ctx->b_rng[cur ^ 1]), d_counts + 33 + l, st));
            ctx->launches += 3;
            n_r_max = std::min<int64_t>(4 * n_r_max, Gc * Gc);
        }
        ctx->stats[l].kernel_launches += ctx->launches;
        ctx->launches = 0;
        cur ^= 1;
    }
    // 4. join the side stream (record gathering, pools of levels the quadtree never reached),
    //    then one device -> host read of every counter and one synchronisation
    for (int l = 1; l < nl; ++l) CK(cudaStreamWaitEvent(st, ctx->pool_ready[l], 0));
    CK(cudaEventRecord(ctx->main_ready, ctx->side));
    CK(cudaStreamWaitEvent(st, ctx->main_ready, 0));
    const bool trace = ctx->timing >= 2 && getenv("FIC_TRACE");
    if (trace) CK(cudaEventRecord(ctx->ev[fic::kMaxLevels - 1][0], st));
    if (ctx->counts_kernel) {
        CK(fic::launch_copy_counts(d_counts, ctx->h_counts, 64, st));
        ctx->stats[0].kernel_launches += 1;
    } else
        CK(cudaMemcpyAsync(ctx->h_counts, d_counts, 64 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
    if (trace) CK(cudaEventRecord(ctx->ev[fic::kMaxLevels - 1][1], st));
    const auto hs0 = std::chrono::steady_clock::now();
    CK(cudaStreamSynchronize(st));
    const auto hs1 = std::chrono::steady_clock::now();
    if (trace) fprintf(stderr, "[trace] host waited %.3f ms in the sync\n", std::chrono::duration<double, std::milli>(hs1 - hs0).count());
    if (trace) {
        float a = 0, b = 0;
        cudaEventElapsedTime(&a, ctx->ev[0][0], ctx->ev[fic::kMaxLevels - 1][0]);
        cudaEventElapsedTime(&b, ctx->ev[0][0], ctx->ev[fic::kMaxLevels - 1][1]);
        fprintf(stderr, "[trace] joined at %.3f ms, counters copied at %.3f ms\n", a, b);
    }
    const unsigned long long *h = ctx->h_counts;
    if (*reinterpret_cast<const int32_t *>(h + 24) == FIC_ERR_EMPTY_POOL)
        return fail(ctx, FIC_ERR_EMPTY_POOL, "empty domain pool at a level that has ranges");
    if (*reinterpret_cast<const int32_t *>(h + 24) != 0)
        return fail(ctx, FIC_ERR_CUDA, "internal consistency check failed in finalize");
    for (int l = 0; l < nl; ++l) {
        fic_level_stats &ls = ctx->stats[l];
        const Pool &P = ctx->levels[l];
        ls.B = B_max >> l;
        ls.n_candidates = P.n_c;
        ls.n_ranges = bound[l] > 0 ? (int64_t)h[32 + l] : 0;
        ls.n_accepted = (int64_t)h[16 + l];
        ls.exact_evals = (int64_t)h[8 + l];
        ls.n_kept = -1;  // filled below from the pool counters
    }
    for (int l = 0; l < nl; ++l) {
        fic_level_stats &ls = ctx->stats[l];
        ls.n_kept = (int64_t)ctx->h_counts[48 + l];
        ctx->levels[l].n_k = ls.n_kept;
        ls.pairs = ls.n_ranges * ls.n_kept * 8;
        const int64_t sc = (int64_t)ctx->h_counts[40 + l];
        ls.pairs_scanned = sc > 0 ? sc : ls.n_ranges * ls.n_kept;
    }
    if (ctx->timing) {
        for (int l = 0; l < nl; ++l) {
            fic_level_stats &ls = ctx->stats[l];
            if (bound[l] == 0) continue;
            float a = 0, b = 0, c = 0;
            cudaEventElapsedTime(&b, ctx->ev[l][1], ctx->ev[l][2]);
            if (ctx->timing >= 2) {
                cudaEventElapsedTime(&a, ctx->ev[l][0], ctx->ev[l][4]);
                cudaEventElapsedTime(&c, ctx->ev[l][2], ctx->ev[l][3]);
            }
            ls.ms_pool = a; ls.ms_search = b; ls.ms_finalize = c;
            if (ctx->timing >= 2 && getenv("FIC_TRACE")) {
                float g = 0, p0 = 0;
                if (l > 0) cudaEventElapsedTime(&g, ctx->ev[l - 1][3], ctx->ev[l][1]);
                cudaEventElapsedTime(&p0, ctx->ev[0][0], ctx->ev[l][1]);
                fprintf(stderr, "[trace] level %d: search starts at %.3f ms, gap after previous finalize %.3f ms, search %.3f, finalize %.3f\n", l, p0, g, b, c);
            }
        }
    }
    for (int l = 0; l < nl; ++l) ctx->levels[l].t2f_ready = 0;
    ctx->child_clean = true;  // every bitmap byte finalize marked was consumed by select_grid
    const int64_t total = (int64_t)ctx->h_counts[0] + (last_direct >= 0 ? (int64_t)ctx->h_counts[16 + last_direct] : 0);
    *h_n_out = total;
    if (total > capacity) return fail(ctx, FIC_ERR_CAPACITY, "output capacity too small");
    return FIC_OK;
}

fic_status fic_encode(fic_ctx *ctx, const uint8_t *img, int32_t N, int32_t B_max, int32_t B_min, int32_t L,
                      const double *h_tau, const double *h_s, const int32_t *h_n_s, const double *h_rms_tol,
                      int32_t shard, int32_t n_shards, fic_record *out, int64_t capacity, int64_t *h_n_out) {
    return encode_impl(ctx, img, N, B_max, B_min, L, h_tau, nullptr, h_s, h_n_s, h_rms_tol, shard, n_shards, out,
                       capacity, h_n_out);
}

fic_status fic_encode_topk(fic_ctx *ctx, const uint8_t *img, int32_t N, int32_t B_max, int32_t B_min, int32_t L,
                           const int64_t *h_K, const double *h_s, const int32_t *h_n_s, const double *h_rms_tol,
                           int32_t shard, int32_t n_shards, fic_record *out, int64_t capacity,
                           int64_t *h_n_out) {
    if (h_K) {
        int nl = 0;
        for (int32_t B = B_max; B >= B_min && B > 0 && nl < 64; B /= 2) ++nl;
        for (int l = 0; l < nl; ++l)
            if (h_K[l] < 1) {
                if (h_n_out) *h_n_out = 0;
                return ctx ? fail(ctx, FIC_ERR_ARG, "pool size K must be >= 1") : FIC_ERR_ARG;
            }
    }
    return encode_impl(ctx, img, N, B_max, B_min, L, nullptr, h_K, h_s, h_n_s, h_rms_tol, shard, n_shards, out,
                       capacity, h_n_out);
}

fic_status fic_encode_host(fic_ctx *ctx, const uint8_t *h_img, int32_t N, int32_t B_max,
                           int32_t B_min, int32_t L, const double *h_tau, const double *h_s,
                           const int32_t *h_n_s, const double *h_rms_tol, int32_t shard,
                           int32_t n_shards, fic_record *h_out, int64_t capacity, int64_t *h_n_out) {
    CKS(ctx_check(ctx));
    if (!h_img || !h_n_out || (!h_out && capacity > 0) || N < 1) return fail(ctx, FIC_ERR_ARG, "null argument");
    CK(grow(ctx, ctx->b_img, (size_t)N * N));
    CK(grow(ctx, ctx->b_out, sizeof(fic_record) * (size_t)(capacity > 0 ? capacity : 1)));
    CK(cudaMemcpyAsync(ctx->b_img.p, h_img, (size_t)N * N, cudaMemcpyHostToDevice, ctx->stream));
    fic_status st = fic_encode(ctx, ptr<uint8_t>(ctx->b_img), N, B_max, B_min, L, h_tau, h_s, h_n_s,
                               h_rms_tol, shard, n_shards, ptr<fic_record>(ctx->b_out), capacity,
                               h_n_out);
    if (st != FIC_OK && st != FIC_ERR_CAPACITY) return st;
    const int64_t n = *h_n_out < capacity ? *h_n_out : capacity;
    if (n > 0)
        CK(cudaMemcpyAsync(h_out, ctx->b_out.p, sizeof(fic_record) * (size_t)n, cudaMemcpyDeviceToHost,
                           ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    return st;
}

fic_status fic_merge_shards(fic_ctx *ctx, const fic_record *in, const int64_t *h_counts,
                            int32_t n_shards, int64_t stride, fic_record *out) {
    CKS(ctx_check(ctx));
    if (!in || !h_counts || !out || n_shards < 1) return fail(ctx, FIC_ERR_ARG, "null argument");
    int64_t mx = 0;
    for (int i = 0; i < n_shards; ++i) {
        if (h_counts[i] < 0 || h_counts[i] > stride) return fail(ctx, FIC_ERR_ARG, "bad shard count");
        if (h_counts[i] > mx) mx = h_counts[i];
    }
    CK(grow(ctx, ctx->b_scounts, sizeof(int64_t) * n_shards));
    CK(cudaMemcpyAsync(ctx->b_scounts.p, h_counts, sizeof(int64_t) * n_shards, cudaMemcpyHostToDevice,
                       ctx->stream));
    CK(fic::launch_merge_shards(in, ptr<int64_t>(ctx->b_scounts), n_shards, stride, mx, out, ctx->stream));
    return FIC_OK;
}

}  // extern "C"
