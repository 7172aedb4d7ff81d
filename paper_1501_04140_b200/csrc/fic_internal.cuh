// fic_internal.cuh -- internal declarations of libfic (B200 / sm_100a).  Not part of the ABI.
//
// Layout of one level's pool in HBM (DESIGN.md §5 "Data layout"):
//   Dtc u8 [n_tiles][chunks][128 x KCH]  tcgen05 A operand (B >= 4), core-matrix layout
//   F2 / Cs / ds                         B = 2 closed-form pool, sorted by C
//   SDf float [n_tiles*128], SD int32, C int64   domain moments (C = n*SDD - SD^2)
// Pad domains (index >= n_kept) carry t2f = +inf, so the search filter never admits them.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <cmath>
#include <string>
#include <utility>

#include "fic.h"

namespace fic {

constexpr int kTileD = 128;  // domains per pool tile
constexpr int kMaxS = 32;    // s values per level (5-bit closed-form levels)
constexpr int kMaxLevels = 8;
// Smallest s > 0 for which the searches may take the isometry as the lowest argmax of SRD_k
// (distinct SRD give distinct binary64 scores; DESIGN.md §6 "Exactness"): a level whose s list
// holds some s in (0, kSLicensed) has finalize re-derive (k, j) from the definition.
constexpr double kSLicensed = 9.5367431640625e-07;  // 2^-20
// Partial.kj flag: s index final, isometry k* not yet evaluated (finalize computes it for the
// winning domain; the B = 2 search defers it because the same domain never competes twice)
constexpr int32_t kPendIso = 1 << 16;

struct Buf {
    void *p = nullptr;
    size_t cap = 0;
};

struct B2Pool {          // B = 2 pool, sorted by C (stable)
    float4 *F = nullptr;    // [slots] features (Y2, yr + yi, yr - yi, C) in sorted order
    int32_t *Cs = nullptr;  // [slots] C in sorted order (pads 0xffffff)
    int32_t *ds = nullptr;  // [slots] kept-domain rank of each sorted position
    int32_t *ctab = nullptr;  // [ctab_n] first sorted position with C >= (t sqrt(Cmax) / ctab_n)^2
    int32_t ctab_n = 0;       // entries: a power of two >= slots / 16, at least 4096
};
// entries of the coarse index of the sorted C (b2_ctab_kernel): ~16 domains per bin on average
inline int32_t b2_ctab_entries(int64_t slots) {
    int64_t e = 4096;
    while (e < slots / 16 && e < (1 << 22)) e *= 2;
    return (int32_t)e;
}

// One level's entropy-filtered domain pool (fic_pool).
struct Pool {
    int32_t N = 0, B = 0, L = 0, n = 0, A = 0;
    int64_t n_c = 0, n_k = 0, n_tiles = 0, n_tiles_max = 0;
    int64_t cmax = 0;  // max C over kept domains (host copy, for the filter margin)
    int64_t *keys = nullptr;
    uint8_t *keep = nullptr;
    int32_t *kept = nullptr;
    float *SDf = nullptr;
    uint8_t *Dtc = nullptr; // tcgen05 A operand: [tiles][chunks][128 x KCH] core-matrix u8, or null
    B2Pool b2;              // B = 2 closed-form pool (sorted by C)
    int mode = 0;           // 0: tcgen05 (Dtc, B >= 4), 3: B = 2 closed form (F2)
    int32_t *SD = nullptr;
    int64_t *C = nullptr;
    unsigned long long *d_misc = nullptr;  // [0] = n_kept, [1] = Cmax, [2] = max |dh|_2 (float bits)
    double dnmax = 0.0;
    Buf b_keys, b_keep, b_kept, b_SDf, b_SD, b_C, b_misc, b_Dtc, b_F2, b_blocksum, b_topk, b_D2;
    Buf b_t2f;           // fp32 filter table of this level, enqueued with the pool (fic_encode)
    int t2f_ready = 0;   // b_t2f holds the table for the level's s set (reset after the level)
    int device = 0;
};

// Best candidate of one range over a subset of domains (lexicographic (e; dom, iso, s_idx)).
struct Partial {
    double e;
    int32_t d;
    int32_t kj;  // iso << 8 | s_idx (kPendIso: iso not yet resolved)
};

// A level's positive s values that form a uniform grid s_j = a + j h (j = 0..K-1, K >= 3, up to
// 1e-12 relative): the 16-value grid, sampled10 and the 5-bit closed-form levels.  The fp32
// filter then scores only the two grid points around s* = 4 Bq / C (the parabola's vertex,
// Eq. 2), which bracket the nearest one -- a tight estimate of the minimum over the whole set
// (not just a lower bound), so threshold seeding works as for the predefined sets.
struct SGrid {
    int32_t on;   // 0: not a uniform grid
    int32_t K;
    float a, h, aoh;  // a, h and a / h as fp32
};
inline SGrid detect_sgrid(const double *spos, int nsp) {
    SGrid g;
    g.on = 0; g.K = nsp; g.a = g.h = g.aoh = 0.f;
    if (nsp < 3) return g;
    const double a = spos[0], h = (spos[nsp - 1] - spos[0]) / (double)(nsp - 1);
    if (!(h > 0.0)) return g;
    for (int j = 0; j < nsp; ++j) {
        const double v = a + (double)j * h;
        if (!(fabs(spos[j] - v) <= 1e-12 * (fabs(spos[j]) + 1e-300))) return g;
    }
    g.on = 1;
    g.a = (float)a; g.h = (float)h; g.aoh = (float)(a / h);
    return g;
}

// Level sizes live on the device (no host round trip between levels): n_r = *d_nr,
// n_kept = d_misc[0], Cmax = d_misc[1]; host fields n_r / n_tiles are UPPER BOUNDS used only
// to size grids and buffers; a CTA's domain tiles are [split nt / nsplit, (split+1) nt / nsplit).
struct SearchParams {
    const uint8_t *img;
    int32_t N;
    const int2 *ranges;
    int32_t n_r;  // upper bound
    const unsigned long long *d_nr;    // actual range count
    const unsigned long long *d_misc;  // pool: [0] n_kept, [1] Cmax, [2] max |dh|
    int64_t slot_stride;               // n_tiles (upper bound) * 128: stride of t2f rows
    const float *SDf;
    const int32_t *SD;
    const int64_t *C;
    const float *t2f;  // [nsp][n_tiles*128]
    int32_t n_k, n_tiles, tiles_per_split, nsplit;
    int32_t nsp;                 // number of s values > 0
    double spos[kMaxS];          // those s values
    int32_t jpos[kMaxS];         // their indices in the level's s list
    int32_t has_zero, j_zero;    // s = 0 present, and its first index
    double smax;                 // max s
    double cmax;                 // max C of the pool (margin bound)
    Partial *part;               // [n_r][ns_cap]
    unsigned long long *exact_count;
    unsigned long long *d_ns;    // splits actually used (written by the search kernel)
    int32_t ns_cap;              // partial stride (max splits)
    int32_t b2_window;           // B = 2: Cauchy-Schwarz C windows (env FIC_B2_WINDOW=0 disables)
    int32_t L, Acnt;             // domain step and candidates per axis (threshold seeding)
    const int32_t *kept;         // kept-domain candidate indices
    int32_t num_sms;             // SMs of the context's device (persistent grids)
    SGrid grid;                  // the positive s form a uniform grid (nsp > 2)
    int32_t prep_done;           // the range preparation was enqueued ahead (launch_tc_prep)
};

struct FinalizeParams {
    const uint8_t *img;
    int32_t N, B, L, A;
    const int2 *ranges;
    int32_t n_r, nsplit;  // n_r: upper bound; nsplit: partial stride (ns_cap)
    const unsigned long long *d_nr;
    const unsigned long long *d_ns;  // splits actually used
    const unsigned long long *d_misc;
    int32_t *d_err;  // set to FIC_ERR_EMPTY_POOL if ranges meet an empty pool
    const Partial *part;
    const int32_t *SD;
    const int32_t *kept;
    int32_t n_k;
    int32_t fix_kj;  // the level's s list holds some s in (0, kSLicensed)
    double s[kMaxS];
    int32_t n_s, has_zero, j_zero;
    double rms_tol;
    int32_t is_min;
    fic_record *rec;
    uint8_t *accepted;
    uint8_t *child;  // child bitmap [(N/(B/2))^2] or null
    // last quadtree level (every range accepted): records straight into the output at
    // *d_base + r (< capacity), the level's count into *d_level_count; rec / accepted unused
    fic_record *out_direct;
    const unsigned long long *d_base;
    int64_t capacity;
    unsigned long long *d_level_count;
};

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (kernel, device): the attribute
// belongs to the function in each device's context, so the cache is a per-device bit mask
// (thread-safe; a second context on another device sets it again there).
template <class F>
inline cudaError_t ensure_smem_attr(F *fn, int bytes, std::atomic<unsigned long long> &done_mask) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    const unsigned long long bit = 1ull << (dev & 63);
    if (done_mask.load(std::memory_order_acquire) & bit) return cudaSuccess;
    e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (e == cudaSuccess) done_mask.fetch_or(bit, std::memory_order_acq_rel);
    return e;
}

// Programmatic dependent launch along the quadtree's critical path (finalize -> compaction ->
// range preparation -> search -> ...): each kernel there is launched with programmatic stream
// serialisation, lets its dependents launch as soon as all of its CTAs are running
// (pdl_trigger), and waits for its predecessor's completion and memory (pdl_wait) before it
// reads anything the predecessor wrote -- the dependent's launch and CTA placement overlap the
// predecessor's tail instead of following it.  Outside such a launch both are no-ops.
// FIC_PDL=0 launches them plainly.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
bool pdl_enabled();
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Args &&...args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

// Dynamic mapping of a CTA to (range group, domain split) from the actual counts: the grid is
// sized from host upper bounds; ns = min(ns_cap, ctas / groups, tiles / min_tiles) splits.
// Max of v over the block, one global atomicMax per block (same-address atomics from every
// thread serialise in L2). Every thread of the block must call it (no early returns before).
__device__ __forceinline__ void block_max_atomic(unsigned long long v, unsigned long long *dst) {
    __shared__ unsigned long long s_max[32];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long w = __shfl_xor_sync(0xffffffffu, v, o);
        v = w > v ? w : v;
    }
    if ((threadIdx.x & 31) == 0) s_max[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < (int)(blockDim.x >> 5); ++w) v = s_max[w] > v ? s_max[w] : v;
        if (v) atomicMax(dst, v);
    }
}

__device__ __forceinline__ bool cta_work(int n_r, int rpc, int n_tiles, int min_tiles, int ns_cap, int &group,
                                         int &split, int &ns) {
    const int groups = (n_r + rpc - 1) / rpc;
    const int ctas = (int)(gridDim.x * gridDim.y);
    ns = groups > 0 ? ctas / groups : 1;
    const int tcap = (n_tiles + min_tiles - 1) / min_tiles;
    if (ns > tcap) ns = tcap;
    if (ns > ns_cap) ns = ns_cap;
    if (ns < 1) ns = 1;
    const int item = (int)(blockIdx.y * gridDim.x + blockIdx.x);
    if (item >= groups * ns) return false;
    // split-major: CTAs that run early cover split 0 of every group, so later splits of a range
    // start from the thresholds its earlier splits already published (B = 2 shares them globally)
    split = item / groups;
    group = item % groups;
    return true;
}

// B = 4, 8 on the tcgen05 f16 form (fp16 operands, fp32 accumulator, exact; fic_tc.cu TCfg);
// -DFIC_TC_F16=0 builds the u8 polyphase form with the magic-number filter instead
#ifndef FIC_TC_F16
#define FIC_TC_F16 1
#endif
// scale of -s/2 in the tcgen05 epilogue's magic-number filter (u8 form at B <= 8, one or two s),
// which the t2f table folds the magic constant into; 0 = plain table (B = 2 keeps the fold)
__host__ __device__ constexpr float tc_t2_fold(int B, int nsp) {
    return (nsp >= 1 && nsp <= 2)
               ? (B == 2 ? 1.f : (FIC_TC_F16 ? 0.f : (B == 4 ? 2.f : (B == 8 ? 64.f : 0.f))))
               : 0.f;
}

// FIC1 body writer (fic_code.cu): per level (index 0 = B_max) the position and s-index widths
struct CodeParams {
    int32_t N, B_max, B_min, L;
    int32_t posbits[kMaxLevels], sbits[kMaxLevels], n_s[kMaxLevels];
};
size_t code_scratch_bytes(int64_t n);
// words: zeroed body buffer (>= ceil(bits / 32) words); *d_total = body length in bits;
// *d_bad (zeroed by the caller) = 1 if some record cannot be coded (out of bounds, unknown level)
cudaError_t launch_code_body(const fic_record *rec, int64_t n, const CodeParams &P, void *scratch,
                             unsigned *words, unsigned long long *d_total, int32_t *d_bad, cudaStream_t st);

// ---- launchers (return cudaError_t of the launch) ---------------------------------------------
cudaError_t launch_entropy_keys(const uint8_t *img, int32_t N, int32_t B, int32_t L, int32_t A,
                                const int64_t *d_delta, int64_t lut_m, int64_t T, int use_tau,
                                int64_t *keys, uint8_t *keep, cudaStream_t st);
// top-K pool selection (reading R27): keep[c] = 1 for the K largest keys (ties: lower index)
size_t topk_scratch_bytes(int64_t n_c);
cudaError_t launch_topk_select(const int64_t *keys, int64_t n_c, int64_t K, void *scratch, uint8_t *keep,
                               cudaStream_t st);
// order-preserving compaction of u8 flags: writes indices and *d_total
cudaError_t launch_select_index(const uint8_t *flags, int64_t n, int64_t *blocksum, int32_t *out,
                                unsigned long long *d_total, cudaStream_t st,
                                unsigned long long *d_total2 = nullptr);
cudaError_t launch_select_grid(const uint8_t *flags, int64_t G, int32_t B, int64_t *blocksum,
                               int2 *out, unsigned long long *d_total, cudaStream_t st);
// appends the flagged records at out[*d_base ...] (only below capacity), *d_total = count
cudaError_t launch_select_records(const uint8_t *flags, int64_t n, int64_t *blocksum,
                                  const fic_record *in, fic_record *out, const unsigned long long *d_base,
                                  int64_t capacity, unsigned long long *d_total, cudaStream_t st);
cudaError_t launch_set_u64(unsigned long long *d, unsigned long long v, cudaStream_t st);
// *d_acc += *d_add (single thread)
cudaError_t launch_accumulate(unsigned long long *d_acc, const unsigned long long *d_add, cudaStream_t st);
cudaError_t launch_copy_counts(const unsigned long long *d_src, unsigned long long *h_dst, int n, cudaStream_t st);

size_t select_blocksum_len(int64_t n);
cudaError_t launch_top_flags(uint8_t *flags, int64_t G, int32_t shard, int32_t n_shards,
                             cudaStream_t st);
cudaError_t launch_pool_moments(const uint8_t *img, int32_t N, int32_t B, int32_t L, int32_t A,
                                const int32_t *kept, const unsigned long long *d_nk,
                                int64_t n_slots, int32_t *SD, float *SDf, int64_t *C,
                                unsigned long long *d_cmax, cudaStream_t st);
struct SList {
    double s[kMaxS];
};

// univ: 0 one row per s (t2_j = s_j^2 C / 16, `fold` folds the magic constant), 1 the
// s-independent filter (RN(1/C)), 2 uniform grid (rows RN(C / 16), RN(4 / (C h)))
cudaError_t launch_t2f(const int64_t *C, const unsigned long long *d_nk, int64_t n_slots, const SList &spos,
                       int32_t nsp, float *t2f, int32_t univ, float fold, cudaStream_t st, float grid_h = 0.f);
cudaError_t launch_finalize(const FinalizeParams &p, cudaStream_t st);
cudaError_t launch_merge_shards(const fic_record *in, const int64_t *d_counts, int32_t n_shards,
                                int64_t stride, int64_t max_count, fic_record *out, cudaStream_t st);

// B = 2 closed-form search (fic_b2.cu)
size_t b2_pool_bytes(int64_t n_slots);
cudaError_t launch_b2_pool(const uint8_t *img, int32_t N, int32_t L, int32_t A, const int32_t *kept,
                           const unsigned long long *d_nk, int64_t n_slots, void *store, B2Pool *out,
                           int32_t *SD, float *SDf, int64_t *C, unsigned long long *d_cmax, cudaStream_t st);
int b2_nsplit_hint(int64_t n_r, int64_t n_tiles, int num_sms);
int b2_t2_width(int32_t nsp);  // floats per slot of the B = 2 t2 table
bool b2_wink_applies(const SearchParams &sp);  // B = 2 uniform-grid windows (b2wink_kernel)
size_t b2_scratch_bytes(int64_t n_r, int32_t ns_cap);  // pass-1 minima + split count
// scan_count: (range, domain) pairs the search evaluated (the windowed path proves the rest
// non-competitive); may be null
cudaError_t launch_b2_search(const SearchParams &sp, const B2Pool &bp, float *T, const int32_t *kept,
                             int32_t L, int32_t A, void *scratch, unsigned long long *scan_count,
                             cudaStream_t st);

// decoding and PSNR (fic_decode.cu)
struct DecSList {
    double s[kMaxLevels * kMaxS];
    int32_t off[kMaxLevels], n_s[kMaxLevels];
};
size_t decode_scratch_bytes(int32_t N, int64_t n_rec);
// passes alternate between scratch and out; *d_bad = 1 on an invalid record (checked by the caller)
cudaError_t launch_decode(const fic_record *rec, int64_t n_rec, int32_t N, int32_t B_max, int32_t n_levels,
                          const DecSList &sl, int32_t iterations, const uint8_t *init, uint8_t *out,
                          void *scratch, int32_t *d_bad, cudaStream_t st);
cudaError_t launch_sse(const uint8_t *a, const uint8_t *b, int64_t n, unsigned long long *d_sse, cudaStream_t st);

// tcgen05 search (fic_tc.cu), B in {4, 8, 16, 32}
int tc_supported(int B);
size_t tc_pool_bytes(int B, int64_t n_tiles);
int tc_nsplit_hint(int32_t B, int64_t n_r, int64_t n_tiles, int num_sms);
// also writes SD, SDf, C and Cmax when tc_pool_has_moments(B) (pool_moments_kernel is skipped)
int tc_pool_has_moments(int B);
// D2: workspace of tc_pool_d2_bytes(B, N, L) bytes (the 2 x 2 decimated image, B >= 16), else null
size_t tc_pool_d2_bytes(int B, int32_t N, int32_t L);
// the decimated image D2 (tc_pool_d2_bytes(B, N, L) bytes, any tc pool B) of img
cudaError_t launch_decimate(const uint8_t *img, int32_t N, int32_t L, uint16_t *D2, cudaStream_t st);
// D2 must hold the decimated image (launch_decimate, earlier in stream order) when
// tc_pool_d2_bytes(B, N, L) != 0
cudaError_t launch_pool_tc(const uint8_t *img, int32_t N, int32_t B, int32_t L, int32_t A,
                           const int32_t *kept, const unsigned long long *d_nk, int64_t n_tiles_max,
                           uint8_t *Dtc, int32_t *SD, float *SDf, int64_t *C, unsigned long long *d_cmax,
                           const uint16_t *D2, cudaStream_t st);
size_t tc_range_bytes(int B, int64_t n_r);  // scratch for the prepared range operand + metadata
// the range operand and moments of a level's ranges alone (they need only the image and the
// range list), ahead of launch_tc_search with sp.prep_done = 1 and the same scratch
cudaError_t launch_tc_prep(int32_t B, const uint8_t *img, int32_t N, const int2 *ranges,
                           const unsigned long long *d_nr, int64_t n_r, uint8_t *scratch, cudaStream_t st);
cudaError_t launch_tc_search(int32_t B, const SearchParams &sp, const uint8_t *Dtc, int64_t n_slots,
                             uint8_t *scratch, cudaStream_t st);

}  // namespace fic
