// fic_tc.cu -- the range x (domain, isometry) cross terms on the 5th-generation tensor cores
// (tcgen05.mma kind::i8, accumulators in TMEM), fused with the score filter and the exact
// first-min update.
//
// Contraction (exact, integer): SRD_k(r, d) = sum_p R_r(p) D'_d(f_k p)  (§2 lines 28-30)
//   D'(p) = sum of the 4 pixels of the 2x2 cell p, so with the four polyphase sub-images
//   P_ab(p) = I(y + 2i + a, x + 2j + b) of the raw 2B x 2B domain block:
//   SRD_k = sum_{ab} sum_p Rperm_k(p) P_ab(p),  Rperm_k(f_k p) = R(p)   (scatter through f_k)
//   i.e. one GEMM   S[m = domain][n = (range, k)] = sum_K A[m][K] B[n][K]
//   with A = the 4 u8 polyphase planes of each domain (K = 4 B^2, zero-padded to a multiple of
//   32) and B = the range scattered through the 8 isometries, replicated over the 4 planes.
//   u8 x u8 products accumulate exactly in s32 (max 4 B^2 255^2 < 2^31 for B <= 16).
// Epilogue (per TMEM lane = domain, per range): the 8 exact SRD_k, Bq = n max_k SRD_k - SR SD,
//   an fp32 lower bound of every binary64 score with a rigorous margin, and -- only when the
//   bound does not exclude the pair -- the canonical binary64 score and the lexicographic
//   (e; dom, k, j) first-min update; the running best of each range is shared by the CTA's
//   128 domain lanes through a shared-memory atomic threshold.
//
// B = 16 uses the QR form instead (A = the decimated D' as q = D' >> 2 and r = D' & 3 planes,
// two accumulators, SRD = 4 S_q + S_r).
//
// Persistent CTAs, one per SM (SegPlan: lockstep rounds of range groups for pools larger than
// ~L2/2, then a flattened (group, tile) tail in equal runs).  Roles: warp 0 = TMEM allocator +
// bulk-copy producer (lane 0 the A stages, lane 1 the per-segment range operand), warp 1 = MMA
// issuer (one elected thread), then EWG epilogue warpgroups (4; 2 at B = 32), each a share
// of the ranges; warp w reads TMEM lanes 32 (w % 4) ...  Pipelines: A stages full/empty
// (producer <-> MMA), two TMEM accumulator buffers full/empty (MMA <-> epilogue, released right
// after the tile's loads), range operand loaded/free (producer <-> MMA).
#include <algorithm>
#include <cfloat>
#include <climits>
#include <cstdlib>
#include <cstring>
#include <type_traits>

#include <cuda_fp16.h>

#include "fic_internal.cuh"

namespace fic {

// ------------------------------------------------------------------------------ configuration
template <int B>
struct TCfg {
    static constexpr int n = B * B;
    // B = 16 (QR): the A operand holds the decimated D' split as q = D' >> 2 and r = D' & 3
    // (two n-byte planes) and two MMAs per tile give S_q = sum R q and S_r = sum R r in two
    // accumulators, SRD = 4 S_q + S_r: half the MMA work, half the A bytes and a quarter of the
    // resident range operand of the 4-polyphase-plane form used at B <= 8 (where the epilogue,
    // not the MMA or the feed, is the bottleneck and a second accumulator would only add work)
    static constexpr bool QR = (B >= 16);
    // B = 4, 8 (F16): the decimated D' itself (<= 1020) and the range (<= 255) as fp16, which
    // represents them exactly, into an fp32 accumulator (kind::f16, K = 16 per instruction): every
    // partial sum is an integer below 2^24 (SRD <= 64 * 255 * 1020 = 16,646,400 at B = 8), so the
    // accumulation is exact and the epilogue gets SRD as floats -- a quarter of the MMA work and
    // half the A bytes of the 4-polyphase-plane u8 form, and no int -> float conversion
    static constexpr bool F16 = FIC_TC_F16 && (B == 4 || B == 8);
    static constexpr int KP = QR ? 2 * n : F16 ? 2 * n : ((4 * n + 31) / 32) * 32;  // A K bytes per domain
    static constexpr int KB = QR ? n : KP;                 // B operand K bytes per (range, k) row
    // ranges per CTA: 8 per epilogue warp per tile, 4 epilogue warpgroups.  B = 4 loads each
    // group's accumulators just before scoring it (FIC_SPLIT_LD), which keeps it under the 96
    // registers of 19 warps: 32 ranges x 4 warpgroups 0.472 ms against 24 x 3 at 128 registers
    // (all loads first) 0.504 ms
#ifndef FIC_B4_NR
#define FIC_B4_NR 32
#endif
#ifndef FIC_PROD_WARP
#define FIC_PROD_WARP 0
#define FIC_MMA_WARP 1
#endif
#ifndef FIC_PROD_NS
#define FIC_PROD_NS 0
#endif
#ifndef FIC_MMA_NS
#define FIC_MMA_NS 0
#endif
#ifndef FIC_B4_EWG
#define FIC_B4_EWG 4
#endif
#ifndef FIC_B8_NR
#define FIC_B8_NR 32
#endif
#ifndef FIC_B8_EWG
#define FIC_B8_EWG 4
#endif
#ifndef FIC_B16_NR
#define FIC_B16_NR 16
#endif
#ifndef FIC_B16_EWG
#define FIC_B16_EWG 4
#endif
    // B = 32 (QR, n = 1024 K bytes per range row): 8 ranges, so the 64 KB range operand and two
    // 64 KB A stages fit shared memory
    static constexpr int NR = (B == 32) ? 8 : (B == 16) ? FIC_B16_NR : (B == 4 ? FIC_B4_NR : FIC_B8_NR);
    static constexpr int N = 8 * NR;                       // MMA N (columns per accumulator)
    // B = 16: one 64 KB stage per tile (q and r planes), two stages.  Finer stages (KCH = 256, 4 or
    // 5 stages: FIC_B16_KCH / FIC_B16_STAGES) were measured slower (C3 B16 0.105 -> 0.107 /
    // 0.108 ms): the feed is bounded by the bulk-copy throughput, not by the bytes in flight
#ifndef FIC_B16_KCH
#define FIC_B16_KCH 512
#endif
#ifndef FIC_B16_STAGES
#define FIC_B16_STAGES 2
#endif
    static constexpr int KCH = QR ? (B == 16 ? FIC_B16_KCH : 512) : (KP < 256 ? KP : 256);  // K bytes per pipeline stage (F16: a tile)
    static constexpr int CH = KP / KCH;                    // stages per domain tile
    static constexpr int STAGE_BYTES = kTileD * KCH;       // A bytes per stage
    // A stages (one tile each in the f16 form): B = 4 8 x 4 KB, B = 8 4 x 16 KB; QR 2 x 64 KB (above)
#ifndef FIC_B4_STAGES
#define FIC_B4_STAGES 8
#endif
    static constexpr int STAGES = QR ? (B == 16 ? FIC_B16_STAGES : 2) : F16 ? (B == 4 ? FIC_B4_STAGES : 4) : (B == 8 ? 2 : 4);
    static constexpr int B_BYTES = N * KB;                 // resident range operand
    // range-operand buffers: 2 where shared memory allows, so the next segment's operand loads
    // while the current segment's MMAs still read the other one
    static constexpr int BBUF = (B == 4 || F16) ? 2 : 1;
    static constexpr int ACC = QR ? 2 * N : N;             // TMEM columns per accumulator buffer
    static constexpr int NBUF = 512 / ACC >= 4 ? 4 : 512 / ACC;  // TMEM accumulator buffers (MMA <-> epilogue)
    static constexpr int EWG = B == 4 ? FIC_B4_EWG : (B == 32 ? 2 : B == 8 ? FIC_B8_EWG : FIC_B16_EWG);  // epilogue warpgroups
    // ranges per warpgroup, in groups of 4 (one 32-column tcgen05.ld); when EWG does not divide
    // NR / 4 the last warpgroup's trailing groups are empty (skipped)
    static constexpr int HALF = ((NR + 4 * EWG - 1) / (4 * EWG)) * 4;
    // warps: producer, MMA issuer, 4 EWG epilogue warps, the exact-path warp
    static constexpr int XWARP = 2 + 4 * EWG;
    static constexpr int THREADS = 64 + 128 * EWG + 32;
    static constexpr int XQ = 512;                         // exact-path work ring (power of two)
    // exact-path best slots per range (slot = domain lane % RBW): 8 at B >= 16, whose 16 ranges
    // per CTA see bursts of items of one range; 1 at B <= 8 (C3: B = 4 0.530 vs 0.537 ms with 8)
    static constexpr int RBW = B >= 16 ? 8 : 1;
};

// One (range, domain) pair the fp32 filter could not exclude, queued for the exact-path warp.
struct XItem {
    int32_t mx;    // max_k SRD_k
    int32_t d;     // pool slot of the domain
    int32_t sd;    // its SD
    int32_t meta;  // range q (5 bits) | k* << 5 | domain lane m << 8
};

constexpr uint32_t kTmemCols = 512;

// ------------------------------------------------------------------------------ PTX helpers
__device__ __forceinline__ uint32_t su32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void tmbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void tmbar_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void tmbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(bar)) : "memory");
}
__device__ __forceinline__ void tmbar_wait_sa(uint32_t bar_sa, uint32_t parity) {  // shared address
    uint32_t done = 0;
    while (!done) {
        asm volatile(
            "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
            : "=r"(done)
            : "r"(bar_sa), "r"(parity)
            : "memory");
    }
}
__device__ __forceinline__ void tmbar_arrive_sa(uint32_t bar_sa) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar_sa) : "memory");
}
__device__ __forceinline__ void tmbar_wait(uint64_t *bar, uint32_t parity) {
    uint32_t done = 0;
    while (!done) {
        asm volatile(
            "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
            : "=r"(done)
            : "r"(su32(bar)), "r"(parity)
            : "memory");
    }
}
// the producer's and MMA warp's waits: probe, then sleep ns between probes -- a spinning control
// warp takes issue slots from the three epilogue warps of its SM sub-partition, which then lag
// the others and (through the shared TMEM buffers) pace the whole tile ring
__device__ __forceinline__ void tmbar_wait_sleep(uint64_t *bar, uint32_t parity, uint32_t ns) {
    uint32_t done = 0;
    for (;;) {
        asm volatile(
            "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
            : "=r"(done)
            : "r"(su32(bar)), "r"(parity)
            : "memory");
        if (done) break;
        __nanosleep(ns);
    }
}
__device__ __forceinline__ void tbulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            su32(dst)),
        "l"(src), "r"(bytes), "r"(su32(bar))
        : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_commit(uint64_t *bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(bar))
                 : "memory");
}
__device__ __forceinline__ void tc_mma_i8(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                          uint32_t accum) {
    asm volatile(
        "{ .reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p; }" ::"r"(
            tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accum)
        : "memory");
}
// the same, issued by the warp's elected lane: called by the whole (converged) warp, so the
// operands stay warp-uniform and ptxas needs no per-lane waterfall to move them to uniform registers
__device__ __forceinline__ void tc_mma_i8_elect(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                                uint32_t accum) {
    asm volatile(
        "{ .reg .pred p, e; setp.ne.b32 p, %4, 0; elect.sync _|e, 0xffffffff; "
        "@e tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p; }" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accum)
        : "memory");
}
__device__ __forceinline__ void tc_commit_elect(uint32_t bar_sa) {
    asm volatile(
        "{ .reg .pred e; elect.sync _|e, 0xffffffff; "
        "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0]; }" ::"r"(bar_sa)
        : "memory");
}
__device__ __forceinline__ void tc_ld8(uint32_t taddr, uint32_t (&v)[8]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
        : "r"(taddr));
}
template <int O, int W>
__device__ __forceinline__ void tc_ld32(uint32_t taddr, uint32_t (&w)[W]) {
    static_assert(O + 32 <= W, "tcgen05.ld destination");
    uint32_t *v = w + O;
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, "
        "%14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
          "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
          "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
        : "r"(taddr));
}
__device__ __forceinline__ void tc_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// K-major, no-swizzle canonical layout: 8-row x 16-byte core matrices; LBO = distance between
// the two 16-byte K halves of one MMA (128 B here), SBO = distance between 8-row groups.
__device__ __forceinline__ uint64_t smem_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
    d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
    d |= (uint64_t)1 << 46;  // descriptor version (sm_100)
    return d;                // base offset 0, lbo mode 0, layout SWIZZLE_NONE
}
// kind::i8 instruction descriptor: D s32, A u8, B u8, both K-major, M = 128, N
__host__ __device__ constexpr uint32_t idesc_i8(int N) {
    return (2u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
}
// kind::f16 instruction descriptor: D f32, A f16, B f16, both K-major, M = 128, N
__host__ __device__ constexpr uint32_t idesc_f16(int N) {
    return (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
}
__device__ __forceinline__ void tc_mma_f16_elect(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                                 uint32_t accum) {
    asm volatile(
        "{ .reg .pred p, e; setp.ne.b32 p, %4, 0; elect.sync _|e, 0xffffffff; "
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p; }" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accum)
        : "memory");
}
// two small non-negative integers (exact in fp16) packed as fp16 bits, low half first
__device__ __forceinline__ uint32_t f16x2_int(int lo, int hi) {
    return (uint32_t)__half_as_ushort(__int2half_rn(lo)) | ((uint32_t)__half_as_ushort(__int2half_rn(hi)) << 16);
}
// byte offset of element (row, kb) in a K-major no-swizzle operand with K bytes per row
__host__ __device__ __forceinline__ uint32_t cm_off(int row, int kb, int K) {
    return (uint32_t)((row >> 3) * (K / 16) * 128 + (kb >> 4) * 128 + (row & 7) * 16 + (kb & 15));
}

// GPU-side isometry source map (same derivation as fic_search.cu, reading R2)
__device__ __forceinline__ void tiso_src(int B, int k, int i, int j, int &si, int &sj) {
    const int b = B - 1;
    if (k >= 4) j = b - j;
    for (int r = 0; r < (k & 3); ++r) {
        const int t = i;
        i = b - j;
        j = t;
    }
    si = i;
    sj = j;
}

// orderable encoding of fp32 for atomicMin
__device__ __forceinline__ uint32_t f2ord(float f) {
    const uint32_t u = __float_as_uint(f);
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float ord2f(uint32_t o) {
    return __uint_as_float((o & 0x80000000u) ? (o & 0x7fffffffu) : ~o);
}

// ------------------------------------------------------------------------------ pool (A operand)
// Tile t, chunk c: 128 domains x KCH bytes in the core-matrix layout (one bulk copy per stage).
// All forms read the 2 x 2 sums D' from the once-decimated image D2 (decimate_kernel below: plane
// p = (y & 1, x & 1) holds D2_p[u][v] = the 2 x 2 block at (2u + oy, 2v + ox), rows of
// d2_pitch(N) elements, so D'(i, j) of the domain at (x, y) is D2_p[(y >> 1) + i][(x >> 1) + j]).
__host__ __device__ __forceinline__ int d2_pitch(int32_t N) { return ((N / 2 + 7) & ~7) + 8; }  // elements
// The 8 D' at element col .. col + 7 of a D2 row (16 bytes at an even byte offset within a
// 16-byte-aligned 32-byte window): two aligned 16-byte loads, words q .. q + 4 selected and
// funnel-shifted by (sh & 3) bytes; returned as 4 pairs (2 x 16 bits)
__device__ __forceinline__ void d2_load8(const uint16_t *row, int col, uint32_t (&pr)[4]) {
    const uint4 *src = reinterpret_cast<const uint4 *>(row + (col & ~7));
    const uint4 lo = __ldg(src), hi = __ldg(src + 1);
    const uint32_t wv[8] = {lo.x, lo.y, lo.z, lo.w, hi.x, hi.y, hi.z, hi.w};
    const int sh = (col & 7) * 2, qs = sh >> 2;
    const uint32_t fs = (uint32_t)(sh & 3) * 8;
    uint32_t sel[5];
#pragma unroll
    for (int k = 0; k < 5; ++k) sel[k] = qs == 0 ? wv[k] : qs == 1 ? wv[k + 1] : qs == 2 ? wv[k + 2] : wv[(k + 3) & 7];
#pragma unroll
    for (int k = 0; k < 4; ++k) pr[k] = __funnelshift_r(sel[k], sel[k + 1], fs);
}

// B = 4, 8 (f16 form): thread per 16-byte K group g = the decimated pixels 8g .. 8g + 7
// (row-major) as fp16, and the domain moments SD, SDD -> C = n SDD - SD^2 reduced over the
// domain's KP / 16 threads (consecutive lanes), which replaces pool_moments_kernel.  u8 form
// (FIC_TC_F16 = 0): the four polyphase planes of the raw block, moments by pool_moments_kernel.
template <int B>
__global__ void __launch_bounds__(256) pool_tc_kernel(const uint8_t *__restrict__ img, const uint16_t *__restrict__ D2,
                                                      int32_t N, int32_t L, int32_t A,
                                                      const int32_t *__restrict__ kept,
                                                      const unsigned long long *__restrict__ d_nk,
                                                      int64_t total16, uint8_t *__restrict__ Dtc,
                                                      int32_t *__restrict__ SD, float *__restrict__ SDf,
                                                      int64_t *__restrict__ Cm, unsigned long long *d_cmax) {
    using Cf = TCfg<B>;
    static_assert(!Cf::QR, "QR pools: pool_qr_kernel");
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;  // one 16-byte group
    const int64_t n_k = (int64_t)*d_nk;
    const int64_t ntiles = (n_k + kTileD - 1) / kTileD;
    constexpr int G16 = Cf::KP / 16;
    const int64_t tile = e / ((int64_t)kTileD * G16);
    const bool live = e < total16 && tile < ntiles;  // (no early return: block_max_atomic)
    const int rem = (int)(e - tile * kTileD * G16);
    const int m = rem / G16, g = rem % G16;
    const int64_t d = tile * kTileD + m;
    auto store16 = [&](int kb0, const uint32_t (&w)[4]) {  // chunk layout: [tile][chunk][128 x KCH]
        const int ch = kb0 / Cf::KCH, kc = kb0 % Cf::KCH;
        uint8_t *dst = Dtc + ((size_t)tile * Cf::CH + ch) * Cf::STAGE_BYTES + cm_off(m, kc, Cf::KCH);
        *reinterpret_cast<uint4 *>(dst) = make_uint4(w[0], w[1], w[2], w[3]);
    };
    if constexpr (Cf::F16) {
        uint32_t w[4] = {0, 0, 0, 0};
        int sd = 0, sdd = 0;
        if (live && d < n_k) {
            const int32_t c = kept[d];
            const int x = (c % A) * L, y = (c / A) * L;
            const int H = N / 2, W = d2_pitch(N);
            const uint16_t *base = D2 + (size_t)(((y & 1) << 1) | (x & 1)) * H * W + (size_t)(y >> 1) * W;
            const int col = x >> 1;
            uint32_t pr[4];  // D' pairs: pixels 8g + 2k, 8g + 2k + 1
            if constexpr (B == 8) {
                d2_load8(base + (size_t)g * W, col, pr);
            } else {  // B = 4: rows 2g, 2g + 1, four pixels each
#pragma unroll
                for (int r = 0; r < 2; ++r) {
                    const uint16_t *row = base + (size_t)(2 * g + r) * W + col;
                    pr[2 * r] = (uint32_t)__ldg(row) | ((uint32_t)__ldg(row + 1) << 16);
                    pr[2 * r + 1] = (uint32_t)__ldg(row + 2) | ((uint32_t)__ldg(row + 3) << 16);
                }
            }
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const int a = (int)(pr[k] & 0xFFFFu), b = (int)(pr[k] >> 16);
                sd += a + b;
                sdd += a * a + b * b;
                w[k] = f16x2_int(a, b);
            }
        }
        if (live) store16(g * 16, w);
#pragma unroll
        for (int o = 1; o < G16; o <<= 1) {
            sd += __shfl_xor_sync(0xffffffffu, sd, o);
            sdd += __shfl_xor_sync(0xffffffffu, sdd, o);
        }
        const long long cc = (long long)Cf::n * sdd - (long long)sd * sd;
        if (g == 0 && live) {
            SD[d] = sd;
            SDf[d] = (float)sd;
            Cm[d] = cc;
        }
        block_max_atomic(g == 0 && live && d < n_k ? (unsigned long long)cc : 0ull, d_cmax);
    } else {
        if (!live) return;
        uint32_t w[4] = {0, 0, 0, 0};
        if (d < n_k) {
            const int32_t c = kept[d];
            const int64_t x = (int64_t)(c % A) * L, y = (int64_t)(c / A) * L;
#pragma unroll
            for (int q = 0; q < 16; ++q) {
                const int kb = g * 16 + q;
                uint32_t v = 0;
                if (kb < 4 * Cf::n) {
                    const int plane = kb / Cf::n, p = kb % Cf::n;
                    const int i = p / B, j = p % B;
                    v = img[(y + 2 * i + (plane >> 1)) * N + x + 2 * j + (plane & 1)];
                }
                w[q >> 2] |= v << (8 * (q & 3));
            }
        }
        store16(g * 16, w);
    }
}

// QR pool (B = 16, 32) in two launches.  (1) decimate_kernel: the 2 x 2 sums of the whole image
// once per parity class (y & 1, x & 1) -- one class when L is even (every domain corner is even),
// four when L is odd -- as uint16 planes D2_p[u][v] = the 2 x 2 block at (2u + oy, 2v + ox), so
// D'(i, j) of the domain at (x, y) is D2_{(y&1, x&1)}[(y >> 1) + i][(x >> 1) + j].  (2)
// pool_qr_kernel: warp per domain (grid-stride over the slots), each lane one or four chunks of 8
// consecutive D' of a row: q = D' >> 2 and r = D' & 3 packed to 8 bytes each (one 8-byte store per
// plane into the K-major core-matrix layout), SD, SDD in int32 (< 2^31 at n = 1024) reduced with
// REDUX.  The 2 x 2 sums, previously formed per domain from the raw 2B x 2B block (each image pixel
// of a C3 pool read ~(2B / L)^2 = 256 times, 333 warp instructions per domain), are formed once.
__global__ void __launch_bounds__(256) decimate_kernel(const uint8_t *__restrict__ img, int32_t N, int32_t planes,
                                                       uint16_t *__restrict__ D2) {
    const int H = N / 2, W = d2_pitch(N);  // rows of W elements (16-byte aligned, zero padded)
    const int64_t per = (int64_t)H * W;
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= per * planes) return;
    const int p = (int)(e / per);
    const int rem = (int)(e - (int64_t)p * per);
    const int u = rem / W, v = rem - (rem / W) * W;
    const int oy = p >> 1, ox = p & 1;
    const int y = 2 * u + oy, x = 2 * v + ox;
    uint16_t s = 0;
    if (v < H && y + 1 < N && x + 1 < N) {
        const uint8_t *r0 = img + (size_t)y * N + x;
        s = (uint16_t)(r0[0] + r0[1] + r0[N] + r0[N + 1]);
    }
    D2[e] = s;
}

template <int B>
__global__ void __launch_bounds__(256) pool_qr_kernel(const uint16_t *__restrict__ D2, int32_t N, int32_t L,
                                                       int32_t A, const int32_t *__restrict__ kept,
                                                       const unsigned long long *__restrict__ d_nk,
                                                       uint8_t *__restrict__ Dtc, int32_t *__restrict__ SD,
                                                       float *__restrict__ SDf, int64_t *__restrict__ Cm,
                                                       unsigned long long *d_cmax) {
    using Cf = TCfg<B>;
    constexpr int CPR = B / 8;            // 8-column chunks per decimated row
    constexpr int CPL = B * CPR / 32;     // chunks per lane (1 at B = 16, 4 at B = 32)
    constexpr int GB = 8 * Cf::KCH;       // bytes of one 8-domain group in one stage (contiguous)
    constexpr int CMP = 144;              // padded core matrix in shared memory (128 B + 16)
    static_assert(Cf::QR && CPL >= 1, "QR pool (launched with 256 threads: 8 warps = 8 domains)");
    // the CTA's 8 domains (one per warp) staged in the core-matrix layout of their 8 rows, so the
    // tile is written with coalesced 16-byte stores of whole 128-byte core matrices (writing each
    // domain's rows straight to global memory touched 64 partial sectors per domain)
    __shared__ __align__(16) uint8_t stg[Cf::CH * (GB / 128) * CMP];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int H = N / 2, W = d2_pitch(N);
    const int64_t n_k = (int64_t)*d_nk;
    const int64_t slots = ((n_k + kTileD - 1) / kTileD) * kTileD;
    unsigned long long cmax = 0;
    for (int64_t g0 = (int64_t)blockIdx.x * 8; g0 < slots; g0 += (int64_t)gridDim.x * 8) {
        const int64_t d = g0 + w;
        int sd = 0, sdd = 0;
        auto put8 = [&](int kb, uint2 v) {  // 8 bytes at K byte kb of this warp's domain
            const int ch = kb / Cf::KCH, kc = kb % Cf::KCH;
            *reinterpret_cast<uint2 *>(stg + (ch * (GB / 128) + (kc >> 4)) * CMP + w * 16 + (kc & 15)) = v;
        };
        if (d < n_k) {
            const int32_t c = kept[d];
            const int x = (c % A) * L, y = (c / A) * L;
            const int col = x >> 1;
            const uint16_t *base = D2 + (size_t)(((y & 1) << 1) | (x & 1)) * H * W + (size_t)(y >> 1) * W;
#pragma unroll
            for (int t = 0; t < CPL; ++t) {
                const int chk = lane + 32 * t;
                const int i = chk / CPR, h = chk % CPR;
                uint32_t pr[4];  // D' pairs (2 x 16 bits)
                d2_load8(base + (size_t)i * W, col + 8 * h, pr);
                uint32_t qv[4], rv[4];
                uint32_t s2 = 0;
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    qv[k] = (pr[k] >> 2) & 0x00FF00FFu;
                    rv[k] = pr[k] & 0x00030003u;
                    s2 += pr[k];  // two 16-bit lanes, each <= 4 * 1020
                    const int a = (int)(pr[k] & 0xFFFFu), b = (int)(pr[k] >> 16);
                    sdd += a * a + b * b;
                }
                sd += (int)(s2 & 0xFFFFu) + (int)(s2 >> 16);
                const int kb = B * i + 8 * h;  // K byte of (i, 8h) in the q plane; the r plane at n + kb
                put8(kb, make_uint2(__byte_perm(qv[0], qv[1], 0x6420), __byte_perm(qv[2], qv[3], 0x6420)));
                put8(Cf::n + kb, make_uint2(__byte_perm(rv[0], rv[1], 0x6420), __byte_perm(rv[2], rv[3], 0x6420)));
            }
        } else {  // pad rows of the last tile: zero q and r planes
#pragma unroll
            for (int t = 0; t < 2 * CPL; ++t) put8(8 * (lane + 32 * t), make_uint2(0u, 0u));
        }
        sd = __reduce_add_sync(0xffffffffu, sd);
        sdd = (int)__reduce_add_sync(0xffffffffu, (unsigned)sdd);
        if (d < slots) {
            const long long cc = (long long)Cf::n * sdd - (long long)sd * sd;
            if (lane == 0) {
                SD[d] = sd;
                SDf[d] = (float)sd;
                Cm[d] = cc;
            }
            if (d < n_k && (unsigned long long)cc > cmax) cmax = (unsigned long long)cc;
        }
        __syncthreads();
        {  // the group's CH x GB bytes, 16 per thread per pass (slots are a multiple of kTileD = 128)
            const int64_t tile = g0 / kTileD;
            const int grp = (int)((g0 - tile * kTileD) >> 3);
            uint8_t *dst = Dtc + (size_t)tile * Cf::CH * Cf::STAGE_BYTES + (size_t)grp * GB;
            for (int e = threadIdx.x; e < Cf::CH * GB / 16; e += blockDim.x) {
                const int ch = e / (GB / 16), r = e % (GB / 16);
                const uint4 v = *reinterpret_cast<const uint4 *>(stg + (ch * (GB / 128) + (r >> 3)) * CMP + (r & 7) * 16);
                *reinterpret_cast<uint4 *>(dst + (size_t)ch * Cf::STAGE_BYTES + (size_t)r * 16) = v;
            }
        }
        __syncthreads();
    }
    block_max_atomic(cmax, d_cmax);
}

// the pools built from D2 with fused moments: QR (B = 16, 32) and the f16 form (B = 4, 8)
static bool TCfg_QR_or_F16(int B) {
    switch (B) {
    case 4: return TCfg<4>::F16;
    case 8: return TCfg<8>::F16;
    case 16: case 32: return true;
    default: return false;
    }
}
size_t tc_pool_d2_bytes(int B, int32_t N, int32_t L) {
    if (!TCfg_QR_or_F16(B)) return 0;
    return (L % 2 == 0 ? 1 : 4) * (size_t)(N / 2) * (size_t)d2_pitch(N) * sizeof(uint16_t);
}

int tc_supported(int B) { return B == 4 || B == 8 || B == 16 || B == 32; }

size_t tc_pool_bytes(int B, int64_t n_tiles) {
    switch (B) {
    case 4: return (size_t)n_tiles * TCfg<4>::CH * TCfg<4>::STAGE_BYTES;
    case 8: return (size_t)n_tiles * TCfg<8>::CH * TCfg<8>::STAGE_BYTES;
    case 16: return (size_t)n_tiles * TCfg<16>::CH * TCfg<16>::STAGE_BYTES;
    case 32: return (size_t)n_tiles * TCfg<32>::CH * TCfg<32>::STAGE_BYTES;
    default: return 0;
    }
}

int tc_pool_has_moments(int B) { return TCfg_QR_or_F16(B) ? 1 : 0; }

cudaError_t launch_decimate(const uint8_t *img, int32_t N, int32_t L, uint16_t *D2, cudaStream_t st) {
    const int64_t d2n = (int64_t)(tc_pool_d2_bytes(16, N, L) / sizeof(uint16_t));  // (size independent of B)
    if (d2n == 0) return cudaSuccess;
    decimate_kernel<<<(unsigned)((d2n + 255) / 256), 256, 0, st>>>(img, N, L % 2 == 0 ? 1 : 4, D2);
    return cudaGetLastError();
}

cudaError_t launch_pool_tc(const uint8_t *img, int32_t N, int32_t B, int32_t L, int32_t A,
                           const int32_t *kept, const unsigned long long *d_nk, int64_t n_tiles_max,
                           uint8_t *Dtc, int32_t *SD, float *SDf, int64_t *C, unsigned long long *d_cmax,
                           const uint16_t *D2, cudaStream_t st) {
    if (B != 4 && B != 8 && B != 16 && B != 32) return cudaErrorInvalidValue;
    if (n_tiles_max == 0) return cudaSuccess;
    if (tc_pool_d2_bytes(B, N, L) && !D2) return cudaErrorInvalidValue;
    if (B <= 8) {
        const int64_t total16 = n_tiles_max * kTileD * (B == 4 ? TCfg<4>::KP / 16 : TCfg<8>::KP / 16);
        const unsigned blocks = (unsigned)((total16 + 255) / 256);
        if (B == 4) pool_tc_kernel<4><<<blocks, 256, 0, st>>>(img, D2, N, L, A, kept, d_nk, total16, Dtc, SD, SDf, C, d_cmax);
        else pool_tc_kernel<8><<<blocks, 256, 0, st>>>(img, D2, N, L, A, kept, d_nk, total16, Dtc, SD, SDf, C, d_cmax);
    } else {  // warp per domain (pool_qr_kernel), one wave (6 CTAs of 256 threads per SM at <= 40
              // registers), grid-stride over the 8-domain groups
        const unsigned bq = (unsigned)std::min<int64_t>((n_tiles_max * kTileD + 7) / 8, 148 * 6);
        if (B == 16) pool_qr_kernel<16><<<bq, 256, 0, st>>>(D2, N, L, A, kept, d_nk, Dtc, SD, SDf, C, d_cmax);
        else pool_qr_kernel<32><<<bq, 256, 0, st>>>(D2, N, L, A, kept, d_nk, Dtc, SD, SDf, C, d_cmax);
    }
    return cudaGetLastError();
}

// ------------------------------------------------------------------------------ range operand
// Per group of NR ranges: rows (rl, k) = Rperm_k replicated over the 4 polyphase planes, K-major
// core-matrix layout, B_BYTES contiguous bytes (one bulk copy per CTA); zero rows past n_r.
template <int B>
__device__ __forceinline__ void tc_range_operand_body(const uint8_t *__restrict__ img, int32_t N,
                                                      const int2 *__restrict__ ranges,
                                                      const unsigned long long *__restrict__ d_nr,
                                                      int64_t total16, uint8_t *__restrict__ Bop, int bx) {
    using Cf = TCfg<B>;
    // source pixel of byte p of row k: Rperm_k(p) = R(f_k^{-1}(p)); under this numbering
    // f_k^{-1} = f_{k'} with k' = [0,3,2,1,4,5,6,7][k] (rotations by 90/270 swap, the rest are
    // involutions).  The block's ranges are first staged in shared memory (row-contiguous
    // loads); each thread then forms its 16 bytes from there, the source index in closed form
    // (mirror, then k' & 3 quarter turns) -- instead of a per-block table and 16 scattered
    // global byte loads per thread.
    constexpr int G16 = Cf::KB / 16;
    constexpr int RPB = (256 / G16 + 7) / 8 + 1;  // ranges a 256-thread block can touch
    __shared__ uint8_t sR[RPB][Cf::n];
    const int64_t e0 = (int64_t)bx * blockDim.x;
    const int64_t e = e0 + threadIdx.x;  // one 16-byte group
    const int64_t n_r = (int64_t)*d_nr;
    auto range_of = [&](int64_t ee) {  // range index of group ee's row
        const int64_t rg = ee / G16;
        return (rg / Cf::N) * Cf::NR + (int)(rg % Cf::N) / 8;
    };
    const int64_t r_first = range_of(e0);
    for (int t = threadIdx.x; t < RPB * Cf::n; t += blockDim.x) {
        const int q = t / Cf::n, p = t % Cf::n;
        const int64_t r = r_first + q;
        uint8_t v = 0;
        if (r < n_r && e0 < total16) {
            const int2 rr = ranges[r];
            v = img[(size_t)(rr.y + p / B) * N + rr.x + p % B];
        }
        sR[q][p] = v;
    }
    __syncthreads();
    if (e >= total16) return;
    if (e / ((int64_t)Cf::N * (Cf::KB / 16)) > (n_r + Cf::NR - 1) / Cf::NR) return;  // past the last group
    const int64_t row_g = e / G16;  // global row = group * N + row
    const int g = (int)(e % G16);
    const int64_t grp = row_g / Cf::N;
    const int row = (int)(row_g % Cf::N);
    const int rl = row >> 3, k = row & 7;
    const int64_t r = grp * Cf::NR + rl;
    const uint8_t *rs = sR[r - r_first];
    const int kinv = (k == 1) ? 3 : (k == 3 ? 1 : k), rot = kinv & 3;
    constexpr int b = B - 1;
    auto src = [&](int p) {  // pixel index of byte p of row k
        const int i = p / B, j0 = p % B;
        const int j = kinv >= 4 ? b - j0 : j0;
        const int si = rot == 0 ? i : rot == 1 ? b - j : rot == 2 ? b - i : j;
        const int sj = rot == 0 ? j : rot == 1 ? i : rot == 2 ? b - j : b - i;
        return si * B + sj;
    };
    uint32_t w[4] = {0, 0, 0, 0};
    if (Cf::F16 && r < n_r) {  // fp16 elements 8g .. 8g + 7 of Rperm_k
#pragma unroll
        for (int q = 0; q < 8; q += 2) w[q >> 1] = f16x2_int(rs[src(g * 8 + q)], rs[src(g * 8 + q + 1)]);
    } else if (r < n_r) {
#pragma unroll
        for (int q = 0; q < 16; ++q) {
            const int kb = g * 16 + q;
            uint32_t v = 0;
            if (kb < (Cf::QR ? Cf::n : 4 * Cf::n)) v = rs[src(kb % Cf::n)];  // 4 polyphase copies, or once (QR)
            w[q >> 2] |= v << (8 * (q & 3));
        }
    }
    uint8_t *dst = Bop + (size_t)grp * Cf::B_BYTES + cm_off(row, g * 16, Cf::KB);
    *reinterpret_cast<uint4 *>(dst) = make_uint4(w[0], w[1], w[2], w[3]);
}

struct TCRangeG {
    double A, margin;
    int32_t SR;
    int32_t valid;
};

// The fp32 filter's margin of one range (DESIGN.md §6 "Exactness"), from its A, the level's
// largest s and the pool's largest C
template <int B>
__device__ __forceinline__ double tc_margin(double A, double smax, double cmax, int univ) {
    double m;
    // fp32 filter error: |Bq| <= sqrt(A C) (Cauchy-Schwarz); the one rounding of Bq (or of Bq / n),
    // hs and t2 roundings, two FFMA roundings -> 8u (hs sqrt(A Cmax) + t2max)
    const double u = 5.9604644775390625e-08;
    const double hs = 0.5 * smax;
    const double bq = sqrt(A * cmax) * 1.01;  // every form converts an exact (or RN(Bq / n)) value once
    const double t2m = smax * smax * cmax * 0.0625;
    // + the int -> float conversion of Bq in the epilogue: exact at B = 2, |error| <= 2 at B = 4,
    // <= 64 at B = 8 (floor of Bq / 2 and Bq / 64)
    if (TCfg<B>::F16) {
        // F16: y = RN(SRD_max - SR (SD / n)) = RN(Bq / n) (one FFMA, SD / n exact), then
        // g = RN(nhs n y + t2): conversions of s / 2 and t2, the two roundings -> 4u (hs |Bq| + t2)
        m = 8.0 * u * (hs * bq + t2m) + 1e-12 * (A + hs * bq + t2m) + 1e-30;
    } else {
        m = 8.0 * u * (hs * bq + t2m) + 1e-12 * (A + hs * bq + t2m) +
                   (B == 4 ? hs * 2.0 : (B == 8 ? hs * 64.0 : 0.0)) + 1e-30;
        // folded magic constant (B <= 8): t2' = RN(t2 - nhs M) adds u |t2 - nhs M| <= u (t2m + hs k M)
        if (B <= 8) m += 2.0 * u * (t2m + hs * (B == 2 ? 1.0 : (B == 4 ? 2.0 : 64.0)) * 12582912.0);
    }
    // s-independent filter (NSP = 0): Bq rounded once, squared, times RN(1/C): <= 4.04u Bq^2/C <= 4.04u A
    if (univ == 1) m = 4.1 * u * A + 1e-12 * A + 1e-30;
    // uniform grid (NSP = 3): g(s) = s (s RN(C/16) - Bq/2) at two fp32 grid points s = fma(j, h, a):
    // Bq RN conversion, s rounding (incl. the 1e-12 grid fit), C/16 rounding, the FFMA and the
    // FMUL: |error| <= ~6u (hs |Bq| + 2 t2) -> 16u (hs |Bq|max + t2max)
    if (univ == 2)
        m = 16.0 * u * (hs * bq + t2m) + 1e-12 * (A + hs * bq + t2m) + 1e-30;
    return m;
}

// Thread per range: SR, A = n SRR - SR^2 (the filter margin is the search's: tc_margin)
template <int B>
__device__ __forceinline__ void tc_range_meta_body(const uint8_t *__restrict__ img, int32_t N,
                                                   const int2 *__restrict__ ranges,
                                                   const unsigned long long *__restrict__ d_nr, int32_t n_pad,
                                                   double smax, const unsigned long long *__restrict__ d_misc,
                                                   TCRangeG *__restrict__ meta, int32_t univ, int bx) {
    // B >= 8: a warp per range (lanes over the pixels), else a thread per range
    constexpr int TPR = B >= 8 ? 32 : 1;
    const int gt = bx * blockDim.x + threadIdx.x;
    const int r = gt / TPR, sub = gt % TPR;
    if (r >= n_pad) return;
    const int n_r = (int)*d_nr;
    constexpr int n = B * B;
    TCRangeG R;
    long long sr = 0, srr = 0;
    R.valid = r < n_r;
    if (R.valid) {
        const int2 rr = ranges[r];
        for (int p = sub; p < n; p += TPR) {
            const int v = img[(size_t)(rr.y + p / B) * N + rr.x + p % B];
            sr += v;
            srr += v * v;
        }
    }
    if constexpr (TPR > 1) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            sr += __shfl_xor_sync(0xffffffffu, sr, o);
            srr += __shfl_xor_sync(0xffffffffu, srr, o);
        }
        if (sub != 0) return;
    }
    R.A = (double)((long long)n * srr - sr * sr);
    R.SR = (int32_t)sr;
    R.margin = 0.0;  // formed by the search from the pool's Cmax (tc_margin): the preparation
                     // needs only the image and the ranges, so it can run before the pool exists
    meta[r] = R;
}

// both range-preparation passes in one launch: blocks [0, nb_op) build the range operand,
// the rest the per-range moments and margins
template <int B>
__global__ void __launch_bounds__(256) tc_range_prep_kernel(const uint8_t *__restrict__ img, int32_t N,
                                                            const int2 *__restrict__ ranges,
                                                            const unsigned long long *__restrict__ d_nr,
                                                            int64_t total16, uint8_t *__restrict__ Bop, int nb_op,
                                                            int32_t n_pad, double smax,
                                                            const unsigned long long *__restrict__ d_misc,
                                                            TCRangeG *__restrict__ meta, int32_t univ) {
    pdl_wait();
    pdl_trigger();
    if ((int)blockIdx.x < nb_op) tc_range_operand_body<B>(img, N, ranges, d_nr, total16, Bop, blockIdx.x);
    else tc_range_meta_body<B>(img, N, ranges, d_nr, n_pad, smax, d_misc, meta, univ, blockIdx.x - nb_op);
}

// ------------------------------------------------------------------------------ pipeline trace
// Diagnostics only (-DFIC_TC_TRACE, scripts/tc_trace.py): clock64 stamps of CTA 0's pipeline
// events -- 0 producer copy issued, 1 MMA saw the stage full, 2 MMA saw the accumulator free,
// 3 MMA committed the tile, 4 epilogue warp 2 saw the tile, 5 its loads done, 6 its tile done,
// 7 the last epilogue warp's tile done, 8 + w - 2 epilogue warp w's loads done; row 29: per
// epilogue warp w, [2w] cycles of tile work, [2w + 1] cycles waiting for tiles, [64 + 2w] cycles
// in push blocks, [64 + 2w + 1] push blocks.
#ifdef FIC_TC_TRACE
__device__ long long g_tc_trace[32][4096];
#define TC_TR(kind, idx)                                                           \
    do {                                                                           \
        if (blockIdx.x == 0 && (idx) < 4096) g_tc_trace[kind][idx] = clock64();   \
    } while (0)
__device__ __forceinline__ long long tc_gtime() {
    long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#define TC_TR_SEG(kind, k)                                                                        \
    do {                                                                                          \
        if (blockIdx.x < 512 && (k) < 8) g_tc_trace[kind][blockIdx.x * 8 + (k)] = tc_gtime();      \
    } while (0)
#define TC_TR_CTA(kind)                                                      \
    do {                                                                     \
        if (threadIdx.x == 0 && blockIdx.x < 4096) g_tc_trace[kind][blockIdx.x] = tc_gtime(); \
    } while (0)
#else
#define TC_TR(kind, idx) \
    do {                 \
    } while (0)
#define TC_TR_CTA(kind) \
    do {                \
    } while (0)
#define TC_TR_SEG(kind, k) \
    do {                   \
    } while (0)
#endif

// ------------------------------------------------------------------------------ search kernel
struct TCParams {
    const unsigned long long *d_nr, *d_misc;  // device sizes: n_r; n_kept, Cmax
    unsigned long long *d_ns;
    int32_t ns_cap;
    const uint8_t *Bop;        // [groups][B_BYTES] range operand
    const TCRangeG *rmeta;     // [groups * NR]
    const uint8_t *img;
    int32_t N;
    const int2 *ranges;
    int32_t n_r;
    const uint8_t *Dtc;
    const int32_t *SD;
    const int64_t *C;
    const float *t2f;  // [nsp][n_slots]
    int64_t n_slots;
    int32_t n_tiles, tiles_per_split, nsplit;
    int32_t nsp;
    double spos[kMaxS];
    int32_t jpos[kMaxS];
    int32_t has_zero, j_zero;
    double smax, cmax;
    Partial *part;
    unsigned long long *exact_count;
    int32_t lockstep;  // full rounds in lockstep (pool larger than ~L2/2), else all flattened
    int32_t num_sms;
    SGrid grid;        // NSP = 3: the positive s are the uniform grid a + j h, j < K
};

using TCRange = TCRangeG;

// NSP = number of s > 0 filtered one by one (1 or 2, the predefined sets); NSP = 0: any larger
// set (grid, sampled10, 5-bit closed form) through the s-independent lower bound
//     min_s e_s >= A - Bq^2 / C        (the unconstrained minimum of the parabola, Eq. 2)
// evaluated as g = -(Bq Bq) u, u = RN(1/C) per domain (t2f row 0), with Bq converted exactly
// (int -> float RN) -- margin 4.1u A (tc_range_meta_kernel).
// Work of one persistent CTA: a sequence of segments (one range group, a run of its domain
// tiles).  Pools larger than about half of L2 (P.lockstep): full rounds first -- while at least
// gridDim.x groups remain, CTA c takes group k gridDim.x + c over every tile, so all SMs stream
// the pool in the same order and each tile comes from HBM about once per round (C4: 33 -> 29.6 ms).
// The remaining groups (the tail; every group when the pool sits in L2, where spreading the SMs
// over the pool beats 148 SMs requesting the same lines) are flattened into (group, tile) order
// and cut into equal runs, one per CTA, so no SM idles in the last round; a group cut by CTA
// boundaries leaves one partial per run (slot c - c_first < ns_cap).
struct SegPlan {  // per CTA, in shared memory (kept out of the tile loops' registers)
    int R, Gc, c, T, gbase, n_tail;
    long long fbeg, f1, W;
};
// segment k of the CTA's plan: (group, first tile, tile count, partial slot, last of its group)
__device__ __forceinline__ void plan_segment(const SegPlan *sp, int k, int &grp, int &ta, int &ntl, int &slot,
                                             bool &lastseg) {
    const volatile SegPlan *v = sp;
    const int R = v->R, T = v->T;
    if (k < R) {
        grp = k * v->Gc + v->c; ta = 0; ntl = T; slot = 0; lastseg = true;
        return;
    }
    const long long fbeg = v->fbeg, f1 = v->f1, W = v->W;
    const long long g = fbeg / T + (k - R);
    const long long s0 = k == R ? fbeg : g * T;
    const long long fe = min(f1, (g + 1) * T);
    grp = v->gbase + (int)g;
    ta = (int)(s0 - g * T);
    ntl = (int)(fe - s0);
    slot = (int)(v->c - (g * T) / W);
    lastseg = fe == (g + 1) * T;
}

template <int B, int NSP>
__global__ void __launch_bounds__(TCfg<B>::THREADS, 1) tcsearch_kernel(const __grid_constant__ TCParams P) {
    pdl_wait();
    pdl_trigger();
    using Cf = TCfg<B>;
    constexpr int n = Cf::n, NR = Cf::NR, NN = Cf::N, KCH = Cf::KCH, CH = Cf::CH;
    constexpr int STAGES = Cf::STAGES;
    constexpr int HALF = Cf::HALF;  // ranges per epilogue warpgroup (the last may have fewer)
    constexpr bool UNEVEN = HALF * Cf::EWG != NR;
    static_assert(NR % 4 == 0 && Cf::NBUF >= (Cf::QR ? 1 : 2) && (Cf::EWG - 1) * HALF < NR,
                  "range groups of 4, >= 2 accumulator buffers, every warpgroup has ranges");
    extern __shared__ __align__(1024) uint8_t smem[];
    uint8_t *sA = smem;                                        // [STAGES][128 x KCH]
    uint8_t *sB = sA + STAGES * Cf::STAGE_BYTES;               // [N x KP]
    TCRange *sR = reinterpret_cast<TCRange *>(sB + Cf::BBUF * Cf::B_BYTES);   // [NR]
    float *sThr = reinterpret_cast<float *>(sR + NR);          // [NR] RU(best - A + margin), CAS-min
    float *sHsn = reinterpret_cast<float *>(sThr + NR);        // [NSP]
    int *sSR = reinterpret_cast<int *>(sHsn + 16);              // [NR] range sums (B = 8 reads them here)
    // [NR][RBW] range bests, RBW slots per range (slot = domain lane % RBW) so the exact warp's
    // updates of one range from different lanes rarely collide; written by the exact warp only
    Partial *sRB = reinterpret_cast<Partial *>(sSR + NR);
    constexpr int NBUF = Cf::NBUF;
    uint64_t *bar = reinterpret_cast<uint64_t *>(sRB + NR * Cf::RBW);  // full[S], empty[S], tfull[NB], tempty[NB], bop
    uint64_t *full = bar, *empty = bar + STAGES, *tfull = bar + 2 * STAGES, *tempty = tfull + NBUF;
    uint64_t *bbar = tempty + NBUF;  // [BBUF] range operand loaded, [BBUF] range operand free
    uint32_t *sTmem = reinterpret_cast<uint32_t *>(bbar + 4);
    XItem *sXQ = reinterpret_cast<XItem *>(sTmem + 4);               // [XQ] exact-path ring (16 B aligned)
    unsigned *sXSeq = reinterpret_cast<unsigned *>(sXQ + Cf::XQ);    // [XQ] slot i holds item i when = i + 1
    unsigned *sXCtl = sXSeq + Cf::XQ;  // [0] items reserved, [1] items consumed, [2] no more items
    float *sM2 = reinterpret_cast<float *>(sXCtl + 4);  // [NR] RU(2 margin) of the group's ranges

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int n_r = (int)*P.d_nr;
    const int T = (int)((P.d_misc[0] + kTileD - 1) / kTileD);  // domain tiles
    const int groups = (n_r + NR - 1) / NR;
    // persistent CTAs (one per SM), work decided before any barrier, uniformly per CTA (SegPlan)
    __shared__ SegPlan plan;
    int nseg_max = 1, nseg = 0;
    {
        const int R = P.lockstep ? groups / (int)gridDim.x : 0;
        const int rem = groups - R * (int)gridDim.x;
        const long long tail = (long long)rem * T;
        long long Gt = gridDim.x;
        Gt = min(Gt, (long long)rem * (P.ns_cap - 1));  // ceil(T / W) + 1 <= ns_cap slots per group
        Gt = min(Gt, max(1LL, tail / 4));               // >= ~4 tiles per run
        Gt = max(Gt, 1LL);
        const long long W = (tail + Gt - 1) / Gt;
        long long fbeg = 0, f1 = 0;
        if (tail > 0 && (long long)blockIdx.x < Gt) {
            fbeg = (long long)blockIdx.x * W;
            f1 = min(tail, fbeg + W);
        }
        const int n_tail = f1 > fbeg ? (int)((f1 - 1) / T - fbeg / T + 1) : 0;
        if (tail > 0) nseg_max = (int)((T + W - 1) / W) + 1;
        nseg = T > 0 ? R + n_tail : 0;
        if (threadIdx.x == 0) {
            plan.R = R; plan.Gc = gridDim.x; plan.c = blockIdx.x; plan.T = T; plan.gbase = R * (int)gridDim.x;
            plan.n_tail = n_tail; plan.fbeg = fbeg; plan.f1 = f1; plan.W = W;
        }
    }
    if (nseg == 0) return;
    if (blockIdx.x == 0 && threadIdx.x == 0) *P.d_ns = (unsigned long long)min(nseg_max, P.ns_cap);

    // ---- setup: barriers, TMEM, per-range constants, the resident range operand
    TC_TR_CTA(30);
    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            tmbar_init(&full[s], 1);
            tmbar_init(&empty[s], 1);
        }
        for (int b = 0; b < NBUF; ++b) {
            tmbar_init(&tfull[b], 1);
            tmbar_init(&tempty[b], 4 * Cf::EWG);
        }
        for (int b = 0; b < 2 * Cf::BBUF; ++b) tmbar_init(&bbar[b], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(sTmem)),
                     "r"(kTmemCols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (threadIdx.x < 16) sHsn[threadIdx.x] = threadIdx.x < P.nsp ? -__double2float_rn(0.5 * P.spos[threadIdx.x]) : 0.f;
    for (int i = threadIdx.x; i < Cf::XQ; i += blockDim.x) sXSeq[i] = 0u;
    if (threadIdx.x < 3) sXCtl[threadIdx.x] = 0u;
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *sTmem;

    if (warp == FIC_PROD_WARP) {
        // ================= producer: one lane issues every bulk copy in order -- each segment's
        // range operand (once the MMAs of the segment BBUF earlier released its buffer) and the A
        // stages (stage / phase carried incrementally; the (tile, chunk) stages of a segment are
        // contiguous in the pool)
        if (lane == 0) {
            int s = 0;
            uint32_t ph = 0;
            int i = 0;
            for (int k = 0; k < nseg; ++k) {
                int grp, ta, ntl, slot;
                bool lastseg;
                plan_segment(&plan, k, grp, ta, ntl, slot, lastseg);
                const int kb = k % Cf::BBUF;
                if (k >= Cf::BBUF) tmbar_wait(&bbar[Cf::BBUF + kb], (uint32_t)(((k / Cf::BBUF) - 1) & 1));
                tmbar_expect_tx(&bbar[kb], Cf::B_BYTES);
                tbulk_g2s(sB + kb * Cf::B_BYTES, P.Bop + (size_t)grp * Cf::B_BYTES, Cf::B_BYTES, &bbar[kb]);
                const uint8_t *src = P.Dtc + (size_t)ta * CH * Cf::STAGE_BYTES;
                for (int c = 0; c < ntl * CH; ++c, ++i) {
#if FIC_PROD_NS
                    if (i >= STAGES) tmbar_wait_sleep(&empty[s], ph ^ 1u, FIC_PROD_NS);
#else
                    if (i >= STAGES) tmbar_wait(&empty[s], ph ^ 1u);
#endif
                    tmbar_expect_tx(&full[s], Cf::STAGE_BYTES);
                    TC_TR(0, i);
                    tbulk_g2s(sA + s * Cf::STAGE_BYTES, src, Cf::STAGE_BYTES, &full[s]);
                    src += Cf::STAGE_BYTES;
                    if (++s == STAGES) { s = 0; ph ^= 1u; }
                }
            }
        }
    } else if (warp == FIC_MMA_WARP) {
        // ================= MMA issuer
        constexpr uint32_t idesc = Cf::F16 ? idesc_f16(NN) : idesc_i8(NN);
        int i = 0, tl = 0;
        const uint32_t tmem_u = __shfl_sync(0xffffffffu, tmem, 0);
        const uint32_t sA_sa = su32(sA), empty_sa = su32(empty), tfull_sa = su32(tfull);
        for (int k = 0; k < nseg; ++k) {
            int grp, ta, ntl, slot;
            bool lastseg;
            plan_segment(&plan, k, grp, ta, ntl, slot, lastseg);
            ntl = __shfl_sync(0xffffffffu, ntl, 0);
            const int kb = k % Cf::BBUF;
            tmbar_wait(&bbar[kb], (uint32_t)((k / Cf::BBUF) & 1));
            const uint32_t bbase = su32(sB + kb * Cf::B_BYTES);
            for (int tt = 0; tt < ntl; ++tt, ++tl) {
                const int buf = tl % NBUF;
                for (int ch = 0; ch < CH; ++ch, ++i) {
                    const int s = i % STAGES;
#if FIC_MMA_NS
                    tmbar_wait_sleep(&full[s], (uint32_t)((i / STAGES) & 1), FIC_MMA_NS);
                    if (lane == 0) TC_TR(1, i);
                    if (ch == 0 && tl >= NBUF) tmbar_wait_sleep(&tempty[buf], (uint32_t)(((tl / NBUF) + 1) & 1), FIC_MMA_NS);
#else
                    tmbar_wait(&full[s], (uint32_t)((i / STAGES) & 1));
                    if (lane == 0) TC_TR(1, i);
                    if (ch == 0 && tl >= NBUF) tmbar_wait(&tempty[buf], (uint32_t)(((tl / NBUF) + 1) & 1));
#endif
                    if (lane == 0 && ch == 0) TC_TR(2, tl);
                    tc_fence_after();
                    {
                        // K bytes kg of the tile: QR's q plane (kg < n) accumulates S_q at column 0
                        // of the buffer, its r plane S_r at column N, both against the same B rows;
                        // the whole warp runs this (uniform operands), one elected lane issues
                        const uint32_t a0 = sA_sa + s * Cf::STAGE_BYTES;
#pragma unroll
                        for (int kk = 0; kk < KCH / 32; ++kk) {
                            const int kg = ch * KCH + kk * 32;
                            const int plane = Cf::QR ? kg / n : 0;
                            const int kp = Cf::QR ? kg - plane * n : kg;
                            const uint32_t dcol = buf * Cf::ACC + plane * NN;
                            const uint64_t ad = smem_desc(a0 + kk * 256, 128, (KCH / 16) * 128);
                            const uint64_t bd = smem_desc(bbase + kp * 8, 128, (Cf::KB / 16) * 128);
                            if constexpr (Cf::F16) tc_mma_f16_elect(tmem_u + dcol, ad, bd, idesc, kp > 0 ? 1u : 0u);
                            else tc_mma_i8_elect(tmem_u + dcol, ad, bd, idesc, kp > 0 ? 1u : 0u);
                        }
                        tc_commit_elect(empty_sa + 8 * s);
                        if (ch == CH - 1) {
                            tc_commit_elect(tfull_sa + 8 * buf);
                            if (lane == 0) TC_TR(3, tl);
                        }
                    }
                }
            }
            tc_commit_elect(su32(&bbar[Cf::BBUF + kb]));  // operand free once these MMAs complete
        }
    } else if (warp == Cf::XWARP) {
        // ================= exact path, off the tile pipeline: the canonical binary64 score (C7)
        // of every queued pair for every s > 0, then -- in queue order, one lane -- the
        // lexicographic first-min update of the (range, domain lane) best and the CAS-min of the
        // range's threshold.  The epilogue warps only push items, so a rare pair no longer
        // stalls its warp (and through the two-buffer TMEM ring every warp) for ~1-2k cycles.
        unsigned head = 0, n_items = 0, idle_ns = 128;
        volatile unsigned *vseq = sXSeq, *vctl = sXCtl;
        for (;;) {
            const unsigned idx = head + lane;
            const bool ready = vseq[idx & (Cf::XQ - 1)] == idx + 1;
            const unsigned rb = __ballot_sync(0xffffffffu, ready);
            const int cnt = rb == 0xffffffffu ? 32 : __ffs(~rb) - 1;  // leading ready slots
            if (cnt == 0) {
                if (vctl[2] && vctl[1] == vctl[0]) break;
                // idle: back off (items are rare; every poll takes issue slots from the epilogue
                // warps of this SMSP, which pace the whole TMEM ring)
                __nanosleep(idle_ns);
                idle_ns = min(idle_ns * 2, 2048u);
                continue;
            }
            idle_ns = 128;
            __threadfence_block();
            double eb = INFINITY;
            int32_t kjb = INT_MAX, qg = 0, mm = 0, dd = 0;
            if (lane < cnt) {
                const XItem it = sXQ[idx & (Cf::XQ - 1)];
                qg = it.meta & 31;
                const int ks = (it.meta >> 5) & 7;
                mm = it.meta >> 8;
                dd = it.d;
                const TCRange &R = sR[qg];
                const double Bq = __dsub_rn(__dmul_rn((double)n, (double)it.mx), __dmul_rn((double)R.SR, (double)it.sd));
                const double c16 = __dmul_rn(0.0625, (double)__ldg(P.C + it.d));
                for (int jj = 0; jj < P.nsp; ++jj) {
                    const double sj = P.spos[jj];
                    const double e = __dadd_rn(__dsub_rn(R.A, __dmul_rn(__dmul_rn(0.5, sj), Bq)),
                                               __dmul_rn(__dmul_rn(sj, sj), c16));
                    const int32_t kj = (ks << 8) | P.jpos[jj];
                    if (e < eb || (e == eb && kj < kjb)) { eb = e; kjb = kj; }
                }
            }
            // the range's best is a lexicographic minimum, so the updates commute: in each pass
            // the lowest pending lane of every range updates it (distinct ranges in parallel);
            // passes = the largest number of items of one range in the batch.  This warp is the
            // only writer of sRB during a segment.
            const bool act = lane < cnt;
            const unsigned key = act ? (unsigned)(qg * Cf::RBW + (mm & (Cf::RBW - 1))) : (0x80000000u | (unsigned)lane);
            const unsigned grp = __match_any_sync(0xffffffffu, key);
            unsigned pending = __ballot_sync(0xffffffffu, act);
            while (pending) {
                const bool lead = ((pending >> lane) & 1u) && lane == __ffs(grp & pending) - 1;
                if (lead) {
                    Partial *bp = &sRB[key];
                    const Partial b = *bp;
                    if (eb < b.e || (eb == b.e && (dd < b.d || (dd == b.d && kjb < b.kj)))) {
                        Partial nb;
                        nb.e = eb; nb.d = dd; nb.kj = kjb;
                        *bp = nb;
                        const TCRange &R = sR[qg];
                        const float t = fminf(__double2float_ru(__dadd_rn(__dsub_rn(eb, R.A), R.margin)), FLT_MAX);
                        int *ti = reinterpret_cast<int *>(&sThr[qg]);
                        int old = *ti;
                        while (t < __int_as_float(old)) {
                            const int prev = atomicCAS(ti, old, __float_as_int(t));
                            if (prev == old) break;
                            old = prev;
                        }
                    }
                }
                pending &= ~__ballot_sync(0xffffffffu, lead);
                __syncwarp();
            }
            head += cnt;
            n_items += cnt;
            __syncwarp();
            if (lane == 0) {
                __threadfence_block();
                vctl[1] = head;  // the updates of items < head are visible
            }
        }
        if (lane == 0 && n_items && P.exact_count) atomicAdd(P.exact_count, (unsigned long long)n_items);
#ifdef FIC_TC_TRACE
        if (lane == 0 && blockIdx.x < 4096) { g_tc_trace[28][blockIdx.x] = n_items; g_tc_trace[27][blockIdx.x] = nseg; }
#endif
    } else {
        // ================= epilogue: lane = domain (TMEM lane), warpgroup = a quarter (third) of
        // the ranges; segment by segment (one range group each), tiles counted across segments
        const int eg = (warp - 2) >> 2;   // epilogue warpgroup
        const int lq = warp & 3;          // TMEM lane quarter accessible by this warp
        const int m = lq * 32 + lane;     // domain lane within the tile
        const int et = threadIdx.x - 64;  // epilogue thread
        // t2f rows per domain: one per s (NSP 1, 2); u = RN(1/C) (NSP 0); RN(C/16), RN(4/(C h)) (grid)
        constexpr int NT = NSP == 3 ? 2 : (NSP ? NSP : 1);
        float nhs[NT];
        // the B = 4 / 8 conversions below yield Bq / 2 and Bq / 64: fold the power of two into -s/2
        // (exact), so g = fma(nhs, bq, t2) keeps its rounding without the multiply
        // F16: g = (-(s/2) n) y + t2 with y = RN(Bq / n)
        constexpr float kBqScale = Cf::F16 ? (float)n : (B == 4 ? 2.0f : (B == 8 ? 64.0f : 1.0f));
#pragma unroll
        for (int jj = 0; jj < NT; ++jj) nhs[jj] = sHsn[jj] * kBqScale;
        static_assert(Cf::EWG <= 5, "named barriers 1..EWG (seeding) and 6 (segments) must not collide");
        auto epi_sync = [&]() { asm volatile("bar.sync 6, %0;" ::"r"(128 * Cf::EWG) : "memory"); };
        volatile unsigned *vctl = sXCtl;
        const int64_t t2row = P.n_slots;
        // fp32 filter score of one (range, domain) pair from the max over isometries of SRD_k
        // F16: mx holds the bits of the fp32 max (non-negative floats order like their bits, so
        // the VIMNMX3 max is the float max), rsr the bits of -SR, sdn = SD / n (exact)
        auto score = [&](int mx, int rsr, int32_t sd, float sdn, const float *t2) -> float {
            float bq;
            if constexpr (Cf::F16) {
                const float y = fmaf(__int_as_float(rsr), sdn, __int_as_float(mx));  // RN(Bq / n)
                bq = (NSP == 0 || NSP == 3) ? y * (float)n : y;
            } else if constexpr (NSP == 3 && B <= 8) {
                bq = (float)(n * mx - rsr * sd);  // exact int32 Bq, one RN conversion
            } else if constexpr (NSP == 3) {
                bq = (float)((long long)n * mx - (long long)rsr * sd);
            } else if constexpr (NSP == 0 && B <= 8) {
                // exact Bq in int32 (|n SRD|, |SR SD| <= 1.06e9 at B = 8), one RN conversion
                bq = (float)(n * mx - rsr * sd);
            } else if constexpr (NSP == 0) {
                // exact Bq (int64 at B = 16), one RN conversion
                bq = (float)((long long)n * mx - (long long)rsr * sd);
            } else if constexpr (B == 2) {
                // |Bq| <= sqrt(A C) < 2^22: exact int -> float by the 1.5 * 2^23 magic; the magic
                // constant itself is folded into t2 (t2f_kernel, fold), so bq = M + Bq here
                bq = __int_as_float(n * mx - rsr * sd + 0x4B400000);
            } else if constexpr (B == 4) {
                // |Bq| <= n^2 127.5 510 < 2^24: magic on Bq / 2, error <= 1 (margin); M folded
                bq = __int_as_float(((n * mx - rsr * sd) >> 1) + 0x4B400000);  // (x 2 in nhs)
            } else if constexpr (B == 8) {
                // |Bq| < 2^28: magic on Bq / 64, error <= 64 (margin); M folded
                bq = __int_as_float(((n * mx - rsr * sd) >> 6) + 0x4B400000);  // (x 64 in nhs)
            } else {
                // QR (B >= 16, one or two s): Bq exact in int64, one RN conversion (the fp32
                // product form rounded n max and SR SD separately: a margin term n 1020 SR that
                // let ~8x more pairs through to the exact path)
                bq = (float)((long long)n * mx - (long long)rsr * sd);
            }
            float g0;
            if constexpr (NSP == 3) {
                // the two grid points around s* = 4 Bq / C: x = (s* - a) / h, j0 = clamp(floor x)
                const float x = fmaf(bq, t2[1], -P.grid.aoh);
                const float j0 = fminf(fmaxf(floorf(x), 0.f), (float)(P.grid.K - 2));
                const float s0 = fmaf(j0, P.grid.h, P.grid.a);
                const float2 sv = make_float2(s0, s0 + P.grid.h);
                const float hb = -0.5f * bq;
                const float2 tt = __ffma2_rn(sv, make_float2(t2[0], t2[0]), make_float2(hb, hb));
                const float2 g2 = __fmul2_rn(sv, tt);  // s (s C/16 - Bq/2) = e_s - A
                g0 = fminf(g2.x, g2.y);
            } else if constexpr (NSP == 0) {
                g0 = -(bq * bq) * t2[0];  // >= -(Bq^2 / C)(1 + 4.04u): continuous minimum
            } else if constexpr (NSP == 2) {  // both s in one packed FFMA2 (the same two roundings)
                const float2 g2 = __ffma2_rn(make_float2(nhs[0], nhs[1]), make_float2(bq, bq), make_float2(t2[0], t2[1]));
                g0 = fminf(g2.x, g2.y);
            } else {
                g0 = fmaf(nhs[0], bq, t2[0]);
#pragma unroll
                for (int jj = 1; jj < NSP; ++jj) g0 = fminf(g0, fmaf(nhs[jj], bq, t2[jj]));
            }
            return g0;
        };
        unsigned tl = 0;  // tiles consumed by this CTA (TMEM buffer ring position)
        uint32_t tfull_sa = su32(tfull);
#ifndef FIC_OPAQUE_SA
#define FIC_OPAQUE_SA 3
#endif
        // held opaque to the compiler (FIC_OPAQUE_SA bit 0: B = 4, bit 1: B >= 8): at the register
        // ceiling it otherwise re-forms the barrier's shared address in every tile (S2UR
        // SR_CgaCtaId: ~6% of the B = 4 stall samples, 0.512 -> 0.504 ms; B = 8, with the split
        // loads, 0.154 -> 0.152 ms); tempty follows tfull
        if (FIC_OPAQUE_SA & (B == 4 ? 1 : 2)) asm volatile("" : "+r"(tfull_sa));
        const uint32_t tempty_sa = tfull_sa + 8u * NBUF;
#ifdef FIC_TC_TRACE
        long long acc_wait = 0, acc_busy = 0;  // per epilogue warp: tfull waits, tile work (cycles)
        long long acc_push = 0, n_push = 0;    // cycles in (and count of) push blocks
#endif
        for (int k = 0; k < nseg; ++k) {
            int grp, ta, ntl, slot;
            bool lastseg;
            plan_segment(&plan, k, grp, ta, ntl, slot, lastseg);
            const int r0 = grp * NR;
            // ---- segment setup: this group's range constants and thresholds (the previous
            // segment's readers of sR / sThr / sRB have passed the barrier)
            epi_sync();
            if (et == 0) TC_TR_SEG(23, k);
            if (et < NR) {
                TCRange R = P.rmeta[r0 + et];
                R.margin = tc_margin<B>(R.A, P.smax, (double)P.d_misc[1], NSP == 0 ? 1 : (NSP == 3 ? 2 : 0));
                sR[et] = R;
                Partial pb;  // s = 0 (if listed): e = A for every (domain, k) -> (A, 0, 0, j_zero)
                if (P.has_zero) { pb.e = R.A; pb.d = 0; pb.kj = P.j_zero; }
                else { pb.e = INFINITY; pb.d = INT_MAX; pb.kj = INT_MAX; }
#pragma unroll
                for (int w = 0; w < Cf::RBW; ++w) sRB[et * Cf::RBW + w] = pb;
                sSR[et] = Cf::F16 ? __float_as_int(-(float)R.SR) : R.SR;
                const float th = P.has_zero ? fminf(__double2float_ru(R.margin), FLT_MAX) : FLT_MAX;
                sThr[et] = R.valid ? th : -FLT_MAX;
                sM2[et] = fminf(__double2float_ru(2.0 * R.margin), FLT_MAX);
            }
            epi_sync();
            if (et == 0) TC_TR_SEG(20, k);
            int rSR[HALF];
#pragma unroll
            for (int q = 0; q < HALF; ++q)
                rSR[q] = (!UNEVEN || eg * HALF + q < NR)
                             ? (Cf::F16 ? __float_as_int(-(float)sR[eg * HALF + q].SR) : sR[eg * HALF + q].SR)
                             : 0;
            // per-domain data of this lane, walked tile by tile (pointers advanced, not recomputed);
            // NSP > 0 is chosen only when the level has exactly NSP values s > 0, so every row exists
            // B >= 8: a 32-bit slot index (one IMAD.WIDE per load instead of 64-bit pointer
            // arithmetic: B = 16 0.149 -> 0.146 ms, B = 8 0.284 -> 0.278); B = 4, at its 128-register
            // ceiling, keeps the advanced pointers (the index form cost it 0.706 -> 0.726)
            constexpr bool kIdx = B >= 8;
            unsigned di = (unsigned)ta * kTileD + m;
            const unsigned t2r = (unsigned)t2row;
            const int32_t *sdp = P.SD + (int64_t)ta * kTileD + m;
            const float *t2p = P.t2f + (int64_t)ta * kTileD + m;
            int32_t sd_n = kIdx ? __ldg(P.SD + di) : __ldg(sdp);
            float t2_n[NT];
#pragma unroll
            for (int jj = 0; jj < NT; ++jj) t2_n[jj] = kIdx ? __ldg(P.t2f + (di + jj * t2r)) : __ldg(t2p + jj * t2row);
            if constexpr (NSP > 0) {
                // ---- seed the thresholds from the segment's first tile: with NSP > 0, g approximates
                // min_{s > 0} e_s - A within the margin, so every range's best is <= A + min_m g +
                // margin and RU(min_m g + 2 margin) is a valid threshold -- the first tile no longer
                // sends every pair better than s = 0 to the exact path
                const unsigned buf0 = tl % NBUF;
                tmbar_wait_sa(tfull_sa + 8 * buf0, (tl / NBUF) & 1);
                if (et == 0) TC_TR_SEG(21, k);
                tc_fence_after();
                const uint32_t tb0 = tmem + ((uint32_t)(lq * 32) << 16) + buf0 * Cf::ACC + eg * HALF * 8;
                // all HALF ranges scored first, then their warp minima as interleaved butterflies,
                // then lane q (< HALF) lowers range q's threshold -- independent chains (scoring,
                // reducing and CAS-ing the ranges one after another took ~5k cycles per segment)
                float gq[HALF];
                const float sdn0 = (float)sd_n * (1.0f / (float)n);
#pragma unroll
                for (int g = 0; g < HALF / 4; ++g) {
                    if (UNEVEN && eg * HALF + g * 4 >= NR) {  // an empty group
#pragma unroll
                        for (int q4 = 0; q4 < 4; ++q4) gq[g * 4 + q4] = INFINITY;
                        continue;
                    }
                    uint32_t sv[Cf::QR ? 64 : 32];
                    tc_ld32<0>(tb0 + g * 32, sv);
                    if constexpr (Cf::QR) {
                        tc_ld32<32>(tb0 + NN + g * 32, sv);
                        tc_wait_ld();
#pragma unroll
                        for (int i = 0; i < 32; ++i) sv[i] = 4u * sv[i] + sv[32 + i];
                    } else {
                        tc_wait_ld();
                    }
#pragma unroll
                    for (int q4 = 0; q4 < 4; ++q4) {
                        const uint32_t *v = sv + q4 * 8;
                        const int mx = max(__vimax3_s32((int)v[0], (int)v[1], (int)v[2]),
                                           __vimax3_s32((int)v[3], (int)v[4], __vimax3_s32((int)v[5], (int)v[6], (int)v[7])));
                        gq[g * 4 + q4] = score(mx, rSR[g * 4 + q4], sd_n, sdn0, t2_n);
                    }
                }
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) {
#pragma unroll
                    for (int q = 0; q < HALF; ++q) gq[q] = fminf(gq[q], __shfl_xor_sync(0xffffffffu, gq[q], o));
                }
                float mine = gq[0];
#pragma unroll
                for (int q = 1; q < HALF; ++q) mine = lane == q ? gq[q] : mine;
                if (lane < HALF && (!UNEVEN || eg * HALF + lane < NR)) {
                    const int r = eg * HALF + lane;
                    const float t = fminf(__fadd_ru(mine, sM2[r]), FLT_MAX);
                    int *ti = reinterpret_cast<int *>(&sThr[r]);
                    int old = *ti;
                    while (t < __int_as_float(old)) {  // (NaN / +inf pads never lower it)
                        const int prev = atomicCAS(ti, old, __float_as_int(t));
                        if (prev == old) break;
                        old = prev;
                    }
                }
                if (et == 0) TC_TR_SEG(22, k);
                asm volatile("bar.sync %0, 128;" ::"r"(1 + eg) : "memory");  // the warpgroup's seeds
            }
            if (et == 0) TC_TR_SEG(24, k);
#ifdef FIC_EPI_UNROLL
#define FIC_STR_(x) #x
#define FIC_PRAGMA_(x) _Pragma(FIC_STR_(x))
            FIC_PRAGMA_(unroll FIC_EPI_UNROLL)
#endif
            for (int tt = 0; tt < ntl; ++tt, ++tl) {
                const unsigned buf = tl % NBUF;
                const int d = (ta + tt) * kTileD + m;
                const int32_t sd = sd_n;
                const float sdn = (float)sd * (1.0f / (float)n);  // exact (SD < 2^24, n a power of two)
                float t2[NT];
#pragma unroll
                for (int jj = 0; jj < NT; ++jj) t2[jj] = t2_n[jj];
                if constexpr (kIdx) di += kTileD;
                else { sdp += kTileD; t2p += kTileD; }
                if (tt + 1 < ntl) {  // prefetch the next tile's per-domain data
                    sd_n = kIdx ? __ldg(P.SD + di) : __ldg(sdp);
#pragma unroll
                    for (int jj = 0; jj < NT; ++jj) t2_n[jj] = kIdx ? __ldg(P.t2f + (di + jj * t2r)) : __ldg(t2p + jj * t2row);
                }
#ifdef FIC_TC_TRACE
                const long long tw0 = clock64();
#endif
                tmbar_wait_sa(tfull_sa + 8 * buf, (tl / NBUF) & 1);
#ifdef FIC_TC_TRACE
                const long long tw1 = clock64();
                acc_wait += tw1 - tw0;
#endif
                if (warp == 2 && lane == 0) TC_TR(4, tl);
                tc_fence_after();
                const uint32_t tbase = tmem + ((uint32_t)(lq * 32) << 16) + buf * Cf::ACC + eg * HALF * 8;
                // four ranges (32 columns) per tcgen05.ld, the next group in flight while one is scored
                constexpr int G = HALF / 4;
                uint32_t vv[Cf::QR ? 64 : G * 32];
                // the tile's accumulators (<= 2 groups of 4 ranges, or QR's two planes) into
                // registers, then the buffer goes straight back to the MMA warp: the next MMA into
                // it overlaps this tile's scoring

                // FIC_SPLIT_LD (bit 0: B = 4, bit 1: B = 8): each group's 32 columns loaded just
                // before it is scored, the buffer released after the last load (one group's
                // accumulators live at a time, the release later by a group's scoring): B = 8
                // 0.1555 -> 0.154 ms and no spills; at B = 4 it is what lets 4 warpgroups fit
                // (0.504 -> 0.472 ms; with 3 warpgroups alone it cost 0.504 -> 0.513)
#ifndef FIC_SPLIT_LD
#define FIC_SPLIT_LD 3
#endif
                // (bit 2: the QR form, B >= 16, with two groups -- each group's q and r planes)
                constexpr bool kSplit = (FIC_SPLIT_LD & (B == 4 ? 1 : B == 8 ? 2 : 4)) != 0 && G >= 2;
                constexpr bool kQRS = kSplit && Cf::QR;  // QR split: a group's combined sums in vv[0, 32)
                auto vgrp = [&](int q) -> const uint32_t * { return kQRS ? vv + (q & 3) * 8 : vv + q * 8; };
                static_assert(G <= 4 && (!Cf::QR || G == 1 || kQRS), "one tile's accumulators fit vv");
                if constexpr (!kSplit) {
                    tc_ld32<0>(tbase, vv);
                    if constexpr (Cf::QR) tc_ld32<32>(tbase + NN, vv);
                    if constexpr (!Cf::QR && G >= 2) if (!UNEVEN || eg * HALF + 4 < NR) tc_ld32<32>(tbase + 32, vv);
                    if constexpr (!Cf::QR && G >= 3) if (!UNEVEN || eg * HALF + 8 < NR) tc_ld32<64>(tbase + 64, vv);
                    if constexpr (!Cf::QR && G >= 4) if (!UNEVEN || eg * HALF + 12 < NR) tc_ld32<96>(tbase + 96, vv);
                    tc_wait_ld();
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) tmbar_arrive_sa(tempty_sa + 8 * buf);
                }
                if (warp == 2 && lane == 0) TC_TR(5, tl);
                if (lane == 0) TC_TR(8 + warp - 2, tl);
                if constexpr (Cf::QR && !kSplit) {  // SRD_k = 4 S_q + S_r (exact: < 2^31)
#pragma unroll
                    for (int i = 0; i < 32; ++i) vv[i] = 4u * vv[i] + vv[32 + i];
                }
                // the filter of GB ranges at a time (branch-free, their chains interleaved), then one
                // branch into the rare queueing path, which re-forms the max of each passing range
                // from the accumulators still in registers (one group of 4 ranges per branch: the whole
                // tile per branch, FIC_B4_GB=8 at B = 4, was measured slower: 0.507 -> 0.553 ms)
#ifndef FIC_B4_GB
#define FIC_B4_GB 4
#endif
                constexpr int GB = (B == 4 && FIC_B4_GB <= G * 4) ? FIC_B4_GB : 4;
                static_assert(GB % 4 == 0 && (G * 4) % GB == 0, "branch groups of whole tcgen05.ld groups");
#pragma unroll
                for (int gb = 0; gb < G * 4 / GB; ++gb) {
                if constexpr (kSplit) {
                    static_assert(GB == 4, "split loads: one group per branch group");
                    if (!UNEVEN || eg * HALF + gb * 4 < NR) {
                        if constexpr (kQRS) {
                            tc_ld32<0>(tbase + gb * 32, vv);
                            tc_ld32<32>(tbase + NN + gb * 32, vv);
                        } else {
                            if (gb == 0) tc_ld32<0>(tbase, vv);
                            else if (gb == 1) { if constexpr (G >= 2) tc_ld32<32>(tbase + 32, vv); }
                            else if (gb == 2) { if constexpr (G >= 3) tc_ld32<64>(tbase + 64, vv); }
                            else { if constexpr (G >= 4) tc_ld32<96>(tbase + 96, vv); }
                        }
                    }
                    tc_wait_ld();
                    if (gb == G - 1) {
                        tc_fence_before();
                        __syncwarp();
                        if (lane == 0) tmbar_arrive_sa(tempty_sa + 8 * buf);
                    }
                    if constexpr (kQRS) {  // SRD_k = 4 S_q + S_r (exact: < 2^31)
#pragma unroll
                        for (int i = 0; i < 32; ++i) vv[i] = 4u * vv[i] + vv[32 + i];
                    }
                }
                unsigned pm = 0;
#pragma unroll
                for (int g = gb * GB / 4; g < (gb + 1) * GB / 4; ++g) {
                    if (UNEVEN && eg * HALF + g * 4 >= NR) continue;  // an empty group
#pragma unroll
                    for (int q4 = 0; q4 < 4; ++q4) {
                        const int q = g * 4 + q4;
                        const uint32_t *v = vgrp(q);
                        const int mx = max(__vimax3_s32((int)v[0], (int)v[1], (int)v[2]),
                                           __vimax3_s32((int)v[3], (int)v[4], __vimax3_s32((int)v[5], (int)v[6], (int)v[7])));
                        // (B = 8, at its 96-register ceiling: the range sums from shared memory)
                        const float g0 = score(mx, B == 8 ? sSR[eg * HALF + q] : rSR[q], sd, sdn, t2);
                        pm |= (g0 <= sThr[eg * HALF + q]) ? (1u << q) : 0u;
                    }
                }
#ifdef FIC_TC_TRACE
                const long long tp0 = clock64();
#endif
                // (a warp-uniform branch on __any_sync instead: B = 4 0.508 -> 0.525 ms)
                if (pm) {  // queue (range, domain, k*, max SRD) of the passing pairs for the exact warp
#pragma unroll
                    for (int q = gb * GB; q < (gb + 1) * GB; ++q) {
                        if (pm >> q & 1) {
                            const uint32_t *v = vgrp(q);
                            const int mx = max(__vimax3_s32((int)v[0], (int)v[1], (int)v[2]),
                                               __vimax3_s32((int)v[3], (int)v[4], __vimax3_s32((int)v[5], (int)v[6], (int)v[7])));
                            int ks = 7;
#pragma unroll
                            for (int k = 6; k >= 0; --k)
                                if ((int)v[k] == mx) ks = k;  // lowest index attaining the max
                            // tighten the range's threshold at once from the fp32 score (the
                            // exact warp's own update, RU(e - A + margin), comes later): with
                            // NSP > 0, g approximates min_{s > 0} e_s - A within the margin, so
                            // e <= A + g + margin and RU(g + 2 margin) is a valid threshold
                            // (NSP = 0: g is only a lower bound of the grid's minimum -- no)
                            if constexpr (NSP > 0) {
                                const float g0 = score(mx, B == 8 ? sSR[eg * HALF + q] : rSR[q], sd, sdn, t2);
                                const float t = fminf(__fadd_ru(g0, sM2[eg * HALF + q]), FLT_MAX);
                                int *ti = reinterpret_cast<int *>(&sThr[eg * HALF + q]);
                                int old = *ti;
                                while (t < __int_as_float(old)) {
                                    const int prev = atomicCAS(ti, old, __float_as_int(t));
                                    if (prev == old) break;
                                    old = prev;
                                }
                            }
                            const unsigned xi = atomicAdd(&sXCtl[0], 1u);
                            while (xi - vctl[1] >= (unsigned)Cf::XQ) __nanosleep(32);  // ring full (rare)
                            XItem it;
                            it.mx = Cf::F16 ? (int)__int_as_float(mx) : mx;
                            it.d = d; it.sd = sd;
                            it.meta = (eg * HALF + q) | (ks << 5) | (m << 8);
                            sXQ[xi & (Cf::XQ - 1)] = it;
                            __threadfence_block();
                            reinterpret_cast<volatile unsigned *>(sXSeq)[xi & (Cf::XQ - 1)] = xi + 1;
                        }
                    }
                }
#ifdef FIC_TC_TRACE
                if (pm) { acc_push += clock64() - tp0; ++n_push; }
#endif
                }
                if (warp == 2 && lane == 0) TC_TR(6, tl);
                if (warp == Cf::XWARP - 1 && lane == 0) TC_TR(7, tl);
#ifdef FIC_TC_TRACE
                acc_busy += clock64() - tw1;
#endif
            }
            // ---- every queued pair of this segment has been scored by the exact warp
            epi_sync();
            if (et == 0) TC_TR_SEG(25, k);
            if (et == 0)
                while (vctl[1] != vctl[0]) __nanosleep(32);
            epi_sync();
            if (et == 0) TC_TR_SEG(26, k);
            __threadfence_block();
            if (et < NR) {  // the segment's partial of each range; the group's last segment also
                const int r = r0 + et;  // fills the unused slots
                Partial b = sRB[et * Cf::RBW];
                for (int w = 1; w < Cf::RBW; ++w) {
                    const Partial c = sRB[et * Cf::RBW + w];
                    if (c.e < b.e || (c.e == b.e && (c.d < b.d || (c.d == b.d && c.kj < b.kj)))) b = c;
                }
                if (r < n_r) {
                    P.part[(size_t)r * P.ns_cap + slot] = b;
                    if (lastseg) {
                        Partial none;
                        none.e = INFINITY; none.d = INT_MAX; none.kj = INT_MAX;
                        for (int s2 = slot + 1; s2 < nseg_max && s2 < P.ns_cap; ++s2) P.part[(size_t)r * P.ns_cap + s2] = none;
                    }
                }
            }
        }
        if (et == 0) vctl[2] = 1u;  // the exact warp may stop once the ring is empty
#ifdef FIC_TC_TRACE
        if (blockIdx.x == 0 && lane == 0) {
            g_tc_trace[29][2 * warp] = acc_busy; g_tc_trace[29][2 * warp + 1] = acc_wait;
            g_tc_trace[29][64 + 2 * warp] = acc_push; g_tc_trace[29][64 + 2 * warp + 1] = n_push;
        }
#endif
    }
    tc_fence_before();
    __syncthreads();
    TC_TR_CTA(31);
    if (warp == 0) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemCols));
    }
}

template <int B, int NSP>
static size_t tc_smem_bytes() {
    using Cf = TCfg<B>;
    return (size_t)Cf::STAGES * Cf::STAGE_BYTES + Cf::BBUF * Cf::B_BYTES + sizeof(TCRange) * Cf::NR + 4 * Cf::NR +
           4 * 16 + 4 * Cf::NR + sizeof(Partial) * Cf::NR * Cf::RBW + 8 * (2 * Cf::STAGES + 2 * Cf::NBUF + 4) + 16 +
           (sizeof(XItem) + 4) * Cf::XQ + 16 + 4 * Cf::NR + 1024;
}

template <int B, int NSP>
static cudaError_t launch_tc_t(const TCParams &p, cudaStream_t st) {
    using Cf = TCfg<B>;
    const size_t smem = tc_smem_bytes<B, NSP>();
    static std::atomic<unsigned long long> attr{0};
    if (cudaError_t e = ensure_smem_attr(tcsearch_kernel<B, NSP>, (int)smem, attr)) return e;
    // persistent: one CTA per SM of the context's device (the kernel partitions the (group, tile)
    // space itself)
    const int num_sms = p.num_sms > 0 ? p.num_sms : 148;
    int ctas = num_sms;
    if (const char *e = getenv("FIC_TC_CTAS")) ctas = std::max(1, atoi(e));  // test hook: small grids
    return launch_pdl(tcsearch_kernel<B, NSP>, dim3((unsigned)ctas), dim3(Cf::THREADS), smem, st, p);
}

template <int B>
static cudaError_t launch_tc_b(const TCParams &p, cudaStream_t st) {
    if (p.nsp <= 1) return launch_tc_t<B, 1>(p, st);
    if (p.nsp <= 2) return launch_tc_t<B, 2>(p, st);
    if (p.grid.on) return launch_tc_t<B, 3>(p, st);
    return launch_tc_t<B, 0>(p, st);
}

int tc_ranges_per_cta(int B) {
    return B == 32 ? TCfg<32>::NR : B == 16 ? TCfg<16>::NR : (B == 4 ? TCfg<4>::NR : TCfg<8>::NR);
}

size_t tc_range_bytes(int B, int64_t n_r) {
    switch (B) {
    case 4: return (size_t)((n_r + TCfg<4>::NR - 1) / TCfg<4>::NR) * (TCfg<4>::B_BYTES + TCfg<4>::NR * sizeof(TCRangeG));
    case 8: return (size_t)((n_r + TCfg<8>::NR - 1) / TCfg<8>::NR) * (TCfg<8>::B_BYTES + TCfg<8>::NR * sizeof(TCRangeG));
    case 16: return (size_t)((n_r + TCfg<16>::NR - 1) / TCfg<16>::NR) * (TCfg<16>::B_BYTES + TCfg<16>::NR * sizeof(TCRangeG));
    case 32: return (size_t)((n_r + TCfg<32>::NR - 1) / TCfg<32>::NR) * (TCfg<32>::B_BYTES + TCfg<32>::NR * sizeof(TCRangeG));
    default: return 0;
    }
}

// the operand and the moments of a level's ranges (scratch: [groups][B_BYTES] operand, then the
// [groups * NR] moments); launch = false only derives the pointers (prepared ahead)
template <int B>
static cudaError_t tc_range_prep(const uint8_t *img, int32_t N, const int2 *ranges, const unsigned long long *d_nr,
                                 int64_t n_r, uint8_t *scratch, TCParams &p, cudaStream_t st, bool launch) {
    using Cf = TCfg<B>;
    const int64_t groups = (n_r + Cf::NR - 1) / Cf::NR;
    uint8_t *Bop = scratch;
    TCRangeG *meta = reinterpret_cast<TCRangeG *>(scratch + (size_t)groups * Cf::B_BYTES);
    p.Bop = Bop;
    p.rmeta = meta;
    if (!launch) return cudaSuccess;
    const int64_t total16 = groups * Cf::N * (Cf::KB / 16);
    const int n_pad = (int)(groups * Cf::NR);
    const int64_t meta_threads = (int64_t)n_pad * (B >= 8 ? 32 : 1);
    const int nb_op = (int)((total16 + 255) / 256), nb_meta = (int)((meta_threads + 255) / 256);
    if (cudaError_t e = launch_pdl(tc_range_prep_kernel<B>, dim3((unsigned)(nb_op + nb_meta)), dim3(256), 0, st,
                                   img, N, ranges, d_nr, total16, Bop, nb_op, n_pad, 0.0,
                                   (const unsigned long long *)nullptr, meta, (int32_t)0))
        return e;
    return cudaGetLastError();
}

cudaError_t launch_tc_prep(int32_t B, const uint8_t *img, int32_t N, const int2 *ranges,
                           const unsigned long long *d_nr, int64_t n_r, uint8_t *scratch, cudaStream_t st) {
    if (n_r == 0) return cudaSuccess;
    TCParams p;
    switch (B) {
    case 4: return tc_range_prep<4>(img, N, ranges, d_nr, n_r, scratch, p, st, true);
    case 8: return tc_range_prep<8>(img, N, ranges, d_nr, n_r, scratch, p, st, true);
    case 16: return tc_range_prep<16>(img, N, ranges, d_nr, n_r, scratch, p, st, true);
    case 32: return tc_range_prep<32>(img, N, ranges, d_nr, n_r, scratch, p, st, true);
    default: return cudaErrorInvalidValue;
    }
}

#ifdef FIC_TC_TRACE
extern "C" int fic_debug_tc_trace(long long *h_out) {  // [32][4096], then zeroed on the device
    cudaError_t e = cudaMemcpyFromSymbol(h_out, g_tc_trace, sizeof(long long) * 32 * 4096);
    static long long zero[32][4096];
    if (e == cudaSuccess) e = cudaMemcpyToSymbol(g_tc_trace, zero, sizeof zero);
    return (int)e;
}
#endif

cudaError_t launch_tc_search(int32_t B, const SearchParams &sp, const uint8_t *Dtc, int64_t n_slots,
                             uint8_t *scratch, cudaStream_t st) {
    if (sp.n_r == 0 || sp.nsp == 0) return cudaSuccess;
    TCParams p;
    memset(&p, 0, sizeof p);
    cudaError_t e0 = cudaSuccess;
    const bool launch = !sp.prep_done;
    switch (B) {
    case 4: e0 = tc_range_prep<4>(sp.img, sp.N, sp.ranges, sp.d_nr, sp.n_r, scratch, p, st, launch); break;
    case 8: e0 = tc_range_prep<8>(sp.img, sp.N, sp.ranges, sp.d_nr, sp.n_r, scratch, p, st, launch); break;
    case 16: e0 = tc_range_prep<16>(sp.img, sp.N, sp.ranges, sp.d_nr, sp.n_r, scratch, p, st, launch); break;
    case 32: e0 = tc_range_prep<32>(sp.img, sp.N, sp.ranges, sp.d_nr, sp.n_r, scratch, p, st, launch); break;
    default: return cudaErrorInvalidValue;
    }
    if (e0 != cudaSuccess) return e0;
    p.img = sp.img; p.N = sp.N; p.ranges = sp.ranges; p.n_r = sp.n_r;
    p.Dtc = Dtc; p.SD = sp.SD; p.C = sp.C; p.t2f = sp.t2f; p.n_slots = n_slots;
    p.d_nr = sp.d_nr; p.d_misc = sp.d_misc; p.nsplit = sp.nsplit; p.n_slots = sp.slot_stride;
    p.d_ns = sp.d_ns; p.ns_cap = sp.ns_cap;
    p.nsp = sp.nsp;
    memcpy(p.spos, sp.spos, sizeof p.spos);
    memcpy(p.jpos, sp.jpos, sizeof p.jpos);
    p.has_zero = sp.has_zero; p.j_zero = sp.j_zero;
    p.smax = sp.smax;
    p.part = sp.part; p.exact_count = sp.exact_count;
    p.num_sms = sp.num_sms;
    p.grid = sp.grid;
    p.lockstep = tc_pool_bytes(B, (n_slots + kTileD - 1) / kTileD) > ((size_t)48 << 20) ? 1 : 0;
    if (const char *e = getenv("FIC_TC_LOCKSTEP")) p.lockstep = atoi(e) != 0;  // test hook
    switch (B) {
    case 4: return launch_tc_b<4>(p, st);
    case 8: return launch_tc_b<8>(p, st);
    case 16: return launch_tc_b<16>(p, st);
    case 32: return launch_tc_b<32>(p, st);
    default: return cudaErrorInvalidValue;
    }
}

// Partial-slot sizing for the persistent search: the level's ns_cap (4 x this hint, at most the
// tile count) bounds the runs a range group can be cut into (SegPlan), so the flattened tail
// can spread a few groups over every SM; the actual slot count is decided on the device.
int tc_nsplit_hint(int32_t B, int64_t n_r, int64_t n_tiles, int num_sms) {
    const int64_t nr = tc_ranges_per_cta(B);
    const int64_t gx = (n_r + nr - 1) / nr;
    if (gx <= 0 || n_tiles <= 0) return 1;
    int64_t ns = ((int64_t)num_sms * 2 + gx - 1) / gx;
    const int64_t max_ns = (n_tiles + 3) / 4;  // at least ~4 tiles per run
    if (ns > max_ns) ns = max_ns;
    if (ns < 1) ns = 1;
    if (ns > 65535) ns = 65535;
    return (int)ns;
}

}  // namespace fic
