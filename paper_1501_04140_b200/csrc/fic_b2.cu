// fic_b2.cu -- the B = 2 level (4-pixel ranges, the largest level by pair count) on CUDA cores,
// from a closed form of the maximum over the 8 isometries.
//
// For B = 2 every pixel lies in one D4 orbit (the 4 corners).  With the corners in cyclic order
// (TL, TR, BR, BL) = (a, b, c, d) for the range and (w, x, y, z) for the decimated domain D',
// the 4-point DFT diagonalises the rotations and conjugates under the mirrors, which gives
// (verified exhaustively in tests against the oracle and by scripts):
//   max_k Bq_k = max( X2 Y2 + xr2 yr + xi2 yi ,  -X2 Y2 + xr2 yi + xi2 yr )
//              = ( (xr2 + xi2)(yr + yi) + | 2 X2 Y2 + (xr2 - xi2)(yr - yi) | ) / 2      (4 flops)
//   X2 = a - b + c - d,  xr2 = 2|a - c|,  xi2 = 2|b - d|      (range features)
//   Y2 = w - x + y - z,  yr = |w - y|,    yi = |x - z|        (domain features)
// with Bq_k = n SRD_k - SR SD (n = 4).  Every product and sum is an integer below 2^24, so the
// fp32 evaluation is exact.  The score filter and the exact path follow fic_tc.cu's: an fp32 lower bound of every binary64 score with a rigorous margin; surviving pairs are
// re-scored exactly (all 8 SRD_k in integers, canonical binary64 Eq. 1/3, lexicographic
// first-min).  Result identical to the oracle's exhaustive loop.
#include <cfloat>
#include <climits>
#include <cmath>
#include <cstdlib>
#include <cstring>

#include <cub/device/device_radix_sort.cuh>

#include "fic_internal.cuh"

namespace fic {

__device__ __forceinline__ uint32_t b2_su32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void b2_bar_init(uint64_t *bar) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b2_su32(bar)) : "memory");
}
__device__ __forceinline__ void b2_expect(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b2_su32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void b2_bulk(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            b2_su32(dst)),
        "l"(src), "r"(bytes), "r"(b2_su32(bar))
        : "memory");
}
__device__ __forceinline__ void b2_wait(uint64_t *bar, uint32_t parity) {
    uint32_t done = 0;
    while (!done) {
        asm volatile(
            "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
            : "=r"(done)
            : "r"(b2_su32(bar)), "r"(parity)
            : "memory");
    }
}

// Domain features: float4 (Y2, yr + yi, yr - yi, C) per slot; zero on pads (t2 = +inf excludes
// them).  The pool is stored sorted by C (stable: ties keep the kept-domain rank order), with
// ds[pos] = kept-domain rank and Cs[pos] = C, so the search can bound a range's admissible
// domains to C windows (Cauchy-Schwarz, see b2win_kernel).
// also the pool moments of the level (SD, SDf, C, Cmax; pool_moments_kernel is not run for B = 2)
__global__ void __launch_bounds__(256) b2_pool_kernel(const uint8_t *__restrict__ img, int32_t N, int32_t L, int32_t A,
                                                      const int32_t *__restrict__ kept,
                                                      const unsigned long long *__restrict__ d_nk, int64_t n_slots,
                                                      float4 *__restrict__ F, uint32_t *__restrict__ key,
                                                      int32_t *__restrict__ val, int32_t *__restrict__ SD,
                                                      float *__restrict__ SDf, int64_t *__restrict__ Cm,
                                                      unsigned long long *d_cmax) {
    const int64_t d = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t n_k = (int64_t)*d_nk;
    unsigned long long cm = 0;  // (no early return: block_max_atomic)
    if (d < n_slots) {
        val[d] = (int32_t)d;
        if (d >= n_k) {
            F[d] = make_float4(0.f, 0.f, 0.f, 0.f);
            key[d] = 0xffffffu;  // pads sort last (C < 2^23)
            SD[d] = 0; SDf[d] = 0.f; Cm[d] = 0;
        } else {
            const int32_t c = kept[d];
            const int64_t x0 = (int64_t)(c % A) * L, y0 = (int64_t)(c / A) * L;
            auto dp = [&](int i, int j) {
                const uint8_t *q = img + (y0 + 2 * i) * N + x0 + 2 * j;
                return (int)q[0] + (int)q[1] + (int)q[N] + (int)q[N + 1];
            };
            const int w = dp(0, 0), x = dp(0, 1), y = dp(1, 1), z = dp(1, 0);
            const int sd = w + x + y + z;
            const int cc = 4 * (w * w + x * x + y * y + z * z) - sd * sd;  // C = n SDD - SD^2 < 2^23
            const int yr = abs(w - y), yi = abs(x - z);
            F[d] = make_float4((float)(w - x + y - z), (float)(yr + yi), (float)(yr - yi), (float)cc);
            key[d] = (uint32_t)cc;
            SD[d] = sd; SDf[d] = (float)sd; Cm[d] = cc;
            cm = (unsigned long long)cc;
        }
    }
    block_max_atomic(cm, d_cmax);
}

__global__ void b2_gather_kernel(const float4 *__restrict__ Fu, const int32_t *__restrict__ ds, int64_t n_slots,
                                 float4 *__restrict__ F) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n_slots) F[i] = Fu[ds[i]];
}

// Coarse index of the C-sorted pool: ctab[t] = first sorted position whose C (as fp32) is
// >= (t dl)^2, dl = sqrt(Cmax) / n_tab -- monotone in t; b2wink_kernel starts its frontiers
// there instead of binary-searching every window centre
__global__ void b2_ctab_kernel(const int32_t *__restrict__ Cs, const unsigned long long *__restrict__ d_nk,
                               const unsigned long long *__restrict__ d_cmax, int32_t *__restrict__ ctab,
                               int32_t n_tab) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n_tab) return;
    const int n = (int)*d_nk;
    const float dl = sqrtf((float)*d_cmax) / (float)n_tab;
    const float v = ((float)t * dl) * ((float)t * dl);
    int lo = 0, hi = n;
    while (lo < hi) {
        const int m = (lo + hi) >> 1;
        if ((float)__ldg(Cs + m) >= v) hi = m;
        else lo = m + 1;
    }
    ctab[t] = lo;
}

struct B2PoolLayout {
    size_t F, Fu, Cs, key, ds, val, ctab, tmp, tmp_bytes, total;
};
static B2PoolLayout b2_layout(int64_t slots) {
    B2PoolLayout L;
    auto al = [](size_t x) { return (x + 255) & ~(size_t)255; };
    size_t o = 0;
    L.F = o; o += al(sizeof(float4) * slots);
    L.Fu = o; o += al(sizeof(float4) * slots);
    L.Cs = o; o += al(sizeof(uint32_t) * slots);
    L.key = o; o += al(sizeof(uint32_t) * slots);
    L.ds = o; o += al(sizeof(int32_t) * slots);
    L.val = o; o += al(sizeof(int32_t) * slots);
    L.ctab = o; o += al(sizeof(int32_t) * b2_ctab_entries(slots));
    L.tmp_bytes = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, L.tmp_bytes, (const uint32_t *)nullptr, (uint32_t *)nullptr,
                                    (const int32_t *)nullptr, (int32_t *)nullptr, (int)slots, 0, 24);
    L.tmp = o; o += al(L.tmp_bytes);
    L.total = o;
    return L;
}

size_t b2_pool_bytes(int64_t n_slots) { return b2_layout(n_slots).total; }

cudaError_t launch_b2_pool(const uint8_t *img, int32_t N, int32_t L, int32_t A, const int32_t *kept,
                           const unsigned long long *d_nk, int64_t n_slots, void *store, B2Pool *out,
                           int32_t *SD, float *SDf, int64_t *C, unsigned long long *d_cmax, cudaStream_t st) {
    const B2PoolLayout Ly = b2_layout(n_slots);
    char *base = static_cast<char *>(store);
    out->F = reinterpret_cast<float4 *>(base + Ly.F);
    out->Cs = reinterpret_cast<int32_t *>(base + Ly.Cs);
    out->ds = reinterpret_cast<int32_t *>(base + Ly.ds);
    out->ctab = reinterpret_cast<int32_t *>(base + Ly.ctab);
    out->ctab_n = b2_ctab_entries(n_slots);
    if (n_slots == 0) return cudaSuccess;
    float4 *Fu = reinterpret_cast<float4 *>(base + Ly.Fu);
    uint32_t *key = reinterpret_cast<uint32_t *>(base + Ly.key);
    int32_t *val = reinterpret_cast<int32_t *>(base + Ly.val);
    const unsigned g = (unsigned)((n_slots + 255) / 256);
    b2_pool_kernel<<<g, 256, 0, st>>>(img, N, L, A, kept, d_nk, n_slots, Fu, key, val, SD, SDf, C, d_cmax);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    size_t tb = Ly.tmp_bytes;
    e = cub::DeviceRadixSort::SortPairs(base + Ly.tmp, tb, key, reinterpret_cast<uint32_t *>(out->Cs), val, out->ds,
                                        (int)n_slots, 0, 24, st);
    if (e != cudaSuccess) return e;
    b2_gather_kernel<<<g, 256, 0, st>>>(Fu, out->ds, n_slots, out->F);
    b2_ctab_kernel<<<(unsigned)(out->ctab_n / 256), 256, 0, st>>>(out->Cs, d_nk, d_cmax, out->ctab, out->ctab_n);
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------------------------
// Search, in two passes.
//
// Pass 1 (b2scan_kernel) is the data-parallel bulk of the level: a thread owns kB2RPT ranges
// (registers, packed pairs, so the arithmetic issues as FFMA2/FMUL2: two fp32 FMAs per
// fma-pipe slot), the CTA streams its split's domain features through shared memory
// (cp.async.bulk, kB2NB buffers, released by the last warp -- no CTA barrier).  Per
// (range, domain) it is 5 fp32 FMA lanes + one FMNMX3 and no branch:
//     Q  = X2 Y2 + dx z,  bq = sx y + |Q|                       (= 2 max_k Bq_k, exact)
//     g_j = -(s_j/4) bq + t2_j   (j packed in pairs)            (fp32 lower bound of e_j - A)
//     gmin = min(gmin, g_j ...)
// and it stores gmin per (range, split).  |g_j - (e_j - A)| <= margin for every pair, so
//     thr = RU(min_splits gmin + 2 margin) >= best - A + margin
// and a pair with g > thr can neither win nor tie.
//
// Pass 2 (b2exact_kernel), one warp per range: only the splits with gmin <= thr can hold such a
// pair (usually the winner's split alone); the warp rescans them with the same fp32 arithmetic,
// sends every pair with g <= thr to the canonical binary64 score, and reduces the lexicographic
// first minimum (e; d, k, j) over its lanes.  The result equals the exhaustive loop.
struct B2Params {
    const uint8_t *img;
    int32_t N, L, A;
    const int2 *ranges;
    int32_t n_r;
    const float4 *F;       // [n_slots] (Y2, yr + yi, yr - yi, C), sorted by C
    const float *T;        // [n_slots][tw] t2_j = RN((s_j s_j)(C/16)), +inf on pads (sorted order)
    const int32_t *Cs;     // [n_slots] C (sorted)
    const int32_t *ds;     // [n_slots] kept-domain rank of each sorted position
    const int32_t *ctab;   // [ctab_n] coarse index of Cs (b2_ctab_kernel)
    int32_t ctab_n;
    int32_t tw;
    SGrid grid;  // uniform grid of the positive s: NP = 0 kernels, T = (RN(C/16), RN(2 / (C h)))
    const int32_t *kept;
    const unsigned long long *d_nr, *d_misc;  // device sizes: n_r; n_kept, Cmax
    int32_t nsplit;
    int32_t nsp;
    double spos[kMaxS];
    float nhs[kMaxS];  // -RN(s_j / 4) (host-rounded, identical to the device conversion)
    int32_t jpos[kMaxS];
    int32_t has_zero, j_zero;
    double smax;
    Partial *part;
    unsigned long long *exact_count;
    float *gmin;                    // [n_r][ns_cap] pass-1 minimum of g per (range, split)
    unsigned long long *d_nscan;    // splits pass 1 used
    unsigned long long *d_ns;       // splits of the partials finalize merges (= 1 here)
    unsigned long long *scan_count; // (range, domain) pairs evaluated by the fp32 filter
    int32_t ns_cap;
};

constexpr int kB2Threads = 256;
constexpr int kB2RPT = 8;  // ranges per thread (4 packed pairs)
constexpr int kB2NB = 3;   // stage buffers
constexpr int kB2Unroll = 4;

// filter margin of one range (e units): |Bq| <= sqrt(A C); fp32 -hs and t2 roundings and one
// FFMA -> 4u (hs |Bq| + t2)
__device__ __forceinline__ double b2_margin(double A, double smax, double cmax, bool grid = false) {
    const double u = 5.9604644775390625e-08;
    const double hs = 0.5 * smax, t2m = smax * smax * cmax * 0.0625;
    // grid: g(s) = s (s RN(C/16) - bq/4) at fp32 grid points s = fma(j, h, a) -- the s rounding
    // (and the 1e-12 grid fit), C/16, FFMA and FMUL roundings: <= ~6u (hs |Bq| + 2 t2)
    return (grid ? 16.0 : 4.0) * u * (hs * sqrt(A * cmax) * 1.01 + t2m) + 1e-12 * (A + t2m) + 1e-30;
}

// fp32 score of the uniform grid's two points around s* = 4 Bq / C (bq = 2 Bq here): the pair
// brackets the nearest grid point, so min of the two = min_j (e_j - A) within the margin
__device__ __forceinline__ float b2_grid_g(const SGrid &G, float bq, float c16, float ug) {
    const float x = fmaf(bq, ug, -G.aoh);
    const float j0 = fminf(fmaxf(floorf(x), 0.f), (float)(G.K - 2));
    const float s0 = fmaf(j0, G.h, G.a), s1 = s0 + G.h;
    const float hb = -0.25f * bq;
    return fminf(s0 * fmaf(s0, c16, hb), s1 * fmaf(s1, c16, hb));
}

__device__ __forceinline__ float2 b2_bc(float v) { return make_float2(v, v); }

// range features from the 4 pixels a, b, c, d (TL, TR, BR, BL)
struct B2Range {
    float x2, dx, sx;  // 2 X2, xr2 - xi2, xr2 + xi2
    int32_t A;         // n SRR - SR^2
};
__device__ __forceinline__ B2Range b2_range(int a, int b, int c, int d) {
    B2Range R;
    R.x2 = (float)(2 * (a - b + c - d));
    R.sx = (float)(2 * abs(a - c) + 2 * abs(b - d));
    R.dx = (float)(2 * abs(a - c) - 2 * abs(b - d));
    const int sr = a + b + c + d, srr = a * a + b * b + c * c + d * d;
    R.A = 4 * srr - sr * sr;
    return R;
}

// NP = pairs of s values (1, 8 or 16), each filtered one by one.  (The s-independent bound of
// tcsearch_kernel<B, 0> would not give the pass-2 threshold below: that needs |g - (e - A)| <=
// margin, which only the per-s filter has.)
template <int NP>
__global__ void __launch_bounds__(kB2Threads, 3) b2scan_kernel(const __grid_constant__ B2Params P) {
    constexpr int RPT = kB2RPT, NB = kB2NB, TW = NP == 0 ? 2 : 2 * NP;
    constexpr int TPS = NP == 1 ? 2 : 1;  // tiles per stage
    constexpr int SDOM = TPS * kTileD;    // domains per stage
    constexpr int NWARP = kB2Threads / 32;
    extern __shared__ __align__(128) unsigned char smem[];
    float4 *Fs = reinterpret_cast<float4 *>(smem);         // [NB][SDOM]
    float *Ts = reinterpret_cast<float *>(Fs + NB * SDOM);  // [NB][SDOM][TW]
    uint64_t *full = reinterpret_cast<uint64_t *>(Ts + NB * SDOM * TW);
    int *relcnt = reinterpret_cast<int *>(full + NB);

    const int n_r = (int)*P.d_nr;
    const int n_tiles = (int)((P.d_misc[0] + kTileD - 1) / kTileD);
    int group, split, ns;
    if (!cta_work(n_r, kB2Threads * RPT, n_tiles, 2 * TPS, P.ns_cap, group, split, ns)) return;
    if (group == 0 && split == 0 && threadIdx.x == 0) *P.d_nscan = (unsigned long long)ns;
    const int t0 = (int)(((int64_t)split * n_tiles) / ns);
    const int t1 = (int)(((int64_t)(split + 1) * n_tiles) / ns);
    const int nstages = (max(0, t1 - t0) + TPS - 1) / TPS;
    auto issue = [&](int s) {
        const int b = s % NB;
        const int ta = t0 + s * TPS, tb = min(t1, ta + TPS);
        const uint32_t b1 = (uint32_t)(tb - ta) * kTileD * 16;
        const uint32_t b2 = (uint32_t)(tb - ta) * kTileD * TW * 4;
        b2_expect(&full[b], b1 + b2);
        b2_bulk(Fs + b * SDOM, P.F + (size_t)ta * kTileD, b1, &full[b]);
        b2_bulk(Ts + b * SDOM * TW, P.T + (size_t)ta * kTileD * TW, b2, &full[b]);
    };
    if (threadIdx.x == 0) {
        for (int b = 0; b < NB; ++b) {
            b2_bar_init(&full[b]);
            relcnt[b] = 0;
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0)
        for (int s = 0; s < NB && s < nstages; ++s) issue(s);

    // ranges of this thread: r = group * threads * RPT + q * threads + tid (coalesced per q)
    const int rg0 = group * kB2Threads * RPT + threadIdx.x;
    float2 X[RPT / 2], DX[RPT / 2], SX[RPT / 2];
    float gm[RPT];
#pragma unroll
    for (int q = 0; q < RPT; ++q) {
        const int r = rg0 + q * kB2Threads;
        int a = 0, b = 0, c = 0, d = 0;
        if (r < n_r) {
            const int2 rr = P.ranges[r];
            const uint8_t *p0 = P.img + (size_t)rr.y * P.N + rr.x;
            a = p0[0]; b = p0[1]; d = p0[P.N]; c = p0[P.N + 1];
        }
        const B2Range R = b2_range(a, b, c, d);
        if (q & 1) { X[q / 2].y = R.x2; SX[q / 2].y = R.sx; DX[q / 2].y = R.dx; }
        else { X[q / 2].x = R.x2; SX[q / 2].x = R.sx; DX[q / 2].x = R.dx; }
        gm[q] = INFINITY;
    }
    float2 nh[NP == 0 ? 1 : NP];  // -(s_j / 4) (times 2 max Bq); zero on pads (t2 = +inf there)
#pragma unroll
    for (int jp = 0; jp < NP; ++jp) {
        nh[jp].x = 2 * jp < P.nsp ? P.nhs[2 * jp] : 0.f;
        nh[jp].y = 2 * jp + 1 < P.nsp ? P.nhs[2 * jp + 1] : 0.f;
    }

    for (int s = 0; s < nstages; ++s) {
        const int b = s % NB;
        b2_wait(&full[b], (uint32_t)((s / NB) & 1));
        const float4 *Fb = Fs + b * SDOM;
        const float *Tb = Ts + b * SDOM * TW;
        const int nd = min(t1 - (t0 + s * TPS), TPS) * kTileD;
#pragma unroll kB2Unroll
        for (int dl = 0; dl < nd; ++dl) {
            const float4 f = Fb[dl];
            float2 t2[NP == 0 ? 1 : NP];
#pragma unroll
            for (int jp = 0; jp < (NP == 0 ? 1 : NP); ++jp) t2[jp] = reinterpret_cast<const float2 *>(Tb + dl * TW)[jp];
#pragma unroll
            for (int p = 0; p < RPT / 2; ++p) {
                float2 Q = __fmul2_rn(DX[p], b2_bc(f.z));
                Q = __ffma2_rn(X[p], b2_bc(f.x), Q);
                const float2 bq = __ffma2_rn(SX[p], b2_bc(f.y), make_float2(fabsf(Q.x), fabsf(Q.y)));
                if constexpr (NP == 0) {  // uniform grid: the two points around s*, packed over the range pair
                    const float2 x = __ffma2_rn(bq, b2_bc(t2[0].y), b2_bc(-P.grid.aoh));
                    const float jx = fminf(fmaxf(floorf(x.x), 0.f), (float)(P.grid.K - 2));
                    const float jy = fminf(fmaxf(floorf(x.y), 0.f), (float)(P.grid.K - 2));
                    const float2 s0 = __ffma2_rn(make_float2(jx, jy), b2_bc(P.grid.h), b2_bc(P.grid.a));
                    const float2 s1 = __fadd2_rn(s0, b2_bc(P.grid.h));
                    const float2 hb = __fmul2_rn(bq, b2_bc(-0.25f));
                    const float2 g0 = __fmul2_rn(s0, __ffma2_rn(s0, b2_bc(t2[0].x), hb));
                    const float2 g1 = __fmul2_rn(s1, __ffma2_rn(s1, b2_bc(t2[0].x), hb));
                    gm[2 * p] = fminf(gm[2 * p], fminf(g0.x, g1.x));
                    gm[2 * p + 1] = fminf(gm[2 * p + 1], fminf(g0.y, g1.y));
                }
#pragma unroll
                for (int jp = 0; jp < NP; ++jp) {
                    const float2 g0 = __ffma2_rn(nh[jp], b2_bc(bq.x), t2[jp]);
                    const float2 g1 = __ffma2_rn(nh[jp], b2_bc(bq.y), t2[jp]);
                    gm[2 * p] = fminf(gm[2 * p], fminf(g0.x, g0.y));
                    gm[2 * p + 1] = fminf(gm[2 * p + 1], fminf(g1.x, g1.y));
                }
            }
        }
        // release the buffer: the last warp to finish it refills it (no CTA-wide barrier)
        __syncwarp();
        if ((threadIdx.x & 31) == 0) {
            __threadfence_block();
            const int old = atomicAdd(&relcnt[b], 1);
            if (old == NWARP - 1) {
                relcnt[b] = 0;
                __threadfence_block();
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                if (s + NB < nstages) issue(s + NB);
            }
        }
    }
#pragma unroll
    for (int q = 0; q < RPT; ++q) {
        const int r = rg0 + q * kB2Threads;
        if (r < n_r) P.gmin[(size_t)r * P.ns_cap + split] = gm[q];
    }
}

// k* of one (range, domain): all 8 SRD_k in integers (isometry convention of the oracle,
// reading R2), lowest index of the maximum.  Only the rare zero-s tie needs it in the search;
// otherwise finalize resolves it for the winner (kPendIso).
__device__ __noinline__ int b2_kstar(const B2Params &P, int2 rr, int32_t d) {
    const int32_t c = P.kept[d];
    const int64_t x0 = (int64_t)(c % P.A) * P.L, y0 = (int64_t)(c / P.A) * P.L;
    int D[2][2];
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j) {
            const uint8_t *q = P.img + (y0 + 2 * i) * P.N + x0 + 2 * j;
            D[i][j] = (int)q[0] + (int)q[1] + (int)q[P.N] + (int)q[P.N + 1];
        }
    const uint8_t *p0 = P.img + (size_t)rr.y * P.N + rr.x;
    const int R[2][2] = {{p0[0], p0[1]}, {p0[P.N], p0[P.N + 1]}};
    // f_k(i,j) for B = 2 (b = 1): 0 (i,j) 1 (1-j,i) 2 (1-i,1-j) 3 (j,1-i) 4 (i,1-j) 5 (j,i) 6 (1-i,j) 7 (1-j,1-i)
    int best = INT_MIN, ks = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        int s = 0;
#pragma unroll
        for (int i = 0; i < 2; ++i)
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                int si = i, sj = j;
                switch (k) {
                case 1: si = 1 - j; sj = i; break;
                case 2: si = 1 - i; sj = 1 - j; break;
                case 3: si = j; sj = 1 - i; break;
                case 4: si = i; sj = 1 - j; break;
                case 5: si = j; sj = i; break;
                case 6: si = 1 - i; sj = j; break;
                case 7: si = 1 - j; sj = 1 - i; break;
                default: break;
                }
                s += R[i][j] * D[si][sj];
            }
        if (s > best) { best = s; ks = k; }
    }
    return ks;
}

__device__ __forceinline__ bool b2_less(double e, int32_t d, int32_t kj, double be, int32_t bd, int32_t bkj) {
    if (e != be) return e < be;
    if (d != bd) return d < bd;
    return kj < bkj;
}

// Pass 2: one warp per range (see above).
__global__ void __launch_bounds__(256) b2exact_kernel(const __grid_constant__ B2Params P) {
    const int lane = threadIdx.x & 31;
    const int r = (int)((blockIdx.x * blockDim.x + threadIdx.x) >> 5);
    if (blockIdx.x == 0 && threadIdx.x == 0) *P.d_ns = 1ull;
    const int n_r = (int)*P.d_nr;
    if (r >= n_r) return;
    const int64_t n_k = (int64_t)P.d_misc[0];
    const int n_tiles = (int)((n_k + kTileD - 1) / kTileD);
    const double cmax = (double)P.d_misc[1];
    const int ns = (int)*P.d_nscan;
    const int2 rr = P.ranges[r];
    const uint8_t *p0 = P.img + (size_t)rr.y * P.N + rr.x;
    const B2Range R = b2_range(p0[0], p0[1], p0[P.N + 1], p0[P.N]);
    const double A = (double)R.A;
    const double margin = b2_margin(A, P.smax, cmax, P.grid.on != 0);
    float gmn = INFINITY;
    for (int i = lane; i < ns; i += 32) gmn = fminf(gmn, P.gmin[(size_t)r * P.ns_cap + i]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) gmn = fminf(gmn, __shfl_xor_sync(0xffffffffu, gmn, o));
    float thr = gmn < INFINITY ? fminf(__double2float_ru(__dadd_rn((double)gmn, 2.0 * margin)), FLT_MAX) : FLT_MAX;
    double be;
    int32_t bd, bkj;
    if (P.has_zero) {  // s = 0: e = A for every (domain, k); first is (0, 0, j_zero)
        be = A; bd = 0; bkj = P.j_zero;
        thr = fminf(thr, fminf(__double2float_ru(margin), FLT_MAX));
    } else {
        be = INFINITY; bd = INT_MAX; bkj = INT_MAX;
    }
    unsigned n_exact = 0;
    for (int sp = 0; sp < ns; ++sp) {
        if (!(P.gmin[(size_t)r * P.ns_cap + sp] <= thr)) continue;  // warp-uniform
        const int64_t d0 = ((int64_t)sp * n_tiles / ns) * kTileD;
        const int64_t d1 = min(n_k, ((int64_t)(sp + 1) * n_tiles / ns) * kTileD);
        for (int64_t pos = d0 + lane; pos < d1; pos += 32) {
            const float4 f = P.F[pos];
            const float bq = fmaf(R.sx, f.y, fabsf(fmaf(R.x2, f.x, R.dx * f.z)));
            float g = INFINITY;
            if (P.grid.on) g = b2_grid_g(P.grid, bq, P.T[pos * 2], P.T[pos * 2 + 1]);
            else
                for (int jj = 0; jj < P.nsp; ++jj) g = fminf(g, fmaf(P.nhs[jj], bq, P.T[pos * P.tw + jj]));
            if (g <= thr) {
                ++n_exact;
                const int32_t d = P.ds[pos];
                const double Bq = 0.5 * (double)bq, c16 = __dmul_rn(0.0625, (double)f.w);
                double e0 = INFINITY;
                int j0 = 0;
                for (int jj = 0; jj < P.nsp; ++jj) {
                    const double sv = P.spos[jj];
                    const double e = __dadd_rn(__dsub_rn(A, __dmul_rn(__dmul_rn(0.5, sv), Bq)),
                                               __dmul_rn(__dmul_rn(sv, sv), c16));
                    if (e < e0) { e0 = e; j0 = jj; }  // lowest j among equal e (same k* for every s > 0)
                }
                int32_t kj = P.jpos[j0] | kPendIso;
                if (e0 == be && d == bd)  // only the zero-s seed (d = 0, k = 0) ties here
                    kj = (b2_kstar(P, rr, d) << 8) | P.jpos[j0];
                if (b2_less(e0, d, kj, be, bd, bkj)) {
                    be = e0; bd = d; bkj = kj;
                    thr = fminf(thr, fminf(__double2float_ru(__dadd_rn(__dsub_rn(e0, A), margin)), FLT_MAX));
                }
            }
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const double oe = __shfl_xor_sync(0xffffffffu, be, o);
        const int32_t od = __shfl_xor_sync(0xffffffffu, bd, o);
        const int32_t okj = __shfl_xor_sync(0xffffffffu, bkj, o);
        if (b2_less(oe, od, okj, be, bd, bkj)) { be = oe; bd = od; bkj = okj; }
        n_exact += __shfl_xor_sync(0xffffffffu, n_exact, o);
    }
    if (lane == 0) {
        Partial pb;
        pb.e = be;
        pb.d = bd;
        pb.kj = bkj;
        P.part[(size_t)r * P.ns_cap] = pb;
        if (n_exact && P.exact_count) atomicAdd(P.exact_count, (unsigned long long)n_exact);
    }
}

// float <-> int key with the same order (a signed-int min is a float min)
__device__ __forceinline__ int b2_fkey(float f) {
    const int i = __float_as_int(f);
    return i >= 0 ? i : i ^ 0x7fffffff;
}
__device__ __forceinline__ float b2_fdec(int k) { return __int_as_float(k >= 0 ? k : k ^ 0x7fffffff); }

// ---------------------------------------------------------------------------------------------
// Windowed search (predefined s: no s = 0, at most 2 values), one warp per range.
//
// Cauchy-Schwarz on the centred vectors gives |Bq_k| <= sqrt(A C) for every isometry, so for
// every domain and every s
//     e_s = A - (s/2) Bq + (s^2/16) C  >=  lb_s(C) = (sqrt(A) - s sqrt(C)/4)^2 ,
// and a domain can only win or tie if lb_s(C) <= best for some s in the level's set.  lb_s is
// minimal (0) at the centre C*_s = 16 A / s^2 and grows monotonically away from it, and the
// pool is sorted by C, so the warp expands outward from the centres, best-first: each step
// takes the 32 domains next to the frontier with the smallest lb, scores them (fp32 filter,
// canonical binary64 path for every pair with g <= thr, as in pass 2), and a frontier stops
// once its lb exceeds the current best.  With s_a > s_b (centres c_a <= c_b) four frontiers
// cover the windows: below c_a (lb_a is the smaller bound there), c_a upward and c_b downward
// (they stop where they meet), above c_b (lb_b smaller).  Rounding: a frontier stops only if
// |sqrt(A) - s sqrt(C)/4| > sqrt(ub)(1 + 1e-6) + 1e-3, which covers the binary64 error of the
// canonical score (< 4.4e-16 (2 sqrt(A) + delta)^2 for A < 2^21).  Unvisited domains are
// provably worse than the best, so the result equals the exhaustive loop.
__device__ __forceinline__ int b2_lower_bound(const int32_t *__restrict__ Cs, int n, double v, int lane) {
    int lo = 0, hi = n;  // invariant: Cs[< lo] < v <= Cs[>= hi]
    while (hi - lo > 32) {
        const int64_t span = hi - lo;
        const int p = lo + (int)((span * (lane + 1)) / 33);
        const unsigned m = __ballot_sync(0xffffffffu, (double)__ldg(Cs + p) >= v);
        const int f = m ? __ffs(m) - 1 : 32;
        const int phi = __shfl_sync(0xffffffffu, p, f < 32 ? f : 31);
        const int plo = __shfl_sync(0xffffffffu, p, f > 0 ? f - 1 : 0);
        if (f < 32) hi = phi;
        if (f > 0) lo = plo + 1;
    }
    const int p = lo + lane;
    const unsigned m = __ballot_sync(0xffffffffu, p < hi ? (double)__ldg(Cs + p) >= v : true);
    return lo + (__ffs(m) - 1);
}

// canonical binary64 score of one (range, domain): min over s > 0 with the lowest j (Eq. 1/3, C7)
__device__ __forceinline__ double b2_canon(const B2Params &P, double A, float bq, float cf, int &j0) {
    const double Bq = 0.5 * (double)bq, c16 = __dmul_rn(0.0625, (double)cf);
    double e0 = INFINITY;
    j0 = 0;
    for (int jj = 0; jj < P.nsp; ++jj) {
        const double sv = P.spos[jj];
        const double e = __dadd_rn(__dsub_rn(A, __dmul_rn(__dmul_rn(0.5, sv), Bq)), __dmul_rn(__dmul_rn(sv, sv), c16));
        if (e < e0) { e0 = e; j0 = jj; }  // lowest j among equal e (same k* for every s > 0)
    }
    return e0;
}

#ifndef FIC_B2_WINSTEP
#define FIC_B2_WINSTEP 128
#endif
#ifndef FIC_B2_MINB
#define FIC_B2_MINB 4
#endif
constexpr int kWinStep = FIC_B2_WINSTEP;  // domains per frontier per round
constexpr int kWinPer = 4 * (kWinStep / 32);  // features per lane per round

constexpr int kStash = 64;  // phase-1 candidates kept per warp (overflow: full phase-2 sweep)

// 6 CTAs (48 warps) per SM: the rounds are L2-latency bound, and more resident warps beat the
// few spills of the 40-register budget (C3 B = 2: 74 regs 0.312 ms, 64 0.273, 48 0.260, 40 0.251,
// 32 0.265)
__global__ void __launch_bounds__(256, FIC_B2_MINB) b2win_kernel(const __grid_constant__ B2Params P) {
    __shared__ int sStash[8][kStash];
    __shared__ int sNst[8];
    pdl_wait();
    pdl_trigger();
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    if (lane == 0) sNst[wib] = 0;
    __syncwarp();
    const int r = (int)((blockIdx.x * blockDim.x + threadIdx.x) >> 5);
    if (blockIdx.x == 0 && threadIdx.x == 0) *P.d_ns = 1ull;
    const int n_r = (int)*P.d_nr;
    if (r >= n_r) return;
    const int n_k = (int)P.d_misc[0];
    const double cmax = (double)P.d_misc[1];
    const int2 rr = P.ranges[r];
    const uint8_t *p0 = P.img + (size_t)rr.y * P.N + rr.x;
    const B2Range R = b2_range(p0[0], p0[1], p0[P.N + 1], p0[P.N]);
    const double A = (double)R.A;
    // t2_j = RN(RN(s_j^2 / 16) C) from the feature's C (exact in fp32, C < 2^24) instead of a
    // table load: two roundings, 2u t2 more than the table's one -- added to the margin
    const double margin = b2_margin(A, P.smax, cmax) + 2.0 * 5.9604644775390625e-08 * (P.smax * P.smax * cmax * 0.0625);
    const float nh0 = P.nhs[0], nh1 = P.nsp > 1 ? P.nhs[1] : P.nhs[0];
    const float k0 = __double2float_rn(P.spos[0] * P.spos[0] * 0.0625);
    const float k1 = P.nsp > 1 ? __double2float_rn(P.spos[1] * P.spos[1] * 0.0625) : k0;
    const float2 nh01 = make_float2(nh0, nh1), k01 = make_float2(k0, k1);
    auto gof = [&](const float4 fv, float &bq) {  // both s in packed FMUL2 / FFMA2 (same roundings)
        bq = fmaf(R.sx, fv.y, fabsf(fmaf(R.x2, fv.x, R.dx * fv.z)));
        const float2 t2 = __fmul2_rn(k01, make_float2(fv.w, fv.w));
        const float2 g2 = __ffma2_rn(nh01, make_float2(bq, bq), t2);
        return fminf(g2.x, g2.y);
    };
    auto gval = [&](int pos, float &bq, float &cf) {
        const float4 fv = __ldg(P.F + pos);
        cf = fv.w;
        return gof(fv, bq);
    };
    // s_a >= s_b, centres c_a <= c_b
    const int ia = (P.nsp > 1 && P.spos[1] > P.spos[0]) ? 1 : 0, ib = P.nsp > 1 ? 1 - ia : ia;
    const double sa = P.spos[ia], sb = P.spos[ib];
#ifndef FIC_B2_CTAB
#define FIC_B2_CTAB 1
#endif
    // the window centres' positions: a frontier tests only its far end, so any start positions
    // monotone in the centre serve (b2wink_kernel): the coarse index of the sorted C, one load
    // per centre, instead of two warp-wide searches of ~3 dependent rounds each
    int ca, cb;
    if (FIC_B2_CTAB) {
        const float dl = sqrtf((float)cmax) / (float)P.ctab_n;
        int c = 0;
        if (lane < 2 && n_k > 0) {
            const float x = 4.f * sqrtf((float)R.A) / (float)(lane == 0 ? sa : sb);
            const int t = dl > 0.f ? (int)fminf(x / dl, (float)(P.ctab_n - 1)) : 0;
            c = min(__ldg(P.ctab + t), n_k);
        }
        ca = __shfl_sync(0xffffffffu, c, 0);
        cb = max(ca, __shfl_sync(0xffffffffu, c, 1));
    } else {
        ca = n_k > 0 ? b2_lower_bound(P.Cs, n_k, 16.0 * A / (sa * sa), lane) : 0;
        cb = n_k > 0 ? max(ca, b2_lower_bound(P.Cs, n_k, 16.0 * A / (sb * sb), lane)) : 0;
    }
    // window bounds in C (fp32, widened by 1e-4 relative and 1e-3 (1 + sqrt A) absolute in
    // sqrt C -- far above the fp32 rounding of these few operations, so never too narrow)
    const float sqAf = sqrtf((float)R.A);
    const float ka = (float)(4.0 / sa), kb = (float)(4.0 / sb);
    // round-up fp32 copies for the per-round bounds (every rounding upward keeps ub >= best and
    // the stash threshold >= the final one)
    const float A_ru = __double2float_ru(A), marg_ru = __double2float_ru(margin);
    const float marg2_ru = __double2float_ru(2.0 * margin);
    // frontiers: f0 [q0, c_a) grows down (s_a), f1 [c_a, q1) grows up (s_a), f2 [q2, c_b) grows
    // down (s_b), f3 [c_b, q3) grows up (s_b); f1 and f2 share [c_a, c_b) and stop when they meet
    int q0 = ca, q1 = ca, q2 = cb, q3 = cb;
    bool al0 = q0 > 0, al1 = q1 < q2, al2 = q1 < q2, al3 = q3 < n_k;
    float gmin = INFINITY;
    unsigned scanned = 0;
    // phase 1: rounds over the four frontiers with the fp32 filter; the bound ub = A + gmin +
    // margin (>= best) narrows the windows after every round
    while (al0 || al1 || al2 || al3) {
        const int n0 = al0 ? min(kWinStep, q0) : 0;
        const int gap = q2 - q1;
        const int n1 = al1 ? min(kWinStep, gap) : 0;
        const int n2 = al2 ? min(kWinStep, gap - n1) : 0;
        const int n3 = al3 ? min(kWinStep, n_k - q3) : 0;
        const int b0 = q0 - n0, b1 = q1, b2 = q2 - n2, b3 = q3;
        q0 -= n0; q1 += n1; q2 -= n2; q3 += n3;
        scanned += (unsigned)(n0 + n1 + n2 + n3);
        // next frontier C values (lanes 0..3), in flight with this round's features
        int cn = 0;
        if (lane == 0 && q0 > 0) cn = __ldg(P.Cs + q0 - 1);
        if (lane == 1 && q1 < q2) cn = __ldg(P.Cs + q1);
        if (lane == 2 && q1 < q2) cn = __ldg(P.Cs + q2 - 1);
        if (lane == 3 && q3 < n_k) cn = __ldg(P.Cs + q3);
        // all of this lane's loads of the round first (up to 8 domains, L2-latency bound), then
        // the arithmetic; absent slots read position 0 and are masked to +inf
        float4 fv[kWinPer];
        bool ok8[kWinPer];
        const int nf[4] = {n0, n1, n2, n3}, bf[4] = {b0, b1, b2, b3};
#pragma unroll
        for (int k = 0; k < kWinStep / 32; ++k) {
#pragma unroll
            for (int f = 0; f < 4; ++f) {
                const int o = lane + 32 * k;
                ok8[k * 4 + f] = o < nf[f];
                const int pos = ok8[k * 4 + f] ? bf[f] + o : 0;
                fv[k * 4 + f] = __ldg(P.F + pos);
            }
        }
        float g = INFINITY, gv[kWinPer];
#pragma unroll
        for (int i = 0; i < kWinPer; ++i) {
            float bq;
            const float gi = gof(fv[i], bq);
            gv[i] = ok8[i] ? gi : INFINITY;
            g = fminf(g, gv[i]);
        }
        gmin = fminf(gmin, b2_fdec(__reduce_min_sync(0xffffffffu, b2_fkey(g))));
        {
            // stash every domain with g <= RU(gmin + 2 margin) (gmin including this round): the
            // final threshold RU(gmin_final + 2 margin) is never larger, so the stash holds every
            // pair phase 2 has to score
            const float ts = fminf(__fadd_ru(gmin, marg2_ru), FLT_MAX);
            if (__any_sync(0xffffffffu, g <= ts)) {  // (g: this lane's minimum of the round)
#pragma unroll
                for (int i = 0; i < kWinPer; ++i) {
                    if (gv[i] <= ts) {
                        const int slot = atomicAdd(&sNst[wib], 1);
                        if (slot < kStash) sStash[wib][slot] = bf[i & 3] + lane + 32 * (i >> 2);
                    }
                }
            }
        }
        const float ub = gmin < INFINITY ? __fadd_ru(__fadd_ru(A_ru, gmin), marg_ru) : INFINITY;
        const float u = sqrtf(fmaxf(ub, 0.f)) * 1.0001f + 1e-3f * (1.f + sqAf);
        const float la = ka * (sqAf - u), lb = kb * (sqAf - u);
        const float cl = (lane == 0 ? la : lb);
        const float clo = cl > 0.f ? cl * cl * 0.9999f : -1.f;
        const float ch = (lane == 1 ? ka : kb) * (sqAf + u);
        const float chi = ch * ch * 1.0001f;
        // lane f: is frontier f's next domain inside its window?
        bool in = false;
        if (lane == 0) in = q0 > 0 && (float)cn >= clo;
        if (lane == 1) in = q1 < q2 && (float)cn <= chi;
        if (lane == 2) in = q1 < q2 && (float)cn >= clo;
        if (lane == 3) in = q3 < n_k && (float)cn <= chi;
        const unsigned m = __ballot_sync(0xffffffffu, in);
        al0 = m & 1u;
        al1 = (m >> 1) & 1u;
        al2 = (m >> 2) & 1u;
        al3 = (m >> 3) & 1u;
    }
    // phase 2: every pair of the visited runs with g <= thr takes the canonical binary64 path
    // (thr = RU(gmin + 2 margin) >= best - A + margin; unvisited domains have lb > ub >= best):
    // the stashed candidates, or a sweep of the visited runs if the stash overflowed
    float thr = gmin < INFINITY ? fminf(__double2float_ru(__dadd_rn((double)gmin, 2.0 * margin)), FLT_MAX) : -FLT_MAX;
    double be = INFINITY;
    int32_t bd = INT_MAX, bkj = INT_MAX;
    unsigned n_exact = 0;
    __syncwarp();
    const int nst = sNst[wib];
    if (nst <= kStash) {
        for (int i = lane; i < nst; i += 32) {
            const int pos = sStash[wib][i];
            float bq, cf;
            if (gval(pos, bq, cf) <= thr) {
                ++n_exact;
                int j0;
                const double e0 = b2_canon(P, A, bq, cf, j0);
                const int32_t d = __ldg(P.ds + pos);
                const int32_t kj = P.jpos[j0] | kPendIso;
                if (b2_less(e0, d, kj, be, bd, bkj)) { be = e0; bd = d; bkj = kj; }
            }
        }
    }
    const int nrun = nst <= kStash ? 0 : (q1 < q2 ? 2 : 1);  // visited: [q0, q1), [q2, q3) (one run once q1 == q2)
    for (int w = 0; w < nrun; ++w) {
        const int a0 = w == 0 ? q0 : q2;
        const int a1 = (w == 0 && nrun == 2) ? q1 : q3;
        // four domains per lane per pass: the loads first, then the filter (rare exact path)
        for (int pos0 = a0 + lane; pos0 < a1; pos0 += 128) {
            float4 fv[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int pos = min(pos0 + 32 * i, a1 - 1);
                fv[i] = __ldg(P.F + pos);
            }
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int pos = pos0 + 32 * i;
                float bq;
                const float gi = gof(fv[i], bq);
                if (pos < a1 && gi <= thr) {
                    ++n_exact;
                    int j0;
                    const double e0 = b2_canon(P, A, bq, fv[i].w, j0);
                    const int32_t d = __ldg(P.ds + pos);
                    const int32_t kj = P.jpos[j0] | kPendIso;
                    if (b2_less(e0, d, kj, be, bd, bkj)) {
                        be = e0; bd = d; bkj = kj;
                        thr = fminf(thr, fminf(__double2float_ru(__dadd_rn(__dsub_rn(e0, A), margin)), FLT_MAX));
                    }
                }
            }
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const double oe = __shfl_xor_sync(0xffffffffu, be, o);
        const int32_t od = __shfl_xor_sync(0xffffffffu, bd, o);
        const int32_t okj = __shfl_xor_sync(0xffffffffu, bkj, o);
        if (b2_less(oe, od, okj, be, bd, bkj)) { be = oe; bd = od; bkj = okj; }
        n_exact += __shfl_xor_sync(0xffffffffu, n_exact, o);
    }
    if (lane == 0) {
        Partial pb;
        pb.e = be;
        pb.d = bd;
        pb.kj = bkj;
        P.part[(size_t)r * P.ns_cap] = pb;
        if (n_exact && P.exact_count) atomicAdd(P.exact_count, (unsigned long long)n_exact);
        if (P.scan_count) atomicAdd(P.scan_count, (unsigned long long)scanned);
    }
}

// ---------------------------------------------------------------------------------------------
// Windowed search for a uniform grid of s (the 16-value grid, sampled10, the closed-form levels:
// up to 31 positive values; s = 0 may be listed), one warp per range.
//
// b2win_kernel's bound per s: a domain can only win or tie if lb_s(C) = (sqrt(A) - s sqrt(C)/4)^2
// <= best for some s, i.e. sqrt(C) in W_s = [(4/s)(sqrt(A) - sqrt(best)), (4/s)(sqrt(A) +
// sqrt(best))], a window around the centre C*_s = 16 A / s^2.  Both ends of W_s decrease as s
// grows, so the centres (s descending = C* ascending) cut the C-sorted pool into K + 1 gaps and
// inside gap i (between centres i - 1 and i) the union of the windows is W_{i-1}'s part above
// centre i - 1 plus W_i's part below centre i.  Lane i owns gap i: an up frontier (from centre
// i - 1, stops past W_{i-1}'s upper end) and a down frontier (from centre i, stops past W_i's lower
// end) consume it from both ends and stop when they meet.  A frontier tests only its far end,
// so the start positions need only be monotone in i, not exact: they come from the coarse index
// of the sorted C (one load per lane instead of K binary searches).  Rounds take up to 512 / kWkStep
// frontiers (rotating), 128 domains each; filter, stash and phase 2 as in b2win_kernel, with the
// uniform-grid bracket of tcsearch_kernel<B, 3> as the fp32 score (the bracket's RN(2 / (C h))
// only picks the two grid points around s*: an approximate quotient, off by far less than half a
// grid step, picks the same nearest point) and the s = 0 seed (A; 0, 0, j_zero) when listed.
#ifndef FIC_B2WK_STEP
#define FIC_B2WK_STEP 128
#endif
constexpr int kWkStep = FIC_B2WK_STEP;         // domains per frontier task (a multiple of 32)
constexpr int kWkTasks = 512 / kWkStep;         // tasks per round: 16 features per lane
__global__ void __launch_bounds__(256, FIC_B2_MINB) b2wink_kernel(const __grid_constant__ B2Params P) {
    __shared__ int sStash[8][kStash];
    __shared__ int sNst[8];
    pdl_wait();
    pdl_trigger();
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    if (lane == 0) sNst[wib] = 0;
    __syncwarp();
    const int r = (int)((blockIdx.x * blockDim.x + threadIdx.x) >> 5);
    if (blockIdx.x == 0 && threadIdx.x == 0) *P.d_ns = 1ull;
    const int n_r = (int)*P.d_nr;
    if (r >= n_r) return;
    const int n_k = (int)P.d_misc[0];
    const double cmax = (double)P.d_misc[1];
    const int2 rr = P.ranges[r];
    const uint8_t *p0 = P.img + (size_t)rr.y * P.N + rr.x;
    const B2Range R = b2_range(p0[0], p0[1], p0[P.N + 1], p0[P.N]);
    const double A = (double)R.A;
    const double margin = b2_margin(A, P.smax, cmax, true);
    const int K = P.nsp;  // positive s, ascending (a uniform grid); centre i <-> spos[K - 1 - i]
    const float g2h = (float)(2.0 / (double)P.grid.h);
    auto gof = [&](const float4 fv, float &bq) {
        bq = fmaf(R.sx, fv.y, fabsf(fmaf(R.x2, fv.x, R.dx * fv.z)));
        const float ug = fv.w > 0.f ? __fdividef(g2h, fv.w) : 0.f;
        return b2_grid_g(P.grid, bq, fv.w * 0.0625f, ug);  // (C / 16 exact: C < 2^23)
    };
    const float sqAf = sqrtf((float)R.A);
    // gap `lane` (0 .. K): [lo0, hi0), consumed from both ends
    int c = n_k;
    if (lane < K) {
        const float dl = sqrtf((float)cmax) / (float)P.ctab_n;
        const float x = 4.f * sqAf / (float)P.spos[K - 1 - lane];  // sqrt(C*) of centre `lane`
        const int t = dl > 0.f ? (int)fminf(x / dl, (float)(P.ctab_n - 1)) : 0;
        c = min(__ldg(P.ctab + t), n_k);
    }
    const int cprev = __shfl_up_sync(0xffffffffu, c, 1);
    const int lo0 = (lane == 0 || lane > K) ? 0 : cprev;
    const int hi0 = lane < K ? c : (lane == K ? n_k : 0);
    int lo = lo0, hi = hi0;
    // window factors 4 / s: up frontier <-> centre lane - 1, down frontier <-> centre lane
    const float ku = (lane >= 1 && lane <= K) ? (float)(4.0 / P.spos[K - lane]) : 0.f;
    const float kd = lane < K ? (float)(4.0 / P.spos[K - 1 - lane]) : 0.f;
    bool upA = lane >= 1 && lane <= K && lo < hi;
    bool dnA = lane < K && lo < hi;
    const float A_ru = __double2float_ru(A), marg_ru = __double2float_ru(margin);
    const float marg2_ru = __double2float_ru(2.0 * margin);
    const float zcap = P.has_zero ? marg_ru : FLT_MAX;  // s = 0 listed: best <= A
    float gmin = INFINITY;
    unsigned scanned = 0, rot = 0;
    for (;;) {
        const unsigned mu = __ballot_sync(0xffffffffu, upA), md = __ballot_sync(0xffffffffu, dnA);
        if (!(mu | md)) break;
        // up to 4 tasks: bit g = up frontier of gap g, bit 32 + g = its down frontier
        const unsigned long long all = (unsigned long long)mu | ((unsigned long long)md << 32);
        const unsigned long long rotd = rot ? ((all >> rot) | (all << (64 - rot))) : all;
        int tb[kWkTasks], tn[kWkTasks];
        unsigned long long left = rotd;
#pragma unroll
        for (int t = 0; t < kWkTasks; ++t) {
            tb[t] = 0; tn[t] = 0;
            if (!left) continue;
            const int bit = __ffsll((long long)left) - 1;
            left &= left - 1;
            const int task = (bit + (int)rot) & 63, g = task & 31;
            int base = 0, n = 0;
            if (lane == g) {
                n = min(kWkStep, hi - lo);
                if (task < 32) { base = lo; lo += n; }
                else { base = hi - n; hi -= n; }
            }
            tb[t] = __shfl_sync(0xffffffffu, base, g);
            tn[t] = __shfl_sync(0xffffffffu, n, g);
        }
        {
            // next rotation offset: after the last task of this round
            unsigned long long l2 = rotd;
            int last = -1;
#pragma unroll
            for (int t = 0; t < kWkTasks; ++t) {
                if (!l2) break;
                last = __ffsll((long long)l2) - 1;
                l2 &= l2 - 1;
            }
            if (last >= 0) rot = (unsigned)((last + (int)rot + 1) & 63);
        }
        // the frontiers' next C values (in flight with the features)
        int cnu = 0, cnd = 0;
        if (upA && lo < hi) cnu = __ldg(P.Cs + lo);
        if (dnA && lo < hi) cnd = __ldg(P.Cs + hi - 1);
        constexpr int NPL = kWkTasks * (kWkStep / 32);  // features per lane per round
        float4 fv[NPL];
        bool ok8[NPL];
#pragma unroll
        for (int k = 0; k < kWkStep / 32; ++k) {
#pragma unroll
            for (int t = 0; t < kWkTasks; ++t) {
                const int o = lane + 32 * k;
                ok8[k * kWkTasks + t] = o < tn[t];
                const int pos = ok8[k * kWkTasks + t] ? tb[t] + o : 0;
                fv[k * kWkTasks + t] = __ldg(P.F + pos);
            }
        }
#pragma unroll
        for (int t = 0; t < kWkTasks; ++t) scanned += (unsigned)tn[t];
        float g = INFINITY, gv[NPL];
#pragma unroll
        for (int i = 0; i < NPL; ++i) {
            float bq;
            const float gi = gof(fv[i], bq);
            gv[i] = ok8[i] ? gi : INFINITY;
            g = fminf(g, gv[i]);
        }
        gmin = fminf(gmin, b2_fdec(__reduce_min_sync(0xffffffffu, b2_fkey(g))));
        {
            // stash every domain with g <= the current phase-2 threshold bound (never below the
            // final threshold: gmin only decreases)
            const float ts = fminf(fminf(__fadd_ru(gmin, marg2_ru), FLT_MAX), zcap);
            if (__any_sync(0xffffffffu, g <= ts)) {
#pragma unroll
                for (int i = 0; i < NPL; ++i) {
                    if (gv[i] <= ts) {
                        const int slot = atomicAdd(&sNst[wib], 1);
                        if (slot < kStash) sStash[wib][slot] = tb[i % kWkTasks] + lane + 32 * (i / kWkTasks);
                    }
                }
            }
        }
        float ub = gmin < INFINITY ? __fadd_ru(__fadd_ru(A_ru, gmin), marg_ru) : INFINITY;
        if (P.has_zero) ub = fminf(ub, A_ru);
        const float u = sqrtf(fmaxf(ub, 0.f)) * 1.0001f + 1e-3f * (1.f + sqAf);
        const float cl = kd * (sqAf - u);
        const float clo = cl > 0.f ? cl * cl * 0.9999f : -1.f;
        const float ch = ku * (sqAf + u);
        const float chi = ch * ch * 1.0001f;
        upA = upA && lo < hi && (float)cnu <= chi;
        dnA = dnA && lo < hi && (float)cnd >= clo;
    }
    // phase 2 (as b2win_kernel / b2exact_kernel): stashed candidates, or the visited runs
    float thr = gmin < INFINITY ? fminf(__double2float_ru(__dadd_rn((double)gmin, 2.0 * margin)), FLT_MAX) : -FLT_MAX;
    double be;
    int32_t bd, bkj;
    if (P.has_zero) {  // s = 0: e = A for every (domain, k); first is (0, 0, j_zero)
        be = A; bd = 0; bkj = P.j_zero;
        thr = gmin < INFINITY ? fminf(thr, zcap) : zcap;
    } else {
        be = INFINITY; bd = INT_MAX; bkj = INT_MAX;
    }
    unsigned n_exact = 0;
    auto exact = [&](int pos, float bq, float cf) {
        ++n_exact;
        const int32_t d = __ldg(P.ds + pos);
        const double Bq = 0.5 * (double)bq, c16 = __dmul_rn(0.0625, (double)cf);
        double e0 = INFINITY;
        int j0 = 0;
        for (int jj = 0; jj < P.nsp; ++jj) {
            const double sv = P.spos[jj];
            const double e = __dadd_rn(__dsub_rn(A, __dmul_rn(__dmul_rn(0.5, sv), Bq)), __dmul_rn(__dmul_rn(sv, sv), c16));
            if (e < e0) { e0 = e; j0 = jj; }  // lowest j among equal e (same k* for every s > 0)
        }
        int32_t kj = P.jpos[j0] | kPendIso;
        if (e0 == be && d == bd)  // only the zero-s seed (d = 0, k = 0) ties here
            kj = (b2_kstar(P, rr, d) << 8) | P.jpos[j0];
        if (b2_less(e0, d, kj, be, bd, bkj)) {
            be = e0; bd = d; bkj = kj;
            thr = fminf(thr, fminf(__double2float_ru(__dadd_rn(__dsub_rn(e0, A), margin)), FLT_MAX));
        }
    };
    __syncwarp();
    const int nst = sNst[wib];
    if (nst <= kStash) {
        for (int i = lane; i < nst; i += 32) {
            const int pos = sStash[wib][i];
            const float4 fv = __ldg(P.F + pos);
            float bq;
            if (gof(fv, bq) <= thr) exact(pos, bq, fv.w);
        }
    } else {
        // the visited runs of every gap: [lo0, lo) and [hi, hi0)
        for (int g = 0; g <= K; ++g) {
            const int l0 = __shfl_sync(0xffffffffu, lo0, g), l1 = __shfl_sync(0xffffffffu, lo, g);
            const int h1 = __shfl_sync(0xffffffffu, hi, g), h0 = __shfl_sync(0xffffffffu, hi0, g);
            for (int w = 0; w < 2; ++w) {
                const int a0 = w == 0 ? l0 : h1, a1 = w == 0 ? l1 : h0;
                for (int pos = a0 + lane; pos < a1; pos += 32) {
                    const float4 fv = __ldg(P.F + pos);
                    float bq;
                    if (gof(fv, bq) <= thr) exact(pos, bq, fv.w);
                }
            }
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const double oe = __shfl_xor_sync(0xffffffffu, be, o);
        const int32_t od = __shfl_xor_sync(0xffffffffu, bd, o);
        const int32_t okj = __shfl_xor_sync(0xffffffffu, bkj, o);
        if (b2_less(oe, od, okj, be, bd, bkj)) { be = oe; bd = od; bkj = okj; }
        n_exact += __shfl_xor_sync(0xffffffffu, n_exact, o);
    }
    if (lane == 0) {
        Partial pb;
        pb.e = be;
        pb.d = bd;
        pb.kj = bkj;
        P.part[(size_t)r * P.ns_cap] = pb;
        if (n_exact && P.exact_count) atomicAdd(P.exact_count, (unsigned long long)n_exact);
        if (P.scan_count) atomicAdd(P.scan_count, (unsigned long long)scanned);
    }
}

// t2_j per slot, [slot][tw]; +inf on pad slots and pad j
__global__ void b2_t2_kernel(const float4 *__restrict__ F, const unsigned long long *__restrict__ d_nk,
                             int64_t n_slots, const SList spos, int32_t nsp, int32_t tw, float *__restrict__ T,
                             float grid_h) {
    const int64_t d = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (d >= n_slots) return;
    const int64_t n_k = (int64_t)*d_nk;
    if (d >= ((n_k + kTileD - 1) / kTileD) * kTileD) return;
    const double c16 = __dmul_rn(0.0625, (double)F[d].w);  // C (exact in fp32, < 2^23)
    if (grid_h > 0.f) {  // uniform grid: RN(C/16) (+inf on pads), RN(2 / (C h)) (bq = 2 Bq)
        const double C = (double)F[d].w;
        T[d * 2] = d < n_k ? __double2float_rn(c16) : INFINITY;
        T[d * 2 + 1] = (d < n_k && C > 0.0) ? __double2float_rn(2.0 / (C * (double)grid_h)) : 0.f;
        return;
    }
    for (int j = 0; j < tw; ++j) {
        const double s = j < nsp ? spos.s[j] : 0.0;
        T[d * tw + j] = (d < n_k && j < nsp) ? __double2float_rn(__dmul_rn(__dmul_rn(s, s), c16)) : INFINITY;
    }
}

template <int NP>
static size_t b2_smem() {
    constexpr int TPS = NP == 1 ? 2 : 1;
    return (size_t)kB2NB * TPS * kTileD * (16 + 8 * (NP == 0 ? 1 : NP)) + kB2NB * 12 + 64;
}

template <int NP>
static cudaError_t launch_b2_scan(const B2Params &p, cudaStream_t st) {
    const size_t smem = b2_smem<NP>();
    static std::atomic<unsigned long long> attr{0};
    if (cudaError_t e = ensure_smem_attr(b2scan_kernel<NP>, (int)smem, attr)) return e;
    dim3 grid((unsigned)((p.n_r + kB2Threads * kB2RPT - 1) / (kB2Threads * kB2RPT)), (unsigned)p.nsplit);
    b2scan_kernel<NP><<<grid, kB2Threads, smem, st>>>(p);
    return cudaGetLastError();
}

int b2_nsplit_hint(int64_t n_r, int64_t n_tiles, int num_sms) {
    const int64_t gx = (n_r + kB2Threads * kB2RPT - 1) / (kB2Threads * kB2RPT);
    if (gx <= 0 || n_tiles <= 0) return 1;
    static int waves = [] {
        const char *e = getenv("FIC_B2_CTAS_PER_SM");
        return e ? atoi(e) : 6;
    }();
    int64_t ns = ((int64_t)num_sms * waves + gx - 1) / gx;
    const int64_t max_ns = (n_tiles + 1) / 2;
    if (ns > max_ns) ns = max_ns;
    if (ns < 1) ns = 1;
    if (ns > 65535) ns = 65535;
    return (int)ns;
}

// b2wink_kernel: windows enabled, a uniform grid of 3 .. 16 positive s (ascending; one gap per
// lane), env FIC_B2_WINK=0 keeps the two-pass scan.  C3 B = 2 (ms, scan -> windows): grid 1.04 ->
// 0.76 (18% of the pairs scanned), sampled10 1.02 -> 0.57 (13%); the 31 closed-form levels scan
// 33% of the pairs and stay on the scan (1.22 -> 1.26 with windows).  Frontier steps of 32 / 64
// domains (more tasks per round) scanned less but ran slower (grid 0.76 -> 1.10 / 0.82)

bool b2_wink_applies(const SearchParams &sp) {
    static const bool on = [] {
        const char *e = getenv("FIC_B2_WINK");
        return !(e && strcmp(e, "0") == 0);
    }();
    return on && sp.b2_window && sp.grid.on && sp.nsp >= 3 && sp.nsp <= 16;
}

int b2_t2_width(int32_t nsp) { return nsp <= 2 ? 2 : (nsp <= 16 ? 16 : 32); }  // (a grid uses 2 of them)

size_t b2_scratch_bytes(int64_t n_r, int32_t ns_cap) { return 64 + sizeof(float) * (size_t)n_r * ns_cap; }

cudaError_t launch_b2_search(const SearchParams &sp, const B2Pool &bp, float *T, const int32_t *kept,
                             int32_t L, int32_t A, void *scratch, unsigned long long *scan_count,
                             cudaStream_t st) {
    if (sp.n_r == 0 || sp.nsp == 0) return cudaSuccess;
    const bool grid = sp.grid.on && !(sp.b2_window && !sp.has_zero && sp.nsp <= 2);
    const int tw = grid ? 2 : b2_t2_width(sp.nsp);
    const int64_t slots = sp.slot_stride;
    SList sl;
    memcpy(sl.s, sp.spos, sizeof sl.s);
    const bool win = sp.b2_window && !sp.has_zero && sp.nsp <= 2;  // predefined s: C windows
    // a uniform grid of s (the large sets): per-s C windows over the gaps between the centres
    const bool wink = !win && b2_wink_applies(sp);
    if (slots > 0 && !win && !wink) {  // (the window kernels form t2 from the feature's C itself)
        b2_t2_kernel<<<(unsigned)((slots + 255) / 256), 256, 0, st>>>(bp.F, &sp.d_misc[0], slots, sl, sp.nsp, tw, T,
                                                                      grid ? sp.grid.h : 0.f);
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
    }
    B2Params p;
    memset(&p, 0, sizeof p);
    p.img = sp.img; p.N = sp.N; p.L = L; p.A = A; p.ranges = sp.ranges; p.n_r = sp.n_r;
    p.F = bp.F; p.T = T; p.Cs = bp.Cs; p.ds = bp.ds; p.tw = tw; p.kept = kept;
    p.d_nr = sp.d_nr; p.d_misc = sp.d_misc; p.nsplit = sp.nsplit; p.d_ns = sp.d_ns; p.ns_cap = sp.ns_cap;
    p.nsp = sp.nsp;
    memcpy(p.spos, sp.spos, sizeof p.spos);
    memcpy(p.jpos, sp.jpos, sizeof p.jpos);
    for (int j = 0; j < kMaxS; ++j) p.nhs[j] = j < sp.nsp ? -(float)(0.25 * sp.spos[j]) : 0.f;
    p.has_zero = sp.has_zero; p.j_zero = sp.j_zero;
    p.smax = sp.smax;
    p.grid = sp.grid;
    p.grid.on = grid ? 1 : 0;
    p.part = sp.part; p.exact_count = sp.exact_count; p.scan_count = scan_count;
    p.d_nscan = reinterpret_cast<unsigned long long *>(scratch);
    p.gmin = reinterpret_cast<float *>(static_cast<char *>(scratch) + 64);
    if (win) {  // predefined s: Cauchy-Schwarz windows
        p.ctab = bp.ctab; p.ctab_n = bp.ctab_n;
        if (cudaError_t e = launch_pdl(b2win_kernel, dim3((unsigned)((sp.n_r + 7) / 8)), dim3(256), 0, st, p)) return e;
        return cudaGetLastError();
    }
    if (wink) {
        p.ctab = bp.ctab; p.ctab_n = bp.ctab_n;
        p.grid.on = 1;
        if (cudaError_t e = launch_pdl(b2wink_kernel, dim3((unsigned)((sp.n_r + 7) / 8)), dim3(256), 0, st, p)) return e;
        return cudaGetLastError();
    }
    cudaError_t e = grid ? launch_b2_scan<0>(p, st)
                         : tw == 2 ? launch_b2_scan<1>(p, st) : tw == 16 ? launch_b2_scan<8>(p, st) : launch_b2_scan<16>(p, st);
    if (e != cudaSuccess) return e;
    b2exact_kernel<<<(unsigned)((sp.n_r + 7) / 8), 256, 0, st>>>(p);
    return cudaGetLastError();
}

}  // namespace fic
