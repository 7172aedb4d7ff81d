// fic_search.cu -- the range x (domain, isometry) search.
//
// What it computes (§2, lines 28-38; §3.1): for every range block R (B x B)
// and every kept decimated domain D (D' = 4d, 2x2 sums) under each of the 8 isometries T_k
// (applied to the domain), and every s of the level's list,
//     E = sum_i (s d_i + o - r_i)^2,  o = Rbar - s Dbar               (Eq. 1, Eq. 3)
// and per range the lexicographically first minimiser (E; dom, k, s_idx) [R17].
//
// How (DESIGN.md §"Search kernel"):
//   * cross terms SRD_k = sum_p R(p) D'(f_k(p)) = sum_q D'(q) Rperm_k(q) with the range
//     scattered through the isometry (Rperm_k(f_k(p)) = R(p)), so one domain tile in shared
//     memory serves all 8 isometries; fp32 FFMA on exact integers (every partial sum < 2^24:
//     whole sum for B <= 8, 64-pixel chunks folded into int32 for B = 16);
//   * per (range, domain): max_k SRD_k and, per s, an fp32 lower bound of the binary64 score
//     with a rigorous error margin.  Only when the bound does not exclude the pair from beating
//     (or tying) the thread's running best is the canonical binary64 score evaluated
//     (e = (A - (s/2) Bq) + (s s)(C/16), no FMA contraction; the winning isometry is the lowest
//     argmax of SRD_k for s > 0, all k tie for s = 0) -- the result is bit-identical to the
//     exhaustive first-min loop of the oracle;
//   * domain tiles are streamed with cp.async.bulk (TMA bulk copy) into a 2-stage mbarrier
//     pipeline; ranges x domain-splits form the grid; partial bests merged in finalize.
#include <cfloat>
#include <climits>

#include "fic_internal.cuh"

namespace fic {

// ----------------------------------------------------------------------------- PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    uint32_t done = 0;
    while (!done) {
        asm volatile(
            "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
            : "=r"(done)
            : "r"(smem_u32(bar)), "r"(parity)
            : "memory");
    }
}

// --------------------------------------------------------------------------- isometries
// T_k(X)(i,j) = X(src_k(i,j)) with T_k = Mirror^[k>=4] o RotCW^(k mod 4)   (reading R2):
// a clockwise quarter turn maps output (i,j) to source (b-j, i); the horizontal mirror maps
// (i,j) to (i, b-j) and acts after the rotation, i.e. first on the output coordinates.
__device__ __forceinline__ void iso_src(int B, int k, int i, int j, int &si, int &sj) {
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

// ----------------------------------------------------------------------------- ordering
struct Best {
    double e;
    int32_t d, kj;  // kj = iso << 8 | s_idx
};
__device__ __forceinline__ bool lex_less(double e, int32_t d, int32_t kj, const Best &b) {
    if (e < b.e) return true;
    if (e > b.e) return false;
    if (d != b.d) return d < b.d;
    return kj < b.kj;
}

template <int B>
struct SCfg {
    static constexpr int n = B * B;
    static constexpr int KC = n < 64 ? n : 64;     // pixels per stage row block
    static constexpr int NCH = n / KC;             // stages per tile (B = 16: 4)
    static constexpr int TPS = n < 64 ? 64 / n : 1;  // tiles per stage (B <= 4)
    static constexpr int STAGE_F = 64 * kTileD;    // floats per stage (32 KB)
    static constexpr int RS_F = 8 * n * 8;         // [8 ranges][n][8 isometries]
    static constexpr size_t SMEM = (size_t)(2 * STAGE_F + RS_F) * 4 + 64;
};

template <int NSP>
struct WarpRange {
    double A, SR;
    float hsn[NSP], hsSR[NSP];
    double margin;
};

// Exact path: canonical binary64 score of one (range, domain) for every s > 0 (C7 of the
// oracle's reading), lexicographic update of the running best, threshold refresh.
template <int NSP>
__device__ __noinline__ void exact_update(const SearchParams &P, int n, int d, const int (&srd)[8],
                                          const WarpRange<NSP> &W, Best &best, float &thr) {
    int mx = srd[0], ks = 0;
#pragma unroll
    for (int k = 1; k < 8; ++k)
        if (srd[k] > mx) { mx = srd[k]; ks = k; }
    const double Bq = __dsub_rn(__dmul_rn((double)n, (double)mx), __dmul_rn(W.SR, (double)P.SD[d]));
    const double c16 = __dmul_rn(0.0625, (double)P.C[d]);
    for (int jj = 0; jj < P.nsp; ++jj) {
        const double s = P.spos[jj];
        const double hs = __dmul_rn(0.5, s);
        const double t2 = __dmul_rn(__dmul_rn(s, s), c16);
        const double e = __dadd_rn(__dsub_rn(W.A, __dmul_rn(hs, Bq)), t2);
        const int32_t kj = (ks << 8) | P.jpos[jj];
        if (lex_less(e, d, kj, best)) { best.e = e; best.d = d; best.kj = kj; }
    }
    const double t = __dadd_rn(__dsub_rn(best.e, W.A), W.margin);
    thr = fminf(__double2float_ru(t), FLT_MAX);
}

template <int B, int NSP>
__global__ void __launch_bounds__(256, 1) search_kernel(const __grid_constant__ SearchParams P) {
    using Cf = SCfg<B>;
    constexpr int n = Cf::n, NCH = Cf::NCH, TPS = Cf::TPS;
    extern __shared__ __align__(128) unsigned char smem[];
    float *Ds = reinterpret_cast<float *>(smem);
    float *Rs = Ds + 2 * Cf::STAGE_F;
    uint64_t *bar = reinterpret_cast<uint64_t *>(Rs + Cf::RS_F);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int n_r = (int)*P.d_nr;
    const int n_tiles = (int)((P.d_misc[0] + kTileD - 1) / kTileD);
    const double cmax = (double)P.d_misc[1];
    const int r = blockIdx.x * 8 + warp;
    const bool rvalid = r < n_r;
    const int split = blockIdx.y;
    const int t0 = (int)(((int64_t)split * n_tiles) / P.nsplit);
    const int t1 = (int)(((int64_t)(split + 1) * n_tiles) / P.nsplit);
    const int ntl = max(0, t1 - t0);
    const int nstages = (n <= 64) ? (ntl + TPS - 1) / TPS : ntl * NCH;
    const int64_t n_slots = P.slot_stride;

    auto issue = [&](int s) {
        const int buf = s & 1;
        const float *src;
        uint32_t bytes;
        if (n <= 64) {
            const int ta = t0 + s * TPS, tb = min(t1, ta + TPS);
            src = P.Dt + (size_t)ta * n * kTileD;
            bytes = (uint32_t)(tb - ta) * n * kTileD * 4;
        } else {
            const int tile = t0 + s / NCH, ch = s % NCH;
            src = P.Dt + ((size_t)tile * n + (size_t)ch * 64) * kTileD;
            bytes = 64 * kTileD * 4;
        }
        mbar_expect_tx(&bar[buf], bytes);
        bulk_g2s(Ds + buf * Cf::STAGE_F, src, bytes, &bar[buf]);
    };

    if (threadIdx.x == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        fence_mbar_init();
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        if (nstages > 0) issue(0);
        if (nstages > 1) issue(1);
    }

    // ---- prologue: this warp's range scattered through the 8 isometries, and its moments
    int rx = 0, ry = 0;
    if (rvalid) {
        const int2 rr = P.ranges[r];
        rx = rr.x;
        ry = rr.y;
    }
    float *Rw = Rs + warp * n * 8;
    long long sr = 0, srr = 0;
    for (int idx = lane; idx < n; idx += 32) {
        const int i = idx / B, j = idx % B;
        const int v = rvalid ? (int)P.img[(size_t)(ry + i) * P.N + rx + j] : 0;
        sr += v;
        srr += v * v;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            int si, sj;
            iso_src(B, k, i, j, si, sj);
            Rw[(si * B + sj) * 8 + k] = (float)v;
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        sr += __shfl_xor_sync(0xffffffffu, sr, o);
        srr += __shfl_xor_sync(0xffffffffu, srr, o);
    }
    WarpRange<NSP> W;
    W.A = (double)((long long)n * srr - sr * sr);
    W.SR = (double)sr;
#pragma unroll
    for (int jj = 0; jj < NSP; ++jj) {
        const double s = jj < P.nsp ? P.spos[jj] : 0.0;
        W.hsn[jj] = __double2float_rn(__dmul_rn(__dmul_rn(0.5, s), (double)n));
        W.hsSR[jj] = __double2float_rn(__dmul_rn(__dmul_rn(0.5, s), W.SR));
    }
    {
        // bound on the magnitude of the fp32-evaluated terms, over every domain and s:
        // (s/2) n SRD + (s/2) SR SD <= s n 1020 SR ;  s^2 C / 16 <= smax^2 Cmax / 16
        const double mp = P.smax * (double)n * 1020.0 * W.SR + P.smax * P.smax * cmax * 0.0625;
        W.margin = ldexp(W.A + mp, -18) + 1e-30;  // 64 ulp(fp32) of the magnitudes
    }
    Best best;
    if (P.has_zero) {  // s = 0: e = A for every (domain, isometry); first is (0, 0, j_zero)
        best.e = W.A;
        best.d = 0;
        best.kj = P.j_zero;
    } else {
        best.e = INFINITY;
        best.d = INT_MAX;
        best.kj = INT_MAX;
    }
    float thr = P.has_zero ? fminf(__double2float_ru(W.margin), FLT_MAX) : FLT_MAX;
    if (!rvalid) thr = -FLT_MAX;
    unsigned n_exact = 0;
    __syncthreads();

    int iacc[4][8];
    for (int s = 0; s < nstages; ++s) {
        const int buf = s & 1;
        mbar_wait(&bar[buf], (uint32_t)((s >> 1) & 1));
        const float *D = Ds + buf * Cf::STAGE_F;
        int tile_first, nt;
        if (n <= 64) {
            tile_first = t0 + s * TPS;
            nt = min(t1 - tile_first, TPS);
        } else {
            tile_first = t0 + s / NCH;
            nt = 1;
        }
        for (int tt = 0; tt < nt; ++tt) {
            float acc[4][8];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int k = 0; k < 8; ++k) acc[i][k] = 0.f;
            const float *Dtile = D + tt * Cf::KC * kTileD;
            const float *Rp = Rw + (n <= 64 ? 0 : (s % NCH) * 64 * 8);
#pragma unroll
            for (int p = 0; p < Cf::KC; ++p) {
                const float4 dv = *reinterpret_cast<const float4 *>(Dtile + p * kTileD + 4 * lane);
                const float4 ra = *reinterpret_cast<const float4 *>(Rp + p * 8);
                const float4 rb = *reinterpret_cast<const float4 *>(Rp + p * 8 + 4);
                const float dd[4] = {dv.x, dv.y, dv.z, dv.w};
                const float rr[8] = {ra.x, ra.y, ra.z, ra.w, rb.x, rb.y, rb.z, rb.w};
#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                    for (int k = 0; k < 8; ++k) acc[i][k] = fmaf(dd[i], rr[k], acc[i][k]);
            }
            bool last;
            float mx[4];
            if constexpr (n <= 64) {
                // sums of <= 64 products of exact integers < 2^24: the fp32 values are exact
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    float m = acc[i][0];
#pragma unroll
                    for (int k = 1; k < 8; ++k) m = fmaxf(m, acc[i][k]);
                    mx[i] = m;
                }
                last = true;
            } else {
                const int ch = s % NCH;
#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                    for (int k = 0; k < 8; ++k)
                        iacc[i][k] = (ch == 0 ? 0 : iacc[i][k]) + __float2int_rn(acc[i][k]);
                last = ch == NCH - 1;
                if (last) {
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        int m = iacc[i][0];
#pragma unroll
                        for (int k = 1; k < 8; ++k) m = max(m, iacc[i][k]);
                        mx[i] = __int2float_rn(m);
                    }
                }
            }
            if (last) {
                // ---- epilogue: filter every (range, domain) of this tile, exact path if needed
                const int tile = tile_first + tt;
                const int d0 = tile * kTileD + 4 * lane;
                const float4 sdf4 = *reinterpret_cast<const float4 *>(P.SDf + d0);
                const float sdf[4] = {sdf4.x, sdf4.y, sdf4.z, sdf4.w};
                bool pass[4] = {false, false, false, false};
#pragma unroll
                for (int jj = 0; jj < NSP; ++jj) {
                    if (jj < P.nsp) {
                        const float4 t4 = *reinterpret_cast<const float4 *>(P.t2f + jj * n_slots + d0);
                        const float tv[4] = {t4.x, t4.y, t4.z, t4.w};
#pragma unroll
                        for (int i = 0; i < 4; ++i) {
                            const float base = fmaf(W.hsSR[jj], sdf[i], tv[i]);
                            const float g = fmaf(-W.hsn[jj], mx[i], base);
                            pass[i] = pass[i] || (g <= thr);
                        }
                    }
                }
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    if (pass[i]) {
                        int srd[8];
                        if constexpr (n <= 64) {
#pragma unroll
                            for (int k = 0; k < 8; ++k) srd[k] = __float2int_rn(acc[i][k]);
                        } else {
#pragma unroll
                            for (int k = 0; k < 8; ++k) srd[k] = iacc[i][k];
                        }
                        exact_update<NSP>(P, n, d0 + i, srd, W, best, thr);
                        ++n_exact;
                    }
                }
            }
        }
        __syncthreads();
        if (threadIdx.x == 0 && s + 2 < nstages) {
            fence_proxy_async();
            issue(s + 2);
        }
    }

    // ---- warp lexicographic min, one partial per (range, split)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const double oe = __shfl_xor_sync(0xffffffffu, best.e, o);
        const int od = __shfl_xor_sync(0xffffffffu, best.d, o);
        const int okj = __shfl_xor_sync(0xffffffffu, best.kj, o);
        if (lex_less(oe, od, okj, best)) { best.e = oe; best.d = od; best.kj = okj; }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) n_exact += __shfl_xor_sync(0xffffffffu, n_exact, o);
    if (lane == 0 && rvalid) {
        Partial pb;
        pb.e = best.e;
        pb.d = best.d;
        pb.kj = best.kj;
        P.part[(size_t)r * P.ns_cap + split] = pb;
        if (P.exact_count && n_exact) atomicAdd(P.exact_count, (unsigned long long)n_exact);
    }
}

template <int B, int NSP>
static cudaError_t launch_search_t(const SearchParams &p, cudaStream_t st) {
    using Cf = SCfg<B>;
    static bool attr = false;
    if (!attr) {
        cudaError_t e = cudaFuncSetAttribute(search_kernel<B, NSP>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Cf::SMEM);
        if (e != cudaSuccess) return e;
        attr = true;
    }
    dim3 grid((unsigned)((p.n_r + 7) / 8), (unsigned)p.nsplit);
    search_kernel<B, NSP><<<grid, 256, Cf::SMEM, st>>>(p);
    return cudaGetLastError();
}

template <int B>
static cudaError_t launch_search_b(int32_t nsp, const SearchParams &p, cudaStream_t st) {
    if (nsp <= 1) return launch_search_t<B, 1>(p, st);
    if (nsp <= 2) return launch_search_t<B, 2>(p, st);
    return launch_search_t<B, 16>(p, st);
}

cudaError_t launch_search(int32_t B, int32_t nsp, const SearchParams &p, cudaStream_t st) {
    if (p.n_r == 0 || p.nsplit == 0) return cudaSuccess;  // n_r: upper bound
    switch (B) {
    case 2: return launch_search_b<2>(nsp, p, st);
    case 4: return launch_search_b<4>(nsp, p, st);
    case 8: return launch_search_b<8>(nsp, p, st);
    case 16: return launch_search_b<16>(nsp, p, st);
    default: return cudaErrorInvalidValue;
    }
}

int search_nsplit_hint(int32_t B, int64_t n_r, int64_t n_tiles, int num_sms) {
    const int occ = B >= 16 ? 1 : (B >= 8 ? 2 : 3);
    const int64_t gx = (n_r + 7) / 8;
    if (gx <= 0 || n_tiles <= 0) return 1;
    const int64_t target = (int64_t)num_sms * occ * 2;
    int64_t ns = (target + gx - 1) / gx;
    if (ns < 1) ns = 1;
    if (ns > n_tiles) ns = n_tiles;
    if (ns > 65535) ns = 65535;
    return (int)ns;
}

// ----------------------------------------------------------------------------- finalize
// Thread per range: merge the split partials (+ the s = 0 seed), then Eq. (3) offset, the o
// code [R11], E = e / n, the accept test [R14], the record, and the child marks.
__device__ __forceinline__ int o_code_dev(double o) {
    const double w = 1.9921875;  // 510 / 256
    if (o >= 0.0) {
        const double mu = __ddiv_rn(o, w);
        int j = (mu == 0.0) ? 0 : (int)ceil(mu) - 1;
        return 128 + min(j, 127);
    }
    const double mu = __ddiv_rn(-o, w);
    const int j = (int)ceil(mu) - 1;
    return 127 - min(j, 127);
}

// k* of the winning (range, domain) when the search deferred it: all 8 SRD_k in integers with
// the isometry convention of the oracle (reading R2: T_k(D)(i,j) = D(f_k(i,j)), b = B - 1),
// lowest index of the maximum.
__device__ __noinline__ int kstar_dev(const FinalizeParams &P, int2 rr, int32_t d) {
    const int B = P.B, b = B - 1;
    const int32_t c = P.kept[d];
    const int64_t x0 = (int64_t)(c % P.A) * P.L, y0 = (int64_t)(c / P.A) * P.L;
    if (B == 2) {  // (the B = 2 closed form defers k*): 4 range and 16 domain pixels loaded once
        const uint8_t *rp = P.img + (size_t)rr.y * P.N + rr.x;
        const long long r00 = rp[0], r01 = rp[1], r10 = rp[P.N], r11 = rp[P.N + 1];
        long long D[2][2];
        for (int i = 0; i < 2; ++i)
            for (int j = 0; j < 2; ++j) {
                const uint8_t *q = P.img + (y0 + 2 * i) * P.N + x0 + 2 * j;
                D[i][j] = (int)q[0] + (int)q[1] + (int)q[P.N] + (int)q[P.N + 1];
            }
        // SRD_k = sum_ij R(i,j) D(f_k(i,j)) with the isometry convention below (b = 1)
        long long srd[8];
        srd[0] = r00 * D[0][0] + r01 * D[0][1] + r10 * D[1][0] + r11 * D[1][1];
        srd[1] = r00 * D[1][0] + r01 * D[0][0] + r10 * D[1][1] + r11 * D[0][1];
        srd[2] = r00 * D[1][1] + r01 * D[1][0] + r10 * D[0][1] + r11 * D[0][0];
        srd[3] = r00 * D[0][1] + r01 * D[1][1] + r10 * D[0][0] + r11 * D[1][0];
        srd[4] = r00 * D[0][1] + r01 * D[0][0] + r10 * D[1][1] + r11 * D[1][0];
        srd[5] = r00 * D[0][0] + r01 * D[1][0] + r10 * D[0][1] + r11 * D[1][1];
        srd[6] = r00 * D[1][0] + r01 * D[1][1] + r10 * D[0][0] + r11 * D[0][1];
        srd[7] = r00 * D[1][1] + r01 * D[0][1] + r10 * D[1][0] + r11 * D[0][0];
        int ks = 0;
        for (int k = 1; k < 8; ++k)
            if (srd[k] > srd[ks]) ks = k;
        return ks;
    }
    auto Dp = [&](int i, int j) {  // decimated domain value D'(i, j)
        const uint8_t *q = P.img + (y0 + 2 * i) * P.N + x0 + 2 * j;
        return (int)q[0] + (int)q[1] + (int)q[P.N] + (int)q[P.N + 1];
    };
    long long best = LLONG_MIN;
    int ks = 0;
    for (int k = 0; k < 8; ++k) {
        long long s = 0;
        for (int i = 0; i < B; ++i)
            for (int j = 0; j < B; ++j) {
                int si = i, sj = j;
                switch (k) {
                case 1: si = b - j; sj = i; break;
                case 2: si = b - i; sj = b - j; break;
                case 3: si = j; sj = b - i; break;
                case 4: si = i; sj = b - j; break;
                case 5: si = j; sj = i; break;
                case 6: si = b - i; sj = j; break;
                case 7: si = b - j; sj = b - i; break;
                default: break;
                }
                s += (long long)P.img[(size_t)(rr.y + i) * P.N + rr.x + j] * Dp(si, sj);
            }
        if (s > best) { best = s; ks = k; }
    }
    return ks;
}

__global__ void finalize_kernel(const __grid_constant__ FinalizeParams P) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= (int)*P.d_nr) return;
    if (P.d_misc[0] == 0) {  // ranges but no domain block survived the entropy filter
        if (r == 0) *P.d_err = FIC_ERR_EMPTY_POOL;
        return;
    }
    const int2 rr = P.ranges[r];
    const int B = P.B, n = B * B;
    long long sr = 0, srr = 0;
    const uint8_t *rb = P.img + (size_t)rr.y * P.N + rr.x;
    if (B >= 4 && ((reinterpret_cast<uintptr_t>(P.img) | (uintptr_t)P.N) & 15) == 0) {
        // rows of B bytes at 16-byte aligned bases (rr.x % B == 0): independent word loads and
        // byte dot products (sum <= 65280, sum of squares <= 16.6e6: exact in 32 bits)
        unsigned s1 = 0, s2 = 0;
        for (int i = 0; i < B; ++i) {
            const uint32_t *row = reinterpret_cast<const uint32_t *>(rb + (size_t)i * P.N);
            if (B == 16) {
                const uint4 v = *reinterpret_cast<const uint4 *>(row);
                const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                for (int q = 0; q < 4; ++q) { s1 = __dp4a(w[q], 0x01010101u, s1); s2 = __dp4a(w[q], w[q], s2); }
            } else {
                for (int q = 0; q < B / 4; ++q) { const uint32_t w = row[q]; s1 = __dp4a(w, 0x01010101u, s1); s2 = __dp4a(w, w, s2); }
            }
        }
        sr = s1;
        srr = s2;
    } else {
        for (int i = 0; i < B; ++i) {
            const uint8_t *row = rb + (size_t)i * P.N;
            for (int j = 0; j < B; ++j) {
                const int v = row[j];
                sr += v;
                srr += v * v;
            }
        }
    }
    Best best;
    if (P.has_zero) {
        best.e = (double)((long long)n * srr - sr * sr);
        best.d = 0;
        best.kj = P.j_zero;
    } else {
        best.e = INFINITY;
        best.d = INT_MAX;
        best.kj = INT_MAX;
    }
    const int ns = P.nsplit > 0 ? (int)*P.d_ns : 0;
    for (int sp = 0; sp < ns; ++sp) {
        const Partial c = P.part[(size_t)r * P.nsplit + sp];
        if (lex_less(c.e, c.d, c.kj, best)) { best.e = c.e; best.d = c.d; best.kj = c.kj; }
    }
    if (best.kj & kPendIso) best.kj = (kstar_dev(P, rr, best.d) << 8) | (best.kj & 255);
    const int d = best.d, k = best.kj >> 8, j = best.kj & 255;
    // n = B^2 is a power of two: the divisions by n and 4n are exact scalings (bit-identical
    // to __ddiv_rn), done as multiplications
    const double inv_n = 1.0 / (double)n;
    const double E = best.e * inv_n;
    const double s = P.s[j];
    const double Rbar = (double)sr * inv_n;
    const double Dbar = (double)P.SD[d] * (0.25 * inv_n);
    const double o = __dsub_rn(Rbar, __dmul_rn(s, Dbar));
    const bool acc = P.is_min || E <= __dmul_rn(__dmul_rn(P.rms_tol, P.rms_tol), (double)n);
    const int32_t cand = P.kept[d];
    fic_record rec;
    rec.rx = rr.x;
    rec.ry = rr.y;
    rec.B = B;
    rec.dom = d;
    rec.dx = (cand % P.A) * P.L;
    rec.dy = (cand / P.A) * P.L;
    rec.iso = (uint8_t)k;
    rec.s_idx = (uint8_t)j;
    rec.o_code = (uint8_t)o_code_dev(o);
    rec.accepted = (uint8_t)acc;
    rec.err = E;
    // write as 5 x 8 bytes (padding bytes zero)
    uint64_t w[5] = {0, 0, 0, 0, 0};
    memcpy(w, &rec, 28);
    memcpy(&w[4], &rec.err, 8);
    fic_record *slot = P.rec + r;
    if (P.out_direct) {  // last level: every range is accepted, in range order
        if (r == 0) *P.d_level_count = (unsigned long long)*P.d_nr;
        const int64_t o = (int64_t)*P.d_base + r;
        slot = o < P.capacity ? P.out_direct + o : nullptr;
    } else {
        P.accepted[r] = (uint8_t)acc;
    }
    if (slot) {
        uint64_t *dst = reinterpret_cast<uint64_t *>(slot);
#pragma unroll
        for (int q = 0; q < 5; ++q) dst[q] = w[q];
    }
    if (!acc && P.child) {
        const int h = B / 2;
        const int64_t Gc = P.N / h;
        const int64_t cu = rr.x / h, cv = rr.y / h;
        P.child[cv * Gc + cu] = 1;
        P.child[cv * Gc + cu + 1] = 1;
        P.child[(cv + 1) * Gc + cu] = 1;
        P.child[(cv + 1) * Gc + cu + 1] = 1;
    }
}

cudaError_t launch_finalize(const FinalizeParams &p, cudaStream_t st) {
    if (p.n_r == 0) return cudaSuccess;
    finalize_kernel<<<(unsigned)((p.n_r + 127) / 128), 128, 0, st>>>(p);
    return cudaGetLastError();
}

}  // namespace fic
