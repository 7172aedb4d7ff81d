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
// fp32 evaluation is exact.  The score filter and the exact path are those of fic_fourier.cu:
// an fp32 lower bound of every binary64 score with a rigorous margin; surviving pairs are
// re-scored exactly (all 8 SRD_k in integers, canonical binary64 Eq. 1/3, lexicographic
// first-min).  Result identical to the oracle's exhaustive loop.
#include <cfloat>
#include <climits>
#include <cmath>
#include <cstdlib>
#include <cstring>

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

// Domain features: float4 (Y2, yr + yi, yr - yi, C) per slot; zero on pads (t2 = +inf excludes them).
__global__ void b2_pool_kernel(const uint8_t *__restrict__ img, int32_t N, int32_t L, int32_t A,
                               const int32_t *__restrict__ kept, const unsigned long long *__restrict__ d_nk,
                               int64_t n_slots, float4 *__restrict__ F) {
    const int64_t d = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (d >= n_slots) return;
    const int64_t n_k = (int64_t)*d_nk;
    if (d >= ((n_k + kTileD - 1) / kTileD) * kTileD) return;
    if (d >= n_k) {
        F[d] = make_float4(0.f, 0.f, 0.f, 0.f);
        return;
    }
    const int32_t c = kept[d];
    const int64_t x0 = (int64_t)(c % A) * L, y0 = (int64_t)(c / A) * L;
    auto dp = [&](int i, int j) {
        const uint8_t *q = img + (y0 + 2 * i) * N + x0 + 2 * j;
        return (int)q[0] + (int)q[1] + (int)q[N] + (int)q[N + 1];
    };
    const int w = dp(0, 0), x = dp(0, 1), y = dp(1, 1), z = dp(1, 0);
    const int sd = w + x + y + z;
    const int cc = 4 * (w * w + x * x + y * y + z * z) - sd * sd;  // C = n SDD - SD^2 < 2^24
    const int yr = abs(w - y), yi = abs(x - z);
    F[d] = make_float4((float)(w - x + y - z), (float)(yr + yi), (float)(yr - yi), (float)cc);
}

cudaError_t launch_b2_pool(const uint8_t *img, int32_t N, int32_t L, int32_t A, const int32_t *kept,
                           const unsigned long long *d_nk, int64_t n_slots, float4 *F, cudaStream_t st) {
    if (n_slots == 0) return cudaSuccess;
    b2_pool_kernel<<<(unsigned)((n_slots + 255) / 256), 256, 0, st>>>(img, N, L, A, kept, d_nk, n_slots, F);
    return cudaGetLastError();
}

struct B2Params {
    const uint8_t *img;
    int32_t N, L, A;
    const int2 *ranges;
    int32_t n_r;
    const float4 *F;       // [n_slots]
    const float *U;        // [n_tiles][nsp][128] t2_j
    const int64_t *C;      // [n_slots]
    const int32_t *kept;
    const unsigned long long *d_nr, *d_misc;  // device sizes: n_r; n_kept, Cmax
    int32_t nsplit;
    int32_t nsp;
    double spos[kMaxS];
    int32_t jpos[kMaxS];
    int32_t has_zero, j_zero;
    double smax;
    Partial *part;
    unsigned long long *exact_count;
    float *gthr;  // [n_r] threshold shared by all domain splits (CAS-min), initialised to ~FLT_MAX
    unsigned long long *d_ns;
    int32_t ns_cap;
};

struct B2Cold {
    double A, margin, best_e;
    int32_t best_d, best_kj;
    int32_t px;  // range pixels a, b, c, d packed as bytes (TL, TR, BR, BL)
    int32_t SR;
};

// filter margin of one range (e units): |Bq| <= sqrt(A C); fp32 -hs and t2 roundings and one
// FFMA -> 4u (hs |Bq| + t2); shared by the search and the threshold seeding (must be identical)
__device__ __forceinline__ double b2_margin(double A, double smax, double cmax) {
    const double u = 5.9604644775390625e-08;
    const double hs = 0.5 * smax, t2m = smax * smax * cmax * 0.0625;
    return 4.0 * u * (hs * sqrt(A * cmax) * 1.01 + t2m) + 1e-12 * (A + t2m) + 1e-30;
}

constexpr int kB2TPS = 4;   // tiles per stage
constexpr int kB2RPT = 4;   // ranges per thread
constexpr int kB2Threads = 256;

// k* of one (range, domain): all 8 SRD_k in integers (isometry convention of the oracle,
// reading R2), lowest index of the maximum.  Only called when the pair improves the best.
__device__ __noinline__ int b2_kstar(const B2Params &P, int32_t px, int32_t d) {
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
    const int a = px & 255, b = (px >> 8) & 255, cc = (px >> 16) & 255, dd = (px >> 24) & 255;
    const int R[2][2] = {{a, b}, {dd, cc}};
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

// exact path: canonical binary64 score for every s > 0 from the exact max_k Bq_k and C
// (no memory traffic); only a genuine lexicographic improvement fetches k* and publishes the
// new threshold (per thread and, CAS-min, across domain splits)
__device__ __noinline__ float b2_exact(const B2Params &P, B2Cold *cdp, float thr, int r, int32_t d,
                                       float bqf, float cf) {
    B2Cold &cd = *cdp;
    const double Bq = (double)bqf, c16 = __dmul_rn(0.0625, (double)cf);
    double e0 = INFINITY;
    int j0 = 0;
    for (int jj = 0; jj < P.nsp; ++jj) {
        const double s = P.spos[jj];
        const double e = __dadd_rn(__dsub_rn(cd.A, __dmul_rn(__dmul_rn(0.5, s), Bq)),
                                   __dmul_rn(__dmul_rn(s, s), c16));
        if (e < e0) { e0 = e; j0 = jj; }  // lowest j among equal e (same k* for every s > 0)
    }
    if (e0 > cd.best_e || (e0 == cd.best_e && d > cd.best_d)) return thr;
    const int ks = b2_kstar(P, cd.px, d);
    const int32_t kj = (ks << 8) | P.jpos[j0];
    if (e0 == cd.best_e && d == cd.best_d && kj >= cd.best_kj) return thr;
    cd.best_e = e0;
    cd.best_d = d;
    cd.best_kj = kj;
    const float t = fminf(__double2float_ru(__dadd_rn(__dsub_rn(e0, cd.A), cd.margin)), FLT_MAX);
    int *gi = reinterpret_cast<int *>(P.gthr + r);
    int old = *gi;
    while (t < __int_as_float(old)) {
        const int prev = atomicCAS(gi, old, __float_as_int(t));
        if (prev == old) break;
        old = prev;
    }
    return fminf(thr, t);
}

template <int NSP>
__global__ void __launch_bounds__(kB2Threads) b2search_kernel(const __grid_constant__ B2Params P) {
    constexpr int RPT = kB2RPT, TPS = kB2TPS;
    constexpr int FST = TPS * kTileD;  // float4 per stage
    extern __shared__ __align__(128) unsigned char smem[];
    float4 *Fs = reinterpret_cast<float4 *>(smem);             // [2][FST]
    float *Us = reinterpret_cast<float *>(Fs + 2 * FST);        // [2][TPS][nsp][128]
    B2Cold *cold = reinterpret_cast<B2Cold *>(Us + 2 * TPS * NSP * kTileD);  // [RPT][threads]
    uint64_t *bar = reinterpret_cast<uint64_t *>(cold + RPT * kB2Threads);

    const int n_r = (int)*P.d_nr;
    const int n_tiles = (int)((P.d_misc[0] + kTileD - 1) / kTileD);
    const double cmax = (double)P.d_misc[1];
    int group, split, ns;
    if (!cta_work(n_r, kB2Threads * RPT, n_tiles, 2 * TPS, P.ns_cap, group, split, ns)) return;
    if (group == 0 && split == 0 && threadIdx.x == 0) *P.d_ns = (unsigned long long)ns;
    const int t0 = (int)(((int64_t)split * n_tiles) / ns);
    const int t1 = (int)(((int64_t)(split + 1) * n_tiles) / ns);
    const int nstages = (max(0, t1 - t0) + TPS - 1) / TPS;
    auto issue = [&](int s) {
        const int buf = s & 1;
        const int ta = t0 + s * TPS, tb = min(t1, ta + TPS);
        const uint32_t b1 = (uint32_t)(tb - ta) * kTileD * 16;
        const uint32_t b2 = (uint32_t)(tb - ta) * P.nsp * kTileD * 4;
        b2_expect(&bar[buf], b1 + b2);
        b2_bulk(Fs + buf * FST, P.F + (size_t)ta * kTileD, b1, &bar[buf]);
        b2_bulk(Us + buf * TPS * NSP * kTileD, P.U + (size_t)ta * P.nsp * kTileD, b2, &bar[buf]);
    };
    if (threadIdx.x == 0) {
        b2_bar_init(&bar[0]);
        b2_bar_init(&bar[1]);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        if (nstages > 0) issue(0);
        if (nstages > 1) issue(1);
    }

    float X2d[RPT], sx[RPT], dx[RPT], thr[RPT];  // 2 X2, xr2 + xi2, xr2 - xi2
    const int rbase = (group * kB2Threads + threadIdx.x) * RPT;
#pragma unroll
    for (int q = 0; q < RPT; ++q) {
        const int r = rbase + q;
        B2Cold &cd = cold[q * kB2Threads + threadIdx.x];
        int a = 0, b = 0, c = 0, d = 0;
        if (r < n_r) {
            const int2 rr = P.ranges[r];
            const uint8_t *p0 = P.img + (size_t)rr.y * P.N + rr.x;
            a = p0[0]; b = p0[1]; d = p0[P.N]; c = p0[P.N + 1];
        }
        X2d[q] = (float)(2 * (a - b + c - d));
        sx[q] = (float)(2 * abs(a - c) + 2 * abs(b - d));
        dx[q] = (float)(2 * abs(a - c) - 2 * abs(b - d));
        const int sr = a + b + c + d, srr = a * a + b * b + c * c + d * d;
        cd.A = (double)(4 * srr - sr * sr);
        cd.SR = sr;
        cd.px = a | (b << 8) | (c << 16) | (d << 24);
        cd.margin = b2_margin(cd.A, P.smax, cmax);
        if (P.has_zero) { cd.best_e = cd.A; cd.best_d = 0; cd.best_kj = P.j_zero; }
        else { cd.best_e = INFINITY; cd.best_d = INT_MAX; cd.best_kj = INT_MAX; }
        float th = P.has_zero ? fminf(__double2float_ru(cd.margin), FLT_MAX) : FLT_MAX;
        thr[q] = r < n_r ? th : -FLT_MAX;
    }
    float nhs[NSP];
#pragma unroll
    for (int jj = 0; jj < NSP; ++jj) nhs[jj] = jj < P.nsp ? -__double2float_rn(0.25 * P.spos[jj]) : 0.f;  // x 2 Bq
    unsigned n_exact = 0;

    for (int s = 0; s < nstages; ++s) {
        const int buf = s & 1;
        b2_wait(&bar[buf], (uint32_t)((s >> 1) & 1));
#pragma unroll
        for (int q = 0; q < RPT; ++q)
            if (rbase + q < n_r) thr[q] = fminf(thr[q], P.gthr[rbase + q]);
        const float4 *Fb = Fs + buf * FST;
        const float *Ub = Us + buf * TPS * NSP * kTileD;
        const int ta = t0 + s * TPS;
        const int nt = min(t1 - ta, TPS);
        for (int tt = 0; tt < nt; ++tt) {
            const float4 *Ft = Fb + tt * kTileD;
            const float *Ut = Ub + tt * P.nsp * kTileD;
            const int dbase = (ta + tt) * kTileD;
#pragma unroll 2
            for (int dl0 = 0; dl0 < kTileD; dl0 += 2) {
                // two domains per block: the filters of 2 x RPT pairs interleave, one branch
                float4 f2[2];
                float t2v[2][NSP];
                float mn[2];
                float gq[2][RPT], bqq[2][RPT];
#pragma unroll
                for (int u2 = 0; u2 < 2; ++u2) {
                    f2[u2] = Ft[dl0 + u2];
#pragma unroll
                    for (int jj = 0; jj < NSP; ++jj)
                        t2v[u2][jj] = jj < P.nsp ? Ut[jj * kTileD + dl0 + u2] : INFINITY;
                    mn[u2] = 1.0f;  // min over ranges of (lower bound - threshold): <= 0 -> some pass
#pragma unroll
                    for (int q = 0; q < RPT; ++q) {
                        const float4 f = f2[u2];
                        const float bq = fmaf(sx[q], f.y, fabsf(fmaf(X2d[q], f.x, dx[q] * f.z)));  // 2 max_k Bq_k
                        float g = fmaf(nhs[0], bq, t2v[u2][0]);
#pragma unroll
                        for (int jj = 1; jj < NSP; ++jj) g = fminf(g, fmaf(nhs[jj], bq, t2v[u2][jj]));
                        gq[u2][q] = g;
                        bqq[u2][q] = bq;
                        mn[u2] = fminf(mn[u2], g - thr[q]);
                    }
                }
                if (fminf(mn[0], mn[1]) <= 0.0f) {
#pragma unroll
                    for (int u2 = 0; u2 < 2; ++u2) {
#pragma unroll
                        for (int q = 0; q < RPT; ++q) {
                            if (gq[u2][q] <= thr[q]) {
                                thr[q] = b2_exact(P, &cold[q * kB2Threads + threadIdx.x], thr[q], rbase + q,
                                                  dbase + dl0 + u2, 0.5f * bqq[u2][q], f2[u2].w);
                                ++n_exact;
                            }
                        }
                    }
                }
                __syncwarp();  // reconverge after the (rare, divergent) exact path
            }
        }
        __syncthreads();
        if (threadIdx.x == 0 && s + 2 < nstages) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            issue(s + 2);
        }
    }
#pragma unroll
    for (int q = 0; q < RPT; ++q) {
        const int r = rbase + q;
        if (r < n_r) {
            const B2Cold &cd = cold[q * kB2Threads + threadIdx.x];
            Partial pb;
            pb.e = cd.best_e;
            pb.d = cd.best_d;
            pb.kj = cd.best_kj;
            P.part[(size_t)r * P.ns_cap + split] = pb;
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) n_exact += __shfl_xor_sync(0xffffffffu, n_exact, o);
    if ((threadIdx.x & 31) == 0 && n_exact && P.exact_count) atomicAdd(P.exact_count, (unsigned long long)n_exact);
}

// Threshold seeding: each range's exact best over a strided sample of kS domains is an upper
// bound of its final best, so RU(best - A + margin) is a valid initial shared threshold.
constexpr int kS = 32;
__global__ void b2_seed_kernel(const __grid_constant__ B2Params P) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    const int n_r = (int)*P.d_nr;
    if (r >= n_r) return;
    const int64_t n_k = (int64_t)P.d_misc[0];
    if (n_k == 0) return;
    const double cmax = (double)P.d_misc[1];
    const int2 rr = P.ranges[r];
    const uint8_t *p0 = P.img + (size_t)rr.y * P.N + rr.x;
    const int a = p0[0], b = p0[1], d = p0[P.N], c = p0[P.N + 1];
    const float X2d = (float)(2 * (a - b + c - d));
    const float sx = (float)(2 * abs(a - c) + 2 * abs(b - d));
    const float dx = (float)(2 * abs(a - c) - 2 * abs(b - d));
    const int sr = a + b + c + d, srr = a * a + b * b + c * c + d * d;
    const double A = (double)(4 * srr - sr * sr);
    double best = P.has_zero ? A : INFINITY;
    for (int i = 0; i < kS; ++i) {
        const int64_t dd = (i * n_k) / kS;
        const float4 f = P.F[dd];
        const double Bq = 0.5 * (double)fmaf(sx, f.y, fabsf(fmaf(X2d, f.x, dx * f.z)));  // exact
        const double c16 = __dmul_rn(0.0625, (double)f.w);
        for (int jj = 0; jj < P.nsp; ++jj) {
            const double s = P.spos[jj];
            const double e = __dadd_rn(__dsub_rn(A, __dmul_rn(__dmul_rn(0.5, s), Bq)),
                                       __dmul_rn(__dmul_rn(s, s), c16));
            best = fmin(best, e);
        }
    }
    if (best < INFINITY)
        P.gthr[r] = fminf(__double2float_ru(__dadd_rn(__dsub_rn(best, A), b2_margin(A, P.smax, cmax))), FLT_MAX);
}

template <int NSP>
static cudaError_t launch_b2_t(const B2Params &p, cudaStream_t st) {
    const size_t smem = (size_t)2 * kB2TPS * kTileD * 16 + (size_t)2 * kB2TPS * NSP * kTileD * 4 +
                        sizeof(B2Cold) * kB2RPT * kB2Threads + 64;
    static bool attr = false;
    if (!attr) {
        cudaError_t e = cudaFuncSetAttribute(b2search_kernel<NSP>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)smem);
        if (e != cudaSuccess) return e;
        attr = true;
    }
    dim3 grid((unsigned)((p.n_r + kB2Threads * kB2RPT - 1) / (kB2Threads * kB2RPT)), (unsigned)p.nsplit);
    b2search_kernel<NSP><<<grid, kB2Threads, smem, st>>>(p);
    return cudaGetLastError();
}

int b2_nsplit_hint(int64_t n_r, int64_t n_tiles, int num_sms) {
    const int64_t gx = (n_r + kB2Threads * kB2RPT - 1) / (kB2Threads * kB2RPT);
    if (gx <= 0 || n_tiles <= 0) return 1;
    static int waves = [] {
        const char *e = getenv("FIC_B2_CTAS_PER_SM");
        return e ? atoi(e) : 8;
    }();
    int64_t ns = ((int64_t)num_sms * waves + gx - 1) / gx;
    const int64_t max_ns = (n_tiles + kB2TPS - 1) / kB2TPS;
    if (ns > max_ns) ns = max_ns;
    if (ns < 1) ns = 1;
    if (ns > 65535) ns = 65535;
    return (int)ns;
}

cudaError_t launch_b2_search(const SearchParams &sp, const float4 *F, const float *U, const int32_t *kept,
                             int32_t L, int32_t A, float *gthr, cudaStream_t st) {
    if (sp.n_r == 0 || sp.nsp == 0) return cudaSuccess;
    B2Params p;
    memset(&p, 0, sizeof p);
    p.img = sp.img; p.N = sp.N; p.L = L; p.A = A; p.ranges = sp.ranges; p.n_r = sp.n_r;
    p.F = F; p.U = U; p.C = sp.C; p.kept = kept;
    p.d_nr = sp.d_nr; p.d_misc = sp.d_misc; p.nsplit = sp.nsplit; p.d_ns = sp.d_ns; p.ns_cap = sp.ns_cap;
    p.nsp = sp.nsp;
    memcpy(p.spos, sp.spos, sizeof p.spos);
    memcpy(p.jpos, sp.jpos, sizeof p.jpos);
    p.has_zero = sp.has_zero; p.j_zero = sp.j_zero;
    p.smax = sp.smax;
    p.part = sp.part; p.exact_count = sp.exact_count;
    p.gthr = gthr;
    cudaError_t e = cudaMemsetAsync(gthr, 0x7f, sizeof(float) * (size_t)sp.n_r, st);  // ~3.4e38
    if (e != cudaSuccess) return e;
    b2_seed_kernel<<<(unsigned)((sp.n_r + 127) / 128), 128, 0, st>>>(p);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    if (sp.nsp <= 1) return launch_b2_t<1>(p, st);
    if (sp.nsp <= 2) return launch_b2_t<2>(p, st);
    return launch_b2_t<16>(p, st);
}

}  // namespace fic
