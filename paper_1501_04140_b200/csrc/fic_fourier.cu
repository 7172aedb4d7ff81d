// fic_fourier.cu -- the range x (domain, 8 isometries) search in the D4 group-Fourier basis
// (B = 2, 4, 8).  Same result as fic_search.cu, bit for bit; fewer operations.
//
// The 8 isometries (§2 line 28) form the dihedral group D4 acting on the B x B grid,
// and SRD_k = sum_p R(p) D'(f_k(p)) is, orbit by orbit, a correlation over that group.  With the
// real irreducible representations of D4 -- four 1-dimensional characters chi_c and the
// 2-dimensional representation M_h (signed permutation matrices, integer entries):
//     8 SRD_k = sum_c chi_c(k) c_c + 2 tr(M_k^T C2),
//     c_c   = sum_O rh_c(O) dh_c(O),            C2[i][j] = sum_O sum_l dh_il(O) rh_jl(O),
//     rh(O) = sum_{h in H_O} R(f_h p_O) rep(h),  dh(O) = sum_{h=0..7} D'(f_h p_O) rep(h),
// where O runs over the orbits of the grid (base point p_O; H_O one element per orbit point).
// That is 12 multiply-adds per orbit and (range, domain) -- 12 n/8..12 n/4 instead of 8 n -- and
// the 8 values pair up as base_k +- 2 t_k (k, k o rot180), so max_k SRD_k = max_k(base_k + 2|t_k|).
// Everything is integer-valued; R and D' are centred (R-128, D'-510) to keep fp32 sums small.
//
// The fp32 values only feed a FILTER with a rigorous error margin (DESIGN.md §"Exactness"):
// a (range, domain) pair whose lower bound cannot reach the running best is skipped; every other
// pair is re-evaluated exactly (binary64 on exact integers) with the canonical Eq. (1)/(3) score
// and the lexicographic first-min rule of the oracle.
#include <cfloat>
#include <climits>
#include <cmath>
#include <cstring>
#include <vector>

#include "fic_internal.cuh"

namespace fic {

constexpr int kOrbTotal = 14;  // 1 (B=2) + 3 (B=4) + 10 (B=8)
__host__ __device__ constexpr int orb_base(int B) { return B == 2 ? 0 : (B == 4 ? 1 : 4); }
__host__ __device__ constexpr int n_orbits(int B) { return B == 2 ? 1 : (B == 4 ? 3 : 10); }
template <int B>
struct FCfg {
    static constexpr int n = B * B;
    static constexpr int nO = n_orbits(B);
    static constexpr int NC = 8 * nO;                    // coefficients per block
    static constexpr int NCS = ((NC + 1 + 3) / 4) * 4;   // record stride (floats): coeffs, SD
};

__constant__ int8_t c_tab[8][8];           // [h][q]: q<4 chi_q(h); q>=4 M_h[(q-4)/2][(q-4)%2]
__constant__ int16_t c_orb_pts[kOrbTotal][8];
__constant__ uint8_t c_orb_H[kOrbTotal];   // bit h set: h is the first element reaching its point

// ------------------------------------------------------------------------------ host tables
static void host_iso_src(int B, int k, int i, int j, int &si, int &sj) {
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

struct HostTables {
    int8_t tab[8][8];
    int16_t pts[kOrbTotal][8];
    uint8_t H[kOrbTotal];
};

static bool build_tables(HostTables &T) {
    // M_h: f_h is affine; on B = 3 the centre is (1,1): columns = images of unit vectors
    int M[8][2][2];
    for (int h = 0; h < 8; ++h) {
        int a, b, c, d;
        host_iso_src(3, h, 2, 1, a, b);  // (i,j) = (1,1) + e_i
        host_iso_src(3, h, 1, 2, c, d);  // (1,1) + e_j
        M[h][0][0] = a - 1; M[h][1][0] = b - 1;
        M[h][0][1] = c - 1; M[h][1][1] = d - 1;
    }
    for (int h = 0; h < 8; ++h) {
        const int det = M[h][0][0] * M[h][1][1] - M[h][0][1] * M[h][1][0];
        const int diag = M[h][0][1] == 0 ? 1 : -1;
        T.tab[h][0] = 1;
        T.tab[h][1] = (int8_t)det;
        T.tab[h][2] = (int8_t)diag;
        T.tab[h][3] = (int8_t)(det * diag);
        T.tab[h][4] = (int8_t)M[h][0][0];
        T.tab[h][5] = (int8_t)M[h][0][1];
        T.tab[h][6] = (int8_t)M[h][1][0];
        T.tab[h][7] = (int8_t)M[h][1][1];
    }
    for (int B : {2, 4, 8}) {
        std::vector<char> seen(B * B, 0);
        int o = orb_base(B), cnt = 0;
        for (int i = 0; i < B; ++i)
            for (int j = 0; j < B; ++j) {
                if (seen[i * B + j]) continue;
                uint8_t Hm = 0;
                for (int h = 0; h < 8; ++h) {
                    int si, sj;
                    host_iso_src(B, h, i, j, si, sj);
                    const int p = si * B + sj;
                    T.pts[o][h] = (int16_t)p;
                    if (!seen[p]) {
                        seen[p] = 1;
                        Hm |= (uint8_t)(1u << h);
                    }
                }
                T.H[o] = Hm;
                ++o;
                ++cnt;
            }
        if (cnt != n_orbits(B)) return false;
    }
    return true;
}

// host self-test of the factorisation and of the pair combination used in the kernel
static bool self_test(const HostTables &T) {
    unsigned s = 12345u;
    auto rnd = [&](int m) {
        s = s * 1103515245u + 12345u;
        return (int)((s >> 8) % (unsigned)m);
    };
    for (int B : {2, 4, 8}) {
        const int n = B * B, nO = n_orbits(B), ob = orb_base(B);
        for (int trial = 0; trial < 8; ++trial) {
            std::vector<long long> R(n), D(n);
            for (int p = 0; p < n; ++p) { R[p] = rnd(256) - 128; D[p] = rnd(1021) - 510; }
            long long direct[8];
            for (int k = 0; k < 8; ++k) {
                long long acc = 0;
                for (int i = 0; i < B; ++i)
                    for (int j = 0; j < B; ++j) {
                        int si, sj;
                        host_iso_src(B, k, i, j, si, sj);
                        acc += R[i * B + j] * D[si * B + sj];
                    }
                direct[k] = acc;
            }
            long long c[4] = {0, 0, 0, 0}, C2[2][2] = {{0, 0}, {0, 0}};
            for (int o = 0; o < nO; ++o) {
                long long rh[8] = {0}, dh[8] = {0};
                for (int h = 0; h < 8; ++h)
                    for (int q = 0; q < 8; ++q) {
                        dh[q] += T.tab[h][q] * D[T.pts[ob + o][h]];
                        if (T.H[ob + o] >> h & 1) rh[q] += T.tab[h][q] * R[T.pts[ob + o][h]];
                    }
                for (int q = 0; q < 4; ++q) c[q] += rh[q] * dh[q];
                for (int i = 0; i < 2; ++i)
                    for (int j = 0; j < 2; ++j)
                        C2[i][j] += dh[4 + 2 * i] * rh[4 + 2 * j] + dh[5 + 2 * i] * rh[5 + 2 * j];
            }
            const long long b0 = (c[0] + c[1]) + (c[2] + c[3]), b1 = (c[0] + c[1]) - (c[2] + c[3]);
            const long long b4 = (c[0] - c[1]) + (c[2] - c[3]), b5 = (c[0] - c[1]) - (c[2] - c[3]);
            const long long t0 = C2[0][0] + C2[1][1], t1 = C2[1][0] - C2[0][1];
            const long long t4 = C2[0][0] - C2[1][1], t5 = C2[0][1] + C2[1][0];
            const long long v[8] = {b0 + 2 * t0, b1 + 2 * t1, b0 - 2 * t0, b1 - 2 * t1,
                                    b4 + 2 * t4, b5 + 2 * t5, b4 - 2 * t4, b5 - 2 * t5};
            for (int k = 0; k < 8; ++k)
                if (v[k] != 8 * direct[k]) return false;
        }
    }
    return true;
}

cudaError_t fourier_init() {
    HostTables T;
    if (!build_tables(T) || !self_test(T)) return cudaErrorInvalidValue;
    cudaError_t e = cudaMemcpyToSymbol(c_tab, T.tab, sizeof T.tab);
    if (e == cudaSuccess) e = cudaMemcpyToSymbol(c_orb_pts, T.pts, sizeof T.pts);
    if (e == cudaSuccess) e = cudaMemcpyToSymbol(c_orb_H, T.H, sizeof T.H);
    return e;
}

int fourier_record_stride(int B) {
    switch (B) {
    case 2: return FCfg<2>::NCS;
    case 4: return FCfg<4>::NCS;
    case 8: return FCfg<8>::NCS;
    default: return 0;
    }
}

// ----------------------------------------------------------------------- domain coefficients
// Warp per domain slot: D' (2x2 sums), SD, the centred-and-scaled block Dt = n D' - SD (so that
// sum_p R(p) Dt(f_k p) = n SRD_k - SR SD = Bq_k exactly, for any R), its 8 nO D4-Fourier
// coefficients (orbit-major: q = O*8 + component; exact integers |.| <= 8 n 1020 < 2^24) and
// their Euclidean norm rounded up (for the filter's Cauchy-Schwarz error bound) at slot NC.
template <int B>
__global__ void __launch_bounds__(256) pool_coeff_kernel(const uint8_t *__restrict__ img, int32_t N,
                                                         int32_t L, int32_t A,
                                                         const int32_t *__restrict__ kept,
                                                         const unsigned long long *__restrict__ d_nk,
                                                         int64_t n_slots, float *__restrict__ Dc,
                                                         unsigned int *__restrict__ d_dnmax) {
    using Cf = FCfg<B>;
    __shared__ int dsm[8][Cf::n];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t d = (int64_t)blockIdx.x * 8 + warp;
    if (d >= n_slots) return;
    const int64_t n_k = (int64_t)*d_nk;
    const int64_t ntiles = (n_k + kTileD - 1) / kTileD;
    if (d >= ntiles * kTileD) return;
    float *rec = Dc + d * Cf::NCS;
    if (d >= n_k) {
        for (int q = lane; q < Cf::NCS; q += 32) rec[q] = 0.f;
        return;
    }
    const int32_t c = kept[d];
    const int64_t x = (int64_t)(c % A) * L, y = (int64_t)(c / A) * L;
    int sd = 0;
    for (int p = lane; p < Cf::n; p += 32) {
        const int i = p / B, j = p % B;
        const uint8_t *q = img + (y + 2 * i) * N + x + 2 * j;
        const int v = (int)q[0] + (int)q[1] + (int)q[N] + (int)q[N + 1];
        dsm[warp][p] = v;
        sd += v;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sd += __shfl_xor_sync(0xffffffffu, sd, o);
    __syncwarp();
    for (int p = lane; p < Cf::n; p += 32) dsm[warp][p] = Cf::n * dsm[warp][p] - sd;
    __syncwarp();
    double nrm = 0.0;
    for (int q = lane; q < Cf::NC; q += 32) {
        const int o = q >> 3, comp = q & 7, ob = orb_base(B) + o;
        int acc = 0;
#pragma unroll
        for (int h = 0; h < 8; ++h) acc += c_tab[h][comp] * dsm[warp][c_orb_pts[ob][h]];
        rec[q] = (float)acc;
        nrm += (double)acc * (double)acc;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) nrm += __shfl_xor_sync(0xffffffffu, nrm, o);
    if (lane == 0) {
        const float dn = __double2float_ru(sqrt(nrm) * (1.0 + 1e-12));
        rec[Cf::NC] = dn;
        atomicMax(d_dnmax, __float_as_uint(dn));  // non-negative floats order as integers
    }
    for (int q = Cf::NC + 1 + lane; q < Cf::NCS; q += 32) rec[q] = 0.f;
}

cudaError_t launch_pool_coeff(const uint8_t *img, int32_t N, int32_t B, int32_t L, int32_t A,
                              const int32_t *kept, const unsigned long long *d_nk, int64_t n_slots,
                              float *Dc, unsigned int *d_dnmax, cudaStream_t st) {
    if (n_slots == 0) return cudaSuccess;
    const unsigned blocks = (unsigned)((n_slots + 7) / 8);
    switch (B) {
    case 2: pool_coeff_kernel<2><<<blocks, 256, 0, st>>>(img, N, L, A, kept, d_nk, n_slots, Dc, d_dnmax); break;
    case 4: pool_coeff_kernel<4><<<blocks, 256, 0, st>>>(img, N, L, A, kept, d_nk, n_slots, Dc, d_dnmax); break;
    case 8: pool_coeff_kernel<8><<<blocks, 256, 0, st>>>(img, N, L, A, kept, d_nk, n_slots, Dc, d_dnmax); break;
    default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

// U[tile][j][dl] = fp32 of t2_j = (s_j s_j)(C/16); +inf on pad slots (never admitted)
__global__ void fourier_u_kernel(const int64_t *__restrict__ C, const unsigned long long *__restrict__ d_nk,
                                 int64_t n_slots, const SList spos, int32_t nsp, float *__restrict__ U) {
    const int64_t d = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (d >= n_slots) return;
    const int64_t n_k = (int64_t)*d_nk;
    if (d >= ((n_k + kTileD - 1) / kTileD) * kTileD) return;
    const int64_t tile = d / kTileD, dl = d % kTileD;
    const double c16 = __dmul_rn(0.0625, (double)C[d]);
    for (int j = 0; j < nsp; ++j) {
        const double s = spos.s[j];
        U[(tile * nsp + j) * kTileD + dl] =
            d < n_k ? __double2float_rn(__dmul_rn(__dmul_rn(s, s), c16)) : INFINITY;
    }
}

cudaError_t launch_fourier_u(const int64_t *C, const unsigned long long *d_nk, int64_t n_slots, const SList &sl,
                             int32_t nsp, float *U, cudaStream_t st) {
    if (n_slots == 0 || nsp == 0) return cudaSuccess;
    fourier_u_kernel<<<(unsigned)((n_slots + 255) / 256), 256, 0, st>>>(C, d_nk, n_slots, sl, nsp, U);
    return cudaGetLastError();
}

// ------------------------------------------------------------------------------ range prep
struct RangeMeta {
    double A;       // n SRR - SR^2 (exact)
    double margin;  // filter margin in e units (rounding of the fp32 score + binary64 slack)
    float cr;       // Cauchy-Schwarz factor: |m8_f - 8 Bq_max| <= cr * |dh|_2
    int32_t pad;
};

// Thread per range: moments, centred coefficients rh of R - 128 (component-major over ranges:
// Rc[q][r]) and the per-range constants of the filter's rigorous error bound (DESIGN.md
// §"Exactness").  Because sum_p Dt = 0, sum_p (R(p) - 128) Dt(f_k p) = Bq_k.
template <int B>
__global__ void fourier_range_kernel(const uint8_t *__restrict__ img, int32_t N,
                                     const int2 *__restrict__ ranges, const unsigned long long *__restrict__ d_nr,
                                     int32_t r_stride, double smax,
                                     const unsigned long long *__restrict__ d_misc, float *__restrict__ Rc,
                                     RangeMeta *__restrict__ meta) {
    using Cf = FCfg<B>;
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= (int)*d_nr) return;
    const double t2max = smax * smax * (double)d_misc[1] * 0.0625 * (1.0 + 1e-12);
    double dnmax;
    {
        const unsigned int bits = (unsigned int)(d_misc[2] & 0xffffffffu);
        dnmax = (double)__uint_as_float(bits);
    }
    const int2 rr = ranges[r];
    int R[Cf::n];
    long long sr = 0, srr = 0;
#pragma unroll
    for (int p = 0; p < Cf::n; ++p) {
        const int v = img[(size_t)(rr.y + p / B) * N + rr.x + p % B];
        sr += v;
        srr += v * v;
        R[p] = v - 128;
    }
    double nr2 = 0.0;
    for (int o = 0; o < Cf::nO; ++o) {
        const int ob = orb_base(B) + o;
        const int Hm = c_orb_H[ob];
#pragma unroll
        for (int comp = 0; comp < 8; ++comp) {
            int acc = 0;
#pragma unroll
            for (int h = 0; h < 8; ++h)
                if (Hm >> h & 1) acc += c_tab[h][comp] * R[c_orb_pts[ob][h]];
            Rc[(size_t)(o * 8 + comp) * r_stride + r] = (float)acc;
            nr2 += (double)acc * (double)acc;
        }
    }
    const double u = 5.9604644775390625e-08;  // 2^-24
    const double nr = sqrt(nr2) * (1.0 + 1e-12);
    // every product feeding 8 Bq_k is rh_q dh_pi(q) with weight 1 or 2 (pi a permutation), so
    // sum |terms| <= 2 |rh|_2 |dh|_2; fp32 dot products + combination: gamma_{2 nO + 8}
    const double cr = (2.0 * Cf::nO + 8.0) * 1.02 * u * 2.0 * nr;
    const double hs = 0.5 * smax;
    const double m8max = 2.0 * nr * dnmax * 1.01 + cr * dnmax;  // |m8 + cr dn| bound
    const double A = (double)((long long)Cf::n * srr - sr * sr);
    RangeMeta m;
    m.A = A;
    // fp32: hs8 and t2 rounded, two FFMA roundings -> 4u (hs |m8p|/8 + t2); binary64 slack
    m.margin = 4.0 * u * (hs * m8max * 0.125 + t2max) + 1e-12 * (A + hs * m8max * 0.125 + t2max) + 1e-30;
    m.cr = __double2float_ru(cr);
    m.pad = 0;
    meta[r] = m;
}

// ------------------------------------------------------------------------------ search
__device__ __forceinline__ uint32_t smem_u32f(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void fmbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32f(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fmbar_fence_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void fmbar_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32f(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void fbulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32f(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32f(bar))
        : "memory");
}
__device__ __forceinline__ void fmbar_wait(uint64_t *bar, uint32_t parity) {
    uint32_t done = 0;
    while (!done) {
        asm volatile(
            "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
            : "=r"(done)
            : "r"(smem_u32f(bar)), "r"(parity)
            : "memory");
    }
}

struct FSearchParams {
    const float *Dc;       // [n_slots][NCS]
    const float *U;        // [n_tiles][nsp][128]  t2_j
    const int64_t *C;      // [n_slots]
    const float *Rc;       // [NC][r_stride]
    const RangeMeta *meta; // [n_r]
    const unsigned long long *d_nr, *d_misc;  // device sizes
    int32_t r_stride, nsplit;
    int32_t nsp;
    double spos[kMaxS];
    int32_t jpos[kMaxS];
    int32_t has_zero, j_zero;
    Partial *part;
    unsigned long long *exact_count;
};

// cold per-range state, in shared memory (touched only by the exact path)
struct FCold {
    double A, margin, best_e;
    int32_t best_d, best_kj;
};

__device__ __forceinline__ bool flex_less(double e, int32_t d, int32_t kj, double be, int32_t bd,
                                          int32_t bkj) {
    if (e < be) return true;
    if (e > be) return false;
    if (d != bd) return d < bd;
    return kj < bkj;
}

// Exact path of one (range, domain): the 8 values 8 Bq_k from the same coefficients in binary64
// (exact: integers < 2^53), k* = lowest argmax, Bq = 8 Bq_{k*} / 8, canonical binary64 score
// e = (A - (s/2) Bq) + (s s)(C/16) for every s > 0, lexicographic first-min update, and the
// refreshed fp32 thresholds thr_j = RU(best - A + margin).
template <int B, int NSP>
__device__ __forceinline__ void fexact(const FSearchParams &P, const float (&rc)[FCfg<B>::NC],
                                       const float *rec, int32_t d, FCold &cold, float (&thr)[NSP]) {
    using Cf = FCfg<B>;
    double c[4] = {0, 0, 0, 0}, C2[2][2] = {{0, 0}, {0, 0}};
#pragma unroll
    for (int o = 0; o < Cf::nO; ++o) {
        const float *dh = rec + o * 8;
        const float *rh = rc + o * 8;
#pragma unroll
        for (int q = 0; q < 4; ++q) c[q] = fma((double)rh[q], (double)dh[q], c[q]);
#pragma unroll
        for (int i = 0; i < 2; ++i)
#pragma unroll
            for (int j = 0; j < 2; ++j)
                C2[i][j] = fma((double)dh[4 + 2 * i], (double)rh[4 + 2 * j],
                               fma((double)dh[5 + 2 * i], (double)rh[5 + 2 * j], C2[i][j]));
    }
    const double b0 = (c[0] + c[1]) + (c[2] + c[3]), b1 = (c[0] + c[1]) - (c[2] + c[3]);
    const double b4 = (c[0] - c[1]) + (c[2] - c[3]), b5 = (c[0] - c[1]) - (c[2] - c[3]);
    const double t0 = C2[0][0] + C2[1][1], t1 = C2[1][0] - C2[0][1];
    const double t4 = C2[0][0] - C2[1][1], t5 = C2[0][1] + C2[1][0];
    const double v[8] = {b0 + 2 * t0, b1 + 2 * t1, b0 - 2 * t0, b1 - 2 * t1,
                         b4 + 2 * t4, b5 + 2 * t5, b4 - 2 * t4, b5 - 2 * t5};
    int ks = 0;
    double vm = v[0];
#pragma unroll
    for (int k = 1; k < 8; ++k)
        if (v[k] > vm) { vm = v[k]; ks = k; }
    const double Bq = vm * 0.125;  // exact: vm = 8 Bq_{k*}
    const double c16 = __dmul_rn(0.0625, (double)P.C[d]);
    double be = cold.best_e;
    int32_t bd = cold.best_d, bkj = cold.best_kj;
    for (int jj = 0; jj < P.nsp; ++jj) {
        const double s = P.spos[jj];
        const double hs = __dmul_rn(0.5, s);
        const double t2 = __dmul_rn(__dmul_rn(s, s), c16);
        const double e = __dadd_rn(__dsub_rn(cold.A, __dmul_rn(hs, Bq)), t2);
        const int32_t kj = (ks << 8) | P.jpos[jj];
        if (flex_less(e, d, kj, be, bd, bkj)) { be = e; bd = d; bkj = kj; }
    }
    cold.best_e = be;
    cold.best_d = bd;
    cold.best_kj = bkj;
    const float t = fminf(__double2float_ru(__dadd_rn(__dsub_rn(be, cold.A), cold.margin)), FLT_MAX);
#pragma unroll
    for (int jj = 0; jj < NSP; ++jj) thr[jj] = jj < P.nsp ? t : -FLT_MAX;
}

template <int B, int NSP, int RPT>
__global__ void __launch_bounds__(256, (B == 8 ? 1 : 2)) fsearch_kernel(const __grid_constant__ FSearchParams P) {
    using Cf = FCfg<B>;
    constexpr int NC = Cf::NC, NCS = Cf::NCS;
    constexpr int TILE_F = kTileD * NCS;                  // floats of one tile's records
    constexpr int TPS = (TILE_F * 4 >= 24 * 1024) ? 1 : (24 * 1024) / (TILE_F * 4);
    constexpr int STAGE_F = TPS * TILE_F;
    constexpr int USTAGE_F = TPS * NSP * kTileD;
    extern __shared__ __align__(128) unsigned char smem[];
    float *Ds = reinterpret_cast<float *>(smem);          // [2][STAGE_F]
    float *Us = Ds + 2 * STAGE_F;                         // [2][USTAGE_F]
    FCold *cold = reinterpret_cast<FCold *>(Us + 2 * USTAGE_F);  // [RPT][256]
    uint64_t *bar = reinterpret_cast<uint64_t *>(cold + RPT * 256);

    const int split = blockIdx.y;
    const int n_r = (int)*P.d_nr;
    const int n_tiles = (int)((P.d_misc[0] + kTileD - 1) / kTileD);
    const int t0 = (int)(((int64_t)split * n_tiles) / P.nsplit);
    const int t1 = (int)(((int64_t)(split + 1) * n_tiles) / P.nsplit);
    const int ntl = max(0, t1 - t0);
    const int nstages = (ntl + TPS - 1) / TPS;
    auto issue = [&](int s) {
        const int buf = s & 1;
        const int ta = t0 + s * TPS, tb = min(t1, ta + TPS);
        const uint32_t b1 = (uint32_t)(tb - ta) * TILE_F * 4;
        const uint32_t b2 = (uint32_t)(tb - ta) * P.nsp * kTileD * 4;
        fmbar_expect_tx(&bar[buf], b1 + b2);
        fbulk_g2s(Ds + buf * STAGE_F, P.Dc + (size_t)ta * TILE_F, b1, &bar[buf]);
        fbulk_g2s(Us + buf * USTAGE_F, P.U + (size_t)ta * P.nsp * kTileD, b2, &bar[buf]);
    };
    if (threadIdx.x == 0) {
        fmbar_init(&bar[0], 1);
        fmbar_init(&bar[1], 1);
        fmbar_fence_init();
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        if (nstages > 0) issue(0);
        if (nstages > 1) issue(1);
    }

    // ---- this thread's RPT ranges: coefficients + error factor + thresholds in registers
    float rc[RPT][NC], cr[RPT], thr[RPT][NSP];
    const int rbase = (blockIdx.x * 256 + threadIdx.x) * RPT;
#pragma unroll
    for (int q = 0; q < RPT; ++q) {
        const int r = rbase + q;
        const bool valid = r < n_r;
        const int rr = valid ? r : 0;
#pragma unroll
        for (int c = 0; c < NC; ++c) rc[q][c] = valid ? P.Rc[(size_t)c * P.r_stride + rr] : 0.f;
        const RangeMeta m = P.meta[rr];
        cr[q] = m.cr;
        FCold &cd = cold[q * 256 + threadIdx.x];
        cd.A = m.A;
        cd.margin = m.margin;
        if (P.has_zero) {  // s = 0 gives e = A for every (domain, isometry): first is (0, 0, j0)
            cd.best_e = m.A;
            cd.best_d = 0;
            cd.best_kj = P.j_zero;
        } else {
            cd.best_e = INFINITY;
            cd.best_d = INT_MAX;
            cd.best_kj = INT_MAX;
        }
        const float t0v = P.has_zero ? fminf(__double2float_ru(m.margin), FLT_MAX) : FLT_MAX;
#pragma unroll
        for (int jj = 0; jj < NSP; ++jj) thr[q][jj] = (valid && jj < P.nsp) ? t0v : -FLT_MAX;
    }
    float nhs8[NSP];  // -(s_j / 2) / 8
#pragma unroll
    for (int jj = 0; jj < NSP; ++jj)
        nhs8[jj] = -__double2float_rn(0.0625 * (jj < P.nsp ? P.spos[jj] : 0.0));
    unsigned n_exact = 0;

    for (int s = 0; s < nstages; ++s) {
        const int buf = s & 1;
        fmbar_wait(&bar[buf], (uint32_t)((s >> 1) & 1));
        const float *D = Ds + buf * STAGE_F;
        const float *Ub = Us + buf * USTAGE_F;
        const int ta = t0 + s * TPS;
        const int nt = min(t1 - ta, TPS);
        for (int tt = 0; tt < nt; ++tt) {
            const float *Dt = D + tt * TILE_F;
            const float *Ut = Ub + tt * P.nsp * kTileD;
            const int dbase = (ta + tt) * kTileD;
#pragma unroll 1
            for (int dl = 0; dl < kTileD; ++dl) {
                const float *rec = Dt + dl * NCS;
                float acc[RPT][8];
#pragma unroll
                for (int q = 0; q < RPT; ++q)
#pragma unroll
                    for (int k = 0; k < 8; ++k) acc[q][k] = 0.f;
#pragma unroll
                for (int o = 0; o < Cf::nO; ++o) {
                    const float4 da = *reinterpret_cast<const float4 *>(rec + o * 8);
                    const float4 db = *reinterpret_cast<const float4 *>(rec + o * 8 + 4);
#pragma unroll
                    for (int q = 0; q < RPT; ++q) {
                        const float *rh = rc[q] + o * 8;
                        acc[q][0] = fmaf(rh[0], da.x, acc[q][0]);
                        acc[q][1] = fmaf(rh[1], da.y, acc[q][1]);
                        acc[q][2] = fmaf(rh[2], da.z, acc[q][2]);
                        acc[q][3] = fmaf(rh[3], da.w, acc[q][3]);
                        // C2[i][j] += dh(i,0) rh(j,0) + dh(i,1) rh(j,1); dh(0,*) = db.x,y; dh(1,*) = db.z,w
                        acc[q][4] = fmaf(db.x, rh[4], fmaf(db.y, rh[5], acc[q][4]));  // C00
                        acc[q][5] = fmaf(db.x, rh[6], fmaf(db.y, rh[7], acc[q][5]));  // C01
                        acc[q][6] = fmaf(db.z, rh[4], fmaf(db.w, rh[5], acc[q][6]));  // C10
                        acc[q][7] = fmaf(db.z, rh[6], fmaf(db.w, rh[7], acc[q][7]));  // C11
                    }
                }
                const float dn = rec[NC];
                float uj[NSP];
#pragma unroll
                for (int jj = 0; jj < NSP; ++jj) uj[jj] = jj < P.nsp ? Ut[jj * kTileD + dl] : 0.f;
                unsigned pass = 0;
#pragma unroll
                for (int q = 0; q < RPT; ++q) {
                    const float *c = acc[q];
                    const float p01 = c[0] + c[1], m01 = c[0] - c[1];
                    const float p23 = c[2] + c[3], m23 = c[2] - c[3];
                    const float t0v = c[4] + c[7], t4v = c[4] - c[7];
                    const float t5v = c[5] + c[6], t1v = c[6] - c[5];
                    const float v0 = fmaf(2.f, fabsf(t0v), p01 + p23);
                    const float v1 = fmaf(2.f, fabsf(t1v), p01 - p23);
                    const float v4 = fmaf(2.f, fabsf(t4v), m01 + m23);
                    const float v5 = fmaf(2.f, fabsf(t5v), m01 - m23);
                    const float m8 = fmaxf(fmaxf(v0, v1), fmaxf(v4, v5));  // ~ 8 max_k Bq_k
                    const float m8p = fmaf(cr[q], dn, m8);                 // >= 8 max_k Bq_k
                    bool pq = false;
#pragma unroll
                    for (int jj = 0; jj < NSP; ++jj) pq = pq || (fmaf(nhs8[jj], m8p, uj[jj]) <= thr[q][jj]);
                    pass |= (unsigned)pq << q;
                }
                if (pass) {
#pragma unroll
                    for (int q = 0; q < RPT; ++q)
                        if (pass >> q & 1) {
                            fexact<B, NSP>(P, rc[q], rec, dbase + dl, cold[q * 256 + threadIdx.x], thr[q]);
                            ++n_exact;
                        }
                }
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
            const FCold &cd = cold[q * 256 + threadIdx.x];
            Partial pb;
            pb.e = cd.best_e;
            pb.d = cd.best_d;
            pb.kj = cd.best_kj;
            P.part[(size_t)r * P.nsplit + split] = pb;
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) n_exact += __shfl_xor_sync(0xffffffffu, n_exact, o);
    if ((threadIdx.x & 31) == 0 && n_exact && P.exact_count)
        atomicAdd(P.exact_count, (unsigned long long)n_exact);
}

// ------------------------------------------------------------------------------ launchers
template <int B, int NSP, int RPT>
static cudaError_t launch_fsearch_t(const FSearchParams &p, int32_t n_r_max, cudaStream_t st) {
    using Cf = FCfg<B>;
    constexpr int TILE_F = kTileD * Cf::NCS;
    constexpr int TPS = (TILE_F * 4 >= 24 * 1024) ? 1 : (24 * 1024) / (TILE_F * 4);
    constexpr size_t SMEM = (size_t)(2 * TPS * TILE_F + 2 * TPS * NSP * kTileD) * 4 +
                            sizeof(FCold) * RPT * 256 + 64;
    static bool attr = false;
    if (!attr) {
        cudaError_t e = cudaFuncSetAttribute(fsearch_kernel<B, NSP, RPT>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM);
        if (e != cudaSuccess) return e;
        attr = true;
    }
    dim3 grid((unsigned)((n_r_max + 256 * RPT - 1) / (256 * RPT)), (unsigned)p.nsplit);
    fsearch_kernel<B, NSP, RPT><<<grid, 256, SMEM, st>>>(p);
    return cudaGetLastError();
}

int fourier_rpt(int32_t B, int32_t nsp) {
    if (nsp > 2) return 1;
    return B == 2 ? 4 : (B == 4 ? 2 : 1);
}

template <int B>
constexpr int rpt_of() { return B == 2 ? 4 : (B == 4 ? 2 : 1); }

template <int B>
static cudaError_t launch_fsearch_b(const FSearchParams &p, int32_t n_r_max, cudaStream_t st) {
    if (p.nsp <= 1) return launch_fsearch_t<B, 1, rpt_of<B>()>(p, n_r_max, st);
    if (p.nsp <= 2) return launch_fsearch_t<B, 2, rpt_of<B>()>(p, n_r_max, st);
    return launch_fsearch_t<B, 16, 1>(p, n_r_max, st);
}

// Range prep + U + search for B in {2, 4, 8}.  Rc [NC][r_stride], meta [n_r], U [n_tiles][nsp][128].
cudaError_t launch_fourier_level(int32_t B, const SearchParams &sp, const float *Dc, float *Rc,
                                 int32_t r_stride, void *meta, float *U, cudaStream_t st) {
    if (sp.n_r == 0) return cudaSuccess;
    const int64_t n_slots = sp.slot_stride;
    SList sl;
    memcpy(sl.s, sp.spos, sizeof sl.s);
    RangeMeta *m = reinterpret_cast<RangeMeta *>(meta);
    const unsigned rb = (unsigned)((sp.n_r + 127) / 128);
    switch (B) {
    case 2: fourier_range_kernel<2><<<rb, 128, 0, st>>>(sp.img, sp.N, sp.ranges, sp.d_nr, r_stride, sp.smax, sp.d_misc, Rc, m); break;
    case 4: fourier_range_kernel<4><<<rb, 128, 0, st>>>(sp.img, sp.N, sp.ranges, sp.d_nr, r_stride, sp.smax, sp.d_misc, Rc, m); break;
    case 8: fourier_range_kernel<8><<<rb, 128, 0, st>>>(sp.img, sp.N, sp.ranges, sp.d_nr, r_stride, sp.smax, sp.d_misc, Rc, m); break;
    default: return cudaErrorInvalidValue;
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    if (sp.nsp > 0 && n_slots > 0) {
        fourier_u_kernel<<<(unsigned)((n_slots + 255) / 256), 256, 0, st>>>(sp.C, &sp.d_misc[0], n_slots, sl,
                                                                            sp.nsp, U);
        e = cudaGetLastError();
        if (e != cudaSuccess) return e;
    }
    if (sp.nsp == 0) return cudaSuccess;
    FSearchParams p;
    memset(&p, 0, sizeof p);
    p.Dc = Dc; p.U = U; p.C = sp.C; p.Rc = Rc; p.meta = m;
    p.d_nr = sp.d_nr; p.d_misc = sp.d_misc; p.r_stride = r_stride; p.nsplit = sp.nsplit;
    p.nsp = sp.nsp;
    memcpy(p.spos, sp.spos, sizeof p.spos);
    memcpy(p.jpos, sp.jpos, sizeof p.jpos);
    p.has_zero = sp.has_zero; p.j_zero = sp.j_zero;
    p.part = sp.part; p.exact_count = sp.exact_count;
    // grid is sized by the host-side upper bound of n_r
    switch (B) {
    case 2: return launch_fsearch_b<2>(p, sp.n_r, st);
    case 4: return launch_fsearch_b<4>(p, sp.n_r, st);
    case 8: return launch_fsearch_b<8>(p, sp.n_r, st);
    default: return cudaErrorInvalidValue;
    }
}

size_t fourier_meta_bytes() { return sizeof(RangeMeta); }

int fourier_nsplit_hint(int32_t B, int32_t nsp, int64_t n_r, int64_t n_tiles, int num_sms) {
    const int rpt = fourier_rpt(B, nsp);
    const int64_t gx = (n_r + 256 * rpt - 1) / (256 * rpt);
    if (gx <= 0 || n_tiles <= 0) return 1;
    const int64_t target = (int64_t)num_sms * 4;
    int64_t ns = (target + gx - 1) / gx;
    const int64_t max_ns = (n_tiles + 1) / 2;  // at least ~2 tiles per split
    if (ns > max_ns) ns = max_ns;
    if (ns < 1) ns = 1;
    if (ns > 65535) ns = 65535;
    return (int)ns;
}

}  // namespace fic
