/*
 * fic_oracle.c -- plain, slow, obviously-correct CPU ORACLE for the fractal-encoder search of
 * H. Miar Naimi & M. Salarian, "A Fast Fractal Image Compression Algorithm Using Predefined
 * Values for Contrast Scaling" (arXiv 1501.04140), /root/reference/PAPER.md ("P:<line>").
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library.  It shares no code with the CUDA path
 * (paper_1501_04140_b200/): nothing here is included by, linked into, or generated for it.
 *
 * Everything follows the plain definitions, in the paper's order, in int64 / IEEE binary64
 * (compiled with -ffp-contract=off, no fast-math).  The readings of points where the paper is
 * silent are listed in DESIGN.md §"Readings" (R1..R22) and cited below as [Rn].
 *
 *   range blocks      P:28  "partitioned into none overlapping range blocks of size B x B"
 *   domain blocks     P:28  "all square blocks of size 2B x 2B with integer step L"
 *   decimation        P:30  "a decimated domain block, D" -> 2x2 sums D' = 4d        [R1]
 *   8 isometries      P:28  rotations 90/180/270 + mirrors, applied to the DOMAIN    [R2]
 *   distance          P:30  Eq. (1)  E(R,D) = sum_i (s d_i + o - r_i)^2
 *   offset            P:36  Eq. (3)  o = Rbar - s Dbar
 *   s search          P:38  "search S across a pre-sampled set of [0,1]"; P:108 predefined sets
 *   entropy           P:52-56 Eq. (4)-(5), natural log, 256 gray levels, raw 2Bx2B block [R3]
 *   pool filter       P:14  "only domain blocks with entropies greater than a threshold" [R4]
 *   quadtree          P:40  accept "mapped with an acceptable error", else split in 4   [R14,R15]
 *
 * Eq. (1) with o from Eq. (3) is evaluated through exact integer moments (same real value):
 *   A = n SRR - SR^2,  Bq_k = n SRD_k - SR SD,  C = n SDD - SD^2      (int64, exact)
 *   e = (A - (0.5 s) Bq_k) + (s s)(0.0625 C),  E = e / n              (binary64, this order) [R6/C7]
 * The exact-rational literal Eq. (1) in oracle/exact.py pins this (tests/test_oracle_*.py).
 */
#include <math.h>
#include <quadmath.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define FICO_OK 0
#define FICO_ERR_ARG 1
#define FICO_ERR_SHAPE 2
#define FICO_ERR_EMPTY_POOL 3
#define FICO_ERR_CAPACITY 4
#define FICO_ERR_NOMEM 7

typedef struct {
    int32_t rx, ry, B, dom, dx, dy;
    uint8_t iso, s_idx, o_code, accepted;
    double err;
} fico_record; /* 40 bytes, same field meaning as include/fic.h fic_record */

/* ---------------------------------------------------------------- entropy (Eq. 4-5) -------- */

/* lut[c] = round-half-even(c * log2(c) * 2^32), c = 0..mmax (lut[0] = lut[1] = 0).
 * Fixed-point form of the terms of Eq. (5) so that the pool decision is order independent [R6].
 * Computed in binary128 (113-bit) arithmetic: correctly rounded (pinned against mpmath). */
void fico_lut(int64_t *lut, int32_t mmax) {
    for (int32_t c = 0; c <= mmax; ++c) {
        if (c < 2) { lut[c] = 0; continue; }
        __float128 v = (__float128)c * log2q((__float128)c) * (__float128)4294967296.0;
        __float128 r = rintq(v); /* default rounding mode: nearest, ties to even */
        lut[c] = (int64_t)r;
    }
}

/* T = floor(((tau * log2(e)) * m) * 2^32) in binary64, left to right [R5,R6]. */
int64_t fico_threshold(double tau, int32_t m) {
    double t = tau * 1.4426950408889634;
    t = t * (double)m;
    t = t * 4294967296.0;
    return (int64_t)floor(t);
}

/* number of candidates per axis: positions x = a L with x + 2B <= N  (P:20 at L=1) */
int64_t fico_axis_candidates(int32_t N, int32_t B, int32_t L) {
    if (2 * B > N || L < 1) return 0;
    return (int64_t)((N - 2 * B) / L + 1);
}

/* Entropy keys of every candidate domain block (raw 2B x 2B block, m = 4B^2 pixels).
 *   key  = lut[m] - sum_v lut[h_v]   (= m * H_bits * 2^32, exact integer)
 *   keep = tau < 0 || key > T(tau)   ("entropies greater than a threshold")
 *   H    = -sum_v (h_v/m) ln(h_v/m)  (Eq. 5 in binary64, reported for checks only)
 * Candidate order: c = b * A + a, (x, y) = (a L, b L), row-major [R18]. */
int fico_entropy_keys(const uint8_t *img, int32_t N, int32_t B, int32_t L, double tau,
                      int64_t *keys, uint8_t *keep, double *H) {
    int64_t A = fico_axis_candidates(N, B, L);
    if (A <= 0) return FICO_ERR_SHAPE;
    int32_t side = 2 * B, m = side * side;
    int64_t *lut = (int64_t *)malloc(sizeof(int64_t) * (size_t)(m + 1));
    if (!lut) return FICO_ERR_NOMEM;
    fico_lut(lut, m);
    int64_t T = fico_threshold(tau, m);
#pragma omp parallel for schedule(static)
    for (int64_t c = 0; c < A * A; ++c) {
        int32_t h[256];
        memset(h, 0, sizeof(h));
        int64_t x = (c % A) * L, y = (c / A) * L;
        for (int32_t i = 0; i < side; ++i)
            for (int32_t j = 0; j < side; ++j) h[img[(y + i) * (int64_t)N + (x + j)]] += 1;
        int64_t s = 0;
        double ent = 0.0;
        for (int v = 0; v < 256; ++v) {
            s += lut[h[v]];
            if (h[v] > 0) {
                double p = (double)h[v] / (double)m; /* Eq. (4) */
                ent -= p * log(p);                   /* Eq. (5) */
            }
        }
        int64_t key = lut[m] - s;
        if (keys) keys[c] = key;
        if (keep) keep[c] = (uint8_t)(tau < 0.0 || key > T);
        if (H) H[c] = ent;
    }
    free(lut);
    return FICO_OK;
}

/* ---------------------------------------------------------------- isometries -------- */

/* out = T_k(X) with out(i,j) = X(f_k(i,j)), b = B-1 [R2]:
 *   k=0 (i,j)  1 (b-j,i)  2 (b-i,b-j)  3 (j,b-i)     rotations by 0/90/180/270 deg clockwise
 *   k=4 (i,b-j) 5 (j,i)   6 (b-i,j)    7 (b-j,b-i)   the same followed by a horizontal mirror */
void fico_isometry_src(int32_t B, int32_t k, int32_t i, int32_t j, int32_t *si, int32_t *sj) {
    int32_t b = B - 1;
    switch (k) {
    case 0: *si = i; *sj = j; break;
    case 1: *si = b - j; *sj = i; break;
    case 2: *si = b - i; *sj = b - j; break;
    case 3: *si = j; *sj = b - i; break;
    case 4: *si = i; *sj = b - j; break;
    case 5: *si = j; *sj = i; break;
    case 6: *si = b - i; *sj = j; break;
    default: *si = b - j; *sj = b - i; break;
    }
}

void fico_apply_isometry(const int32_t *X, int32_t B, int32_t k, int32_t *out) {
    for (int32_t i = 0; i < B; ++i)
        for (int32_t j = 0; j < B; ++j) {
            int32_t si, sj;
            fico_isometry_src(B, k, i, j, &si, &sj);
            out[i * B + j] = X[si * B + sj];
        }
}

/* ---------------------------------------------------------------- decimation -------- */

/* D'(i,j) = sum of the 2x2 cell of the 2B x 2B block at (x,y); d_i = D'/4 exactly [R1]. */
void fico_decimate(const uint8_t *img, int32_t N, int32_t x, int32_t y, int32_t B, int32_t *Dp) {
    for (int32_t i = 0; i < B; ++i)
        for (int32_t j = 0; j < B; ++j) {
            int64_t r0 = (int64_t)(y + 2 * i) * N + (x + 2 * j), r1 = r0 + N;
            Dp[i * B + j] = (int32_t)img[r0] + img[r0 + 1] + img[r1] + img[r1 + 1];
        }
}

/* ---------------------------------------------------------------- o quantiser [R11] -------- */

/* 8-bit midrise quantiser of o in [-255,255], step w = 510/256; o = 0 -> code 128. */
int32_t fico_o_code(double o) {
    const double w = 1.9921875;
    int32_t j;
    if (o >= 0.0) {
        double mu = o / w;
        j = (mu == 0.0) ? 0 : (int32_t)ceil(mu) - 1;
        if (j > 127) j = 127;
        return 128 + j;
    }
    double mu = (-o) / w;
    j = (int32_t)ceil(mu) - 1;
    if (j > 127) j = 127;
    return 127 - j;
}

/* ---------------------------------------------------------------- one level's pool --------- */

typedef struct {
    int32_t B, n, A;      /* range size, pixels, candidates per axis */
    int64_t n_k;          /* kept domains */
    const int32_t *kept;  /* kept candidate indices (ascending) */
    int32_t *Dp;          /* [n_k][n] decimated domains D' */
    int64_t *SD, *SDD, *C;
    int32_t L;
} fico_pool;

static int pool_build(const uint8_t *img, int32_t N, int32_t B, int32_t L, const int32_t *kept,
                      int64_t n_k, fico_pool *P) {
    P->B = B; P->n = B * B; P->L = L; P->n_k = n_k; P->kept = kept;
    P->A = (int32_t)fico_axis_candidates(N, B, L);
    P->Dp = (int32_t *)malloc(sizeof(int32_t) * (size_t)n_k * P->n);
    P->SD = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n_k ? n_k : 1));
    P->SDD = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n_k ? n_k : 1));
    P->C = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n_k ? n_k : 1));
    if (!P->Dp || !P->SD || !P->SDD || !P->C) return FICO_ERR_NOMEM;
#pragma omp parallel for schedule(static)
    for (int64_t d = 0; d < n_k; ++d) {
        int32_t c = kept[d];
        int32_t x = (c % P->A) * L, y = (c / P->A) * L;
        int32_t *D = P->Dp + d * P->n;
        fico_decimate(img, N, x, y, B, D);
        int64_t sd = 0, sdd = 0;
        for (int32_t p = 0; p < P->n; ++p) { sd += D[p]; sdd += (int64_t)D[p] * D[p]; }
        P->SD[d] = sd; P->SDD[d] = sdd; P->C[d] = (int64_t)P->n * sdd - sd * sd;
    }
    return FICO_OK;
}

static void pool_free(fico_pool *P) {
    free(P->Dp); free(P->SD); free(P->SDD); free(P->C);
}

/* Best affine map of one range: loops kept domain c ascending, isometry k = 0..7,
 * s index j ascending; replace iff e < best (strict) [R17]; no early exit. */
static void match_one(const uint8_t *img, int32_t N, const fico_pool *P, int32_t rx, int32_t ry,
                      const double *s, int32_t n_s, double rms_tol, int32_t is_min,
                      fico_record *out) {
    const int32_t B = P->B, n = P->n;
    int32_t R[32 * 32];
    int32_t perm[8][32 * 32]; /* perm[k][p] = flat index of f_k(i,j), p = i*B+j */
    int64_t SR = 0, SRR = 0;
    for (int32_t i = 0; i < B; ++i)
        for (int32_t j = 0; j < B; ++j) {
            int32_t v = img[(int64_t)(ry + i) * N + (rx + j)];
            R[i * B + j] = v; SR += v; SRR += (int64_t)v * v;
        }
    for (int32_t k = 0; k < 8; ++k)
        for (int32_t i = 0; i < B; ++i)
            for (int32_t j = 0; j < B; ++j) {
                int32_t si, sj;
                fico_isometry_src(B, k, i, j, &si, &sj);
                perm[k][i * B + j] = si * B + sj;
            }
    const int64_t A = (int64_t)n * SRR - SR * SR;
    double best_e = INFINITY;
    int64_t best_c = -1;
    int32_t best_k = 0, best_j = 0;
    for (int64_t c = 0; c < P->n_k; ++c) {
        const int32_t *D = P->Dp + c * n;
        for (int32_t k = 0; k < 8; ++k) {
            int64_t SRD = 0; /* sum_i r_i * T_k(D')_i  (the transformed domain) */
            for (int32_t p = 0; p < n; ++p) SRD += (int64_t)R[p] * D[perm[k][p]];
            const int64_t Bq = (int64_t)n * SRD - SR * P->SD[c];
            for (int32_t j = 0; j < n_s; ++j) {
                double hs = 0.5 * s[j];
                double t2 = (s[j] * s[j]) * (0.0625 * (double)P->C[c]);
                double e = ((double)A - hs * (double)Bq) + t2;
                if (e < best_e) { best_e = e; best_c = c; best_k = k; best_j = j; }
            }
        }
    }
    const double E = best_e / (double)n;
    const double sj = s[best_j];
    const double Rbar = (double)SR / (double)n;
    const double Dbar = (double)P->SD[best_c] / (double)(4 * n);
    const double o = Rbar - sj * Dbar; /* Eq. (3) */
    const int32_t cand = P->kept[best_c];
    memset(out, 0, sizeof(*out)); /* deterministic padding bytes */
    out->rx = rx; out->ry = ry; out->B = B;
    out->dom = (int32_t)best_c;
    out->dx = (cand % P->A) * P->L; out->dy = (cand / P->A) * P->L;
    out->iso = (uint8_t)best_k; out->s_idx = (uint8_t)best_j;
    out->o_code = (uint8_t)fico_o_code(o);
    out->accepted = (uint8_t)(is_min || E <= (rms_tol * rms_tol) * (double)n);
    out->err = E;
}

static int check_level_args(int32_t N, int32_t B, int32_t L, const double *s, int32_t n_s) {
    if (N < 1 || B < 2 || B > 32 || (B & (B - 1)) || L < 1) return FICO_ERR_ARG;
    if (2 * B > N) return FICO_ERR_SHAPE;
    if (n_s < 1 || n_s > 255) return FICO_ERR_ARG;
    for (int32_t j = 0; j < n_s; ++j)
        if (!(s[j] >= 0.0 && s[j] <= 1.0)) return FICO_ERR_ARG;
    return FICO_OK;
}

/* One quadtree level: every range in `ranges` ([n_r][2] = (rx, ry)) against the kept pool. */
int fico_encode_level(const uint8_t *img, int32_t N, int32_t B, int32_t L, const int32_t *kept,
                      int64_t n_k, const int32_t *ranges, int64_t n_r, const double *s,
                      int32_t n_s, double rms_tol, int32_t is_min, fico_record *out) {
    int st = check_level_args(N, B, L, s, n_s);
    if (st) return st;
    if (n_k < 1) return FICO_ERR_EMPTY_POOL;
    fico_pool P;
    st = pool_build(img, N, B, L, kept, n_k, &P);
    if (st) { pool_free(&P); return st; }
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t r = 0; r < n_r; ++r)
        match_one(img, N, &P, ranges[2 * r], ranges[2 * r + 1], s, n_s, rms_tol, is_min, &out[r]);
    pool_free(&P);
    return FICO_OK;
}

/* Kept list of one level: ascending candidate indices with keep = 1. Returns count. */
int64_t fico_kept_list(const uint8_t *img, int32_t N, int32_t B, int32_t L, double tau,
                       int32_t *kept_out /* capacity n_c */) {
    int64_t A = fico_axis_candidates(N, B, L);
    if (A <= 0) return -FICO_ERR_SHAPE;
    uint8_t *keep = (uint8_t *)malloc((size_t)(A * A));
    if (!keep) return -FICO_ERR_NOMEM;
    fico_entropy_keys(img, N, B, L, tau, NULL, keep, NULL);
    int64_t n = 0;
    for (int64_t c = 0; c < A * A; ++c)
        if (keep[c]) kept_out[n++] = (int32_t)c;
    free(keep);
    return n;
}

/* Top-K pool selection (the paper's "pool size", Tables 1-2; reading R27): the K
 * candidates with the largest entropy keys, ties to the lower row-major index; the kept list is
 * still returned in ascending (row-major) candidate order [R18].  K >= n_c keeps every candidate.
 * The ranking is a plain sort (qsort on (key desc, index asc)).  Returns the count. */
typedef struct { int64_t key; int64_t idx; } fico_kc;
static int fico_kc_cmp(const void *a, const void *b) {
    const fico_kc *x = (const fico_kc *)a, *y = (const fico_kc *)b;
    if (x->key != y->key) return x->key > y->key ? -1 : 1;
    return x->idx < y->idx ? -1 : (x->idx > y->idx);
}
static int fico_i32_cmp(const void *a, const void *b) {
    const int32_t x = *(const int32_t *)a, y = *(const int32_t *)b;
    return (x > y) - (x < y);
}
int64_t fico_kept_list_topk(const uint8_t *img, int32_t N, int32_t B, int32_t L, int64_t K,
                            int32_t *kept_out /* capacity n_c */) {
    int64_t A = fico_axis_candidates(N, B, L);
    if (A <= 0) return -FICO_ERR_SHAPE;
    if (K < 1) return -FICO_ERR_ARG;
    const int64_t nc = A * A;
    int64_t *keys = (int64_t *)malloc(sizeof(int64_t) * (size_t)nc);
    fico_kc *kc = (fico_kc *)malloc(sizeof(fico_kc) * (size_t)nc);
    if (!keys || !kc) { free(keys); free(kc); return -FICO_ERR_NOMEM; }
    fico_entropy_keys(img, N, B, L, -1.0, keys, NULL, NULL);
    for (int64_t c = 0; c < nc; ++c) { kc[c].key = keys[c]; kc[c].idx = c; }
    qsort(kc, (size_t)nc, sizeof(fico_kc), fico_kc_cmp);
    const int64_t n = K < nc ? K : nc;
    for (int64_t i = 0; i < n; ++i) kept_out[i] = (int32_t)kc[i].idx;
    qsort(kept_out, (size_t)n, sizeof(int32_t), fico_i32_cmp);
    free(keys);
    free(kc);
    return n;
}

/* Full quadtree encode: level B_max ranges are all (uB, vB) row-major; the 4 children
 * (TL, TR, BL, BR) of every rejected range form the next level, re-sorted row-major [R16].
 * Records of accepted leaves, level by level (B descending), each level row-major (ry, rx).
 * Shard (shard, n_shards): keep only top-level blocks t with t % n_shards == shard (t = row-major
 * index) and their descendants; n_shards = 1 is the whole image. */
int fico_encode_sel(const uint8_t *img, int32_t N, int32_t B_max, int32_t B_min, int32_t L,
                    const double *tau, const int64_t *topk, const double *s_flat, const int32_t *n_s,
                    const double *rms_tol, int32_t shard, int32_t n_shards, fico_record *out,
                    int64_t capacity, int64_t *n_out) {
    *n_out = 0;
    if (B_min < 2 || B_max > 32 || B_min > B_max || (B_max & (B_max - 1)) || (B_min & (B_min - 1)))
        return FICO_ERR_ARG;
    if (N % B_max) return FICO_ERR_SHAPE;
    if (n_shards < 1 || shard < 0 || shard >= n_shards) return FICO_ERR_ARG;
    int32_t G = N / B_max;
    int64_t n_r = 0;
    int32_t *ranges = (int32_t *)malloc(sizeof(int32_t) * 2 * (size_t)G * G);
    for (int32_t v = 0; v < G; ++v)
        for (int32_t u = 0; u < G; ++u)
            if (((int64_t)v * G + u) % n_shards == shard) {
                ranges[2 * n_r] = u * B_max; ranges[2 * n_r + 1] = v * B_max; ++n_r;
            }
    int64_t total = 0, s_off = 0;
    int st = FICO_OK;
    int level = 0;
    for (int32_t B = B_max; B >= B_min; B /= 2, ++level) {
        const double *s = s_flat + s_off;
        s_off += n_s[level];
        st = check_level_args(N, B, L, s, n_s[level]);
        if (st) break;
        int64_t A = fico_axis_candidates(N, B, L);
        int32_t *kept = (int32_t *)malloc(sizeof(int32_t) * (size_t)(A * A));
        int64_t n_k = topk ? fico_kept_list_topk(img, N, B, L, topk[level], kept)
                           : fico_kept_list(img, N, B, L, tau[level], kept);
        if (n_k < 1) { free(kept); st = FICO_ERR_EMPTY_POOL; break; }
        fico_record *rec = (fico_record *)malloc(sizeof(fico_record) * (size_t)(n_r ? n_r : 1));
        st = fico_encode_level(img, N, B, L, kept, n_k, ranges, n_r, s, n_s[level], rms_tol[level],
                               B == B_min, rec);
        free(kept);
        if (st) { free(rec); break; }
        int32_t Gc = N / (B / 2 > 0 ? B / 2 : 1);
        uint8_t *child = NULL;
        if (B > B_min) child = (uint8_t *)calloc((size_t)Gc * Gc, 1);
        for (int64_t r = 0; r < n_r; ++r) {
            if (rec[r].accepted) {
                if (total < capacity) out[total] = rec[r];
                ++total;
            } else if (child) {
                int32_t cu = rec[r].rx / (B / 2), cv = rec[r].ry / (B / 2);
                child[(int64_t)cv * Gc + cu] = 1;
                child[(int64_t)cv * Gc + cu + 1] = 1;
                child[(int64_t)(cv + 1) * Gc + cu] = 1;
                child[(int64_t)(cv + 1) * Gc + cu + 1] = 1;
            }
        }
        free(rec);
        if (!child) break;
        int64_t nn = 0;
        for (int64_t q = 0; q < (int64_t)Gc * Gc; ++q) nn += child[q];
        free(ranges);
        ranges = (int32_t *)malloc(sizeof(int32_t) * 2 * (size_t)(nn ? nn : 1));
        n_r = 0;
        for (int32_t v = 0; v < Gc; ++v)
            for (int32_t u = 0; u < Gc; ++u)
                if (child[(int64_t)v * Gc + u]) {
                    ranges[2 * n_r] = u * (B / 2); ranges[2 * n_r + 1] = v * (B / 2); ++n_r;
                }
        free(child);
        if (n_r == 0) break;
    }
    free(ranges);
    *n_out = total;
    if (st) return st;
    return total > capacity ? FICO_ERR_CAPACITY : FICO_OK;
}

/* ---------------------------------------------------------------- decoding (PIFS) ---------- */
/* The paper encodes only; decoding is the standard PIFS iteration implied by P:28-30 ("an
 * affine transformation that maps the selected domain block").  Readings [R23-R26]:
 *   o dequantiser  o^ = (code - 127.5) * 510/256, the centre of the [R11] midrise cell (exact);
 *   one pass       out(R) = clamp(rint(s * d + o^), 0, 255) per pixel of each leaf R, with
 *                  d = T_k(D'/4) of the 2B x 2B block at (dx, dy) of the PREVIOUS iterate
 *                  (Jacobi, binary64, s * d rounded, then + o^ rounded, rint half-even);
 *   start          the constant image 128 (or a given image); a fixed iteration count;
 *   PSNR           10 log10(255^2 / MSE), MSE = (exact integer sum of squared differences)/n,
 *                  +inf for identical images ("PSNR"). */
double fico_o_value(int32_t code) { return ((double)code - 127.5) * 1.9921875; }

static int32_t fico_level_of(int32_t B_max, int32_t B) {
    int32_t l = 0;
    while ((B_max >> l) > B) ++l;
    return (B_max >> l) == B ? l : -1;
}

int fico_decode(const fico_record *rec, int64_t n_rec, int32_t N, const double *s_flat,
                const int32_t *n_s, int32_t B_max, int32_t n_levels, int32_t iterations,
                const uint8_t *init, uint8_t *out) {
    if (!rec || !s_flat || !n_s || !out || N < 1 || n_levels < 1 || iterations < 0) return FICO_ERR_ARG;
    int64_t off[16];
    off[0] = 0;
    for (int32_t l = 0; l < n_levels && l < 15; ++l) off[l + 1] = off[l] + n_s[l];
    for (int64_t q = 0; q < n_rec; ++q) {  /* validate: in bounds, known level and s index */
        const fico_record *r = &rec[q];
        const int32_t l = fico_level_of(B_max, r->B);
        if (l < 0 || l >= n_levels || r->s_idx >= n_s[l] || r->iso > 7) return FICO_ERR_ARG;
        if (r->rx < 0 || r->ry < 0 || r->rx + r->B > N || r->ry + r->B > N) return FICO_ERR_ARG;
        if (r->dx < 0 || r->dy < 0 || r->dx + 2 * r->B > N || r->dy + 2 * r->B > N) return FICO_ERR_ARG;
    }
    const int64_t np = (int64_t)N * N;
    uint8_t *prev = (uint8_t *)malloc((size_t)np);
    if (!prev) return FICO_ERR_NOMEM;
    if (init) memcpy(out, init, (size_t)np);
    else memset(out, 128, (size_t)np);
    for (int32_t it = 0; it < iterations; ++it) {
        memcpy(prev, out, (size_t)np);
        for (int64_t q = 0; q < n_rec; ++q) {
            const fico_record *r = &rec[q];
            const int32_t B = r->B, l = fico_level_of(B_max, B);
            const double s = s_flat[off[l] + r->s_idx], o = fico_o_value(r->o_code);
            int32_t Dp[32 * 32];
            fico_decimate(prev, N, r->dx, r->dy, B, Dp);
            for (int32_t i = 0; i < B; ++i)
                for (int32_t j = 0; j < B; ++j) {
                    int32_t si, sj;
                    fico_isometry_src(B, r->iso, i, j, &si, &sj);
                    const double d = (double)Dp[si * B + sj] / 4.0;
                    double v = rint(s * d + o);
                    if (v < 0.0) v = 0.0;
                    if (v > 255.0) v = 255.0;
                    out[(int64_t)(r->ry + i) * N + r->rx + j] = (uint8_t)v;
                }
        }
    }
    free(prev);
    return FICO_OK;
}

double fico_psnr(const uint8_t *a, const uint8_t *b, int64_t n) {
    int64_t sse = 0;
    for (int64_t i = 0; i < n; ++i) {
        const int64_t d = (int64_t)a[i] - (int64_t)b[i];
        sse += d * d;
    }
    if (sse == 0) return INFINITY;
    const double mse = (double)sse / (double)n;
    return 10.0 * log10(65025.0 / mse);
}

/* Pool selection per level: entropy threshold tau (keep iff H > tau) [R4]. */
int fico_encode(const uint8_t *img, int32_t N, int32_t B_max, int32_t B_min, int32_t L,
                const double *tau, const double *s_flat, const int32_t *n_s,
                const double *rms_tol, int32_t shard, int32_t n_shards, fico_record *out,
                int64_t capacity, int64_t *n_out) {
    return fico_encode_sel(img, N, B_max, B_min, L, tau, NULL, s_flat, n_s, rms_tol, shard, n_shards,
                           out, capacity, n_out);
}

int fico_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
