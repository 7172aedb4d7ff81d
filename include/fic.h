/*
 * fic.h -- C ABI of the B200 fractal-encoder search library (libfic.so, sm_100a).
 *
 * Method: H. Miar Naimi, M. Salarian, "A Fast Fractal Image Compression Algorithm Using
 * Predefined Values for Contrast Scaling", arXiv 1501.04140 (/root/reference/PAPER.md, cited as
 * P:<line>).  Readings of the points the paper leaves open are DESIGN.md §"Readings" [Rn].
 *
 * Conventions for every call
 *   - Pointers are DEVICE pointers unless the argument name starts with h_ (host memory).
 *   - Images are N x N uint8, row-major, pixel (x, y) = img[y * N + x].
 *   - Work is enqueued on the context's CUDA stream.  Calls that return host-visible counts
 *     (fic_build_domain_pool, fic_encode, fic_encode_host) synchronise that stream before
 *     returning; fic_encode_level is stream-asynchronous.
 *   - No call throws.  Every call returns a fic_status; on failure fic_last_error(ctx) holds a
 *     one-line message (valid until the next call on that ctx).
 *   - Ownership: the caller owns img, ranges and out buffers; the library owns the context's
 *     scratch memory and fic_pool storage (release with fic_pool_destroy / fic_ctx_destroy).
 *   - A context is not thread-safe; use one context per host thread / stream.
 */
#ifndef FIC_H_
#define FIC_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct fic_ctx fic_ctx;   /* per-device: stream, scratch arena, LUTs, level pools   */
typedef struct fic_pool fic_pool; /* one level's entropy-filtered domain pool (device data) */

typedef enum {
    FIC_OK = 0,
    FIC_ERR_ARG = 1,        /* bad scalar argument (B not a power of two, s outside [0,1], ...) */
    FIC_ERR_SHAPE = 2,      /* N not a multiple of B_max, 2B > N, ...                          */
    FIC_ERR_EMPTY_POOL = 3, /* no domain block survives the entropy filter                     */
    FIC_ERR_CAPACITY = 4,   /* output buffer too small; *h_n_out holds the required count       */
    FIC_ERR_CUDA = 5,       /* CUDA runtime error (message in fic_last_error)                  */
    FIC_ERR_NCCL = 6,       /* NCCL failure (fic_ctx_create_nccl / fic_encode_nccl)            */
    FIC_ERR_NOMEM = 7       /* device or host allocation failed                                */
} fic_status;

/* One affine map of the partitioned IFS = one coded range block.  40 bytes. */
typedef struct {
    int32_t rx, ry;   /* range origin (pixels)                                               */
    int32_t B;        /* range size (pixels per side)                                        */
    int32_t dom;      /* rank of the domain in the level's kept list (row-major order) [R18] */
    int32_t dx, dy;   /* domain origin (pixels), multiples of the step L               */
    uint8_t iso;      /* isometry k in 0..7 applied to the decimated domain [R2]             */
    uint8_t s_idx;    /* index of s in the level's s list (listed order)                     */
    uint8_t o_code;   /* 8-bit quantised offset o (Eq. 3) [R11]                        */
    uint8_t accepted; /* E <= t_B^2 * B^2 ("acceptable error") or B == B_min [R14,R15]  */
    double err;       /* E = sum_i (s d_i + o - r_i)^2, Eq. 1, unquantised o, binary64 */
} fic_record;

/* ------------------------------------------------------------------------------------ context */

/* Create a context on CUDA device `device` that enqueues on `cuda_stream` (a cudaStream_t;
 * NULL = legacy default stream).  *out receives the handle. */
fic_status fic_ctx_create(int32_t device, void *cuda_stream, fic_ctx **out);
fic_status fic_ctx_set_stream(fic_ctx *ctx, void *cuda_stream);
fic_status fic_ctx_destroy(fic_ctx *ctx);
const char *fic_last_error(const fic_ctx *ctx);

/* Per-level counters and device times of the last fic_encode / fic_encode_level on ctx.
 * Times are CUDA-event durations on the ctx stream (ms); enable with fic_ctx_set_timing:
 * 1 = ms_search only (two events per level around the search launches), 2 = also ms_pool and
 * ms_finalize (five events per level; the extra events cost device time), 0 = off. */
typedef struct {
    int32_t B;
    int64_t n_candidates, n_kept, n_ranges, n_accepted;
    int64_t pairs;          /* n_ranges * n_kept * 8 range-domain-isometry pairs scored      */
    int64_t exact_evals;    /* (range, domain) pairs that took the exact binary64 path       */
    float ms_pool, ms_search, ms_finalize;
    int64_t kernel_launches; /* libfic kernels launched for this level (pool + search + quadtree) */
    int64_t pairs_scanned;  /* (range, domain) pairs the search evaluated (fp32 filter); the rest of
                               n_ranges * n_kept were proven unable to win or tie (B = 2
                               Cauchy-Schwarz C windows) -- n_ranges * n_kept elsewhere */
} fic_level_stats;

fic_status fic_ctx_set_timing(fic_ctx *ctx, int32_t enable);
fic_status fic_get_stats(const fic_ctx *ctx, fic_level_stats *h_out, int32_t max_levels,
                         int32_t *h_n_levels);

/* --------------------------------------------------------------------------- domain pool */

/* Build one level's domain pool (Abstract P:14):
 *   candidates: 2B x 2B blocks at (x, y) = (aL, bL), x + 2B <= N, y + 2B <= N, row-major;
 *   entropy key of the raw block, keep iff tau < 0 or H > tau (nats, strict) [R3-R6];
 *   kept blocks decimated by 2x2 sums (D' = 4d) [R1] and their moments.
 * img: device [N*N]; B in {2,4,8,16,32} (B = 2 closed form on CUDA cores, 4..32 tcgen05);
 * L >= 1; 2B <= N.
 * Errors: ARG, SHAPE, EMPTY_POOL (the pool is still returned for inspection), CUDA, NOMEM.
 * Synchronises the ctx stream (the kept count is returned on the host). */
fic_status fic_build_domain_pool(fic_ctx *ctx, const uint8_t *img, int32_t N, int32_t B,
                                 int32_t L, double tau_nats, fic_pool **out);

/* Same with the paper's "pool size" selection (Tables 1-2; reading R27) instead of a
 * threshold: the K candidates with the largest entropy keys, ties to the lower row-major index;
 * the kept list stays in ascending candidate order.  K >= n_candidates keeps all.
 * Errors: ARG (K < 1 or as above), SHAPE, CUDA, NOMEM.  Synchronises the ctx stream. */
fic_status fic_build_domain_pool_topk(fic_ctx *ctx, const uint8_t *img, int32_t N, int32_t B,
                                      int32_t L, int64_t K, fic_pool **out);

/* Host view of a pool.  keep_mask [n_candidates] u8, kept [n_kept] int32 (ascending candidate
 * indices), keys [n_candidates] int64 entropy keys (m * H_bits * 2^32 fixed point) -- all
 * device pointers owned by the pool.  Any output pointer may be NULL. */
fic_status fic_pool_info(const fic_pool *pool, int64_t *h_n_candidates, int64_t *h_n_kept,
                         const uint8_t **keep_mask, const int32_t **kept, const int64_t **keys);
fic_status fic_pool_destroy(fic_pool *pool);

/* ------------------------------------------------------------------------------ search */

/* Match every range of `ranges` (device int32 [n_r][2] = (rx, ry), each a multiple of the
 * pool's B) against every kept domain x 8 isometries x every s of h_s (host double [n_s],
 * each in [0,1]; 1 <= n_s <= 32), scoring Eq. 1 with o from Eq. 3, and write the
 * lexicographically first minimiser (E; dom, iso, s_idx) of each range to out[r] (device
 * fic_record [n_r]).  accepted = is_min_level || E <= rms_tol^2 * B^2.
 * Stream-asynchronous.  Errors: ARG, SHAPE, EMPTY_POOL, CUDA. */
fic_status fic_encode_level(fic_ctx *ctx, const uint8_t *img, int32_t N, const fic_pool *pool,
                            const int32_t *ranges, int64_t n_r, const double *h_s, int32_t n_s,
                            double rms_tol, int32_t is_min_level, fic_record *out);

/* Full quadtree encode: levels B = B_max, B_max/2, ..., B_min; level i uses step L,
 * entropy threshold h_tau[i] (nats, < 0 keeps all), the s list h_s[off_i .. off_i+h_n_s[i])
 * (off_i = sum of earlier h_n_s), and RMS tolerance h_rms_tol[i].  Level B_max starts from
 * all (uB, vB) blocks; rejected ranges are split into their 4 children.
 * Sharding (multi-GPU, DESIGN.md §"Multi-GPU"): only top-level blocks t (row-major index) with
 * t % n_shards == shard, and their descendants, are encoded; n_shards = 1 is the whole image.
 * out: device fic_record [capacity]; accepted leaves sorted by B descending, then (ry, rx).
 * *h_n_out receives the number of records (also on FIC_ERR_CAPACITY).  Synchronous. */
fic_status fic_encode(fic_ctx *ctx, const uint8_t *img, int32_t N, int32_t B_max, int32_t B_min,
                      int32_t L, const double *h_tau, const double *h_s, const int32_t *h_n_s,
                      const double *h_rms_tol, int32_t shard, int32_t n_shards, fic_record *out,
                      int64_t capacity, int64_t *h_n_out);

/* fic_encode with per-level pool sizes h_K [levels] (top-K selection, as
 * fic_build_domain_pool_topk) in place of the entropy thresholds.  Errors: as fic_encode, and
 * ARG if some K < 1. */
fic_status fic_encode_topk(fic_ctx *ctx, const uint8_t *img, int32_t N, int32_t B_max, int32_t B_min,
                           int32_t L, const int64_t *h_K, const double *h_s, const int32_t *h_n_s,
                           const double *h_rms_tol, int32_t shard, int32_t n_shards, fic_record *out,
                           int64_t capacity, int64_t *h_n_out);

/* Same as fic_encode with HOST buffers: h_img [N*N] is copied to the device, h_out [capacity]
 * receives the records (device->host copy inside the call).  Synchronous. */
fic_status fic_encode_host(fic_ctx *ctx, const uint8_t *h_img, int32_t N, int32_t B_max,
                           int32_t B_min, int32_t L, const double *h_tau, const double *h_s,
                           const int32_t *h_n_s, const double *h_rms_tol, int32_t shard,
                           int32_t n_shards, fic_record *h_out, int64_t capacity,
                           int64_t *h_n_out);

/* ------------------------------------------------------------------------------ multi-GPU */

/* Host-only: a new NCCL unique id (128 bytes) for fic_ctx_create_nccl; create it on one rank and
 * hand the same bytes to every rank (any out-of-band channel, e.g. torch.distributed).
 * Errors: ARG, NCCL. */
fic_status fic_nccl_unique_id(uint8_t *h_id128);

/* fic_ctx_create plus an NCCL communicator of nranks ranks, this process being `rank` (one GPU
 * per rank; h_id128 from fic_nccl_unique_id).  fic_ctx_destroy releases the communicator.
 * Errors: ARG, CUDA, NCCL. */
fic_status fic_ctx_create_nccl(int32_t device, void *cuda_stream, const uint8_t *h_id128, int32_t nranks,
                               int32_t rank, fic_ctx **out);

/* Sharded fic_encode over the context's communicator: rank r encodes the top-level
 * blocks t % nranks == r (no exchange on the data path), then an ncclAllGather of the record
 * counts and one of the records, and the canonical merge; every rank receives the full code
 * (identical to a one-GPU fic_encode) in `out` (device, capacity records; *h_n_out = count, also
 * on CAPACITY).  Synchronous; collective: every rank of the communicator must call it with the
 * same arguments.  A rank whose shard fails sends its status through the count all-gather, so
 * every rank returns that status (the lowest failing rank's) rather than blocking.
 * Errors: as fic_encode; ARG without a communicator; NCCL. */
fic_status fic_encode_nccl(fic_ctx *ctx, const uint8_t *img, int32_t N, int32_t B_max, int32_t B_min,
                           int32_t L, const double *h_tau, const double *h_s, const int32_t *h_n_s,
                           const double *h_rms_tol, fic_record *out, int64_t capacity, int64_t *h_n_out);

/* fic_encode_nccl with per-level pool sizes h_K [levels] (top-K selection, as fic_encode_topk).
 * Errors: as fic_encode_nccl, and ARG if h_K is null or some K < 1. */
fic_status fic_encode_nccl_topk(fic_ctx *ctx, const uint8_t *img, int32_t N, int32_t B_max, int32_t B_min,
                                int32_t L, const int64_t *h_K, const double *h_s, const int32_t *h_n_s,
                                const double *h_rms_tol, fic_record *out, int64_t capacity, int64_t *h_n_out);

/* Merge per-shard record lists (each sorted by B desc, ry, rx) into one canonical list.
 * in: device fic_record [n_shards][stride]; h_counts: host int64 [n_shards]; out: device
 * fic_record [sum(h_counts)].  Stream-asynchronous. */
fic_status fic_merge_shards(fic_ctx *ctx, const fic_record *in, const int64_t *h_counts,
                            int32_t n_shards, int64_t stride, fic_record *out);

/* ------------------------------------------------------------------------ decoding, quality */

/* PIFS decoding of a code (the paper encodes only; "an affine transformation that maps
 * the selected domain block", readings R23-R25 in DESIGN.md): starting from `init` (device
 * [N*N], or NULL for the constant image 128), `iterations` Jacobi passes, each setting every
 * pixel of every record's B x B range to clamp(rint(s * d + o^), 0, 255), where d is the
 * record's isometry T_iso applied to the 2 x 2-averaged (D'/4, exact) 2B x 2B block at (dx, dy)
 * of the previous pass, s = the record level's s list [s_idx] and o^ = (o_code - 127.5) * 510/256
 * (binary64, s*d then +o^, no contraction).  Pixels no record covers keep their value.
 * rec: device fic_record [n_rec] (e.g. fic_encode's output; any order; ranges must not overlap);
 * h_s / h_n_s: the per-level s lists as passed to fic_encode (level l has B = B_max >> l);
 * out: device [N*N] (may not alias init).  Synchronous.
 * Errors: ARG (null, iterations < 0, a record out of bounds or naming an unknown level / s index /
 * isometry), CUDA. */
fic_status fic_decode(fic_ctx *ctx, const fic_record *rec, int64_t n_rec, int32_t N, int32_t B_max,
                      int32_t n_levels, const double *h_s, const int32_t *h_n_s, int32_t iterations,
                      const uint8_t *init, uint8_t *out);

/* PSNR of two device images of n pixels ("PSNR", reading R26):
 * 10 log10(255^2 / MSE) with MSE = (exact integer sum of squared differences) / n, +inf when
 * identical.  *h_psnr receives the value.  Synchronous.  Errors: ARG, CUDA. */
fic_status fic_psnr(fic_ctx *ctx, const uint8_t *a, const uint8_t *b, int64_t n, double *h_psnr);

/* FIC1 container of a code (NEXT-3; SPEC S:352-413 -- the paper fixes no format, P:154 reports
 * compression ratios): magic "FIC1", header (width u16, height u16, B_max u8, B_min u8,
 * s_mode u8, s_max u16 x 10000, L u16, big-endian; one u8 per level = that level's s count), then
 * the depth-first quadtree walk of the top-level blocks in row-major order, children row-major,
 * one split bit per visited range above B_min, per leaf [dx / L, dy / L (ceil log2 A bits each,
 * A = (N - 2B) / L + 1), isometry (3), s index (ceil log2 |S_B| bits), o code (8)], MSB first,
 * zero-padded to a byte.
 * rec: device fic_record [n_rec], one per leaf (fic_encode's output; any order; the leaves must
 * tile the image); h_n_s: per-level s counts; s_mode: 0 predefined, 1 sampled10, 2 closed form
 * (5 bits), 3 grid; out: device [capacity] bytes.  *h_nbytes = stream length (also when it does
 * not fit).  Synchronous.  Errors: ARG, CAPACITY (stream longer than capacity), CUDA. */
fic_status fic_serialize(fic_ctx *ctx, const fic_record *rec, int64_t n_rec, int32_t N, int32_t B_max,
                         int32_t B_min, int32_t L, const int32_t *h_n_s, int32_t s_mode, double s_max,
                         uint8_t *out, int64_t capacity, int64_t *h_nbytes);

/* Host-only: the entropy fixed-point table lut[c] = round-half-even(c log2(c) 2^32),
 * c = 0..mmax (h_lut host int64 [mmax+1]).  No device work. */
fic_status fic_entropy_lut(int64_t *h_lut, int32_t mmax);

/* Library version string (host-only). */
const char *fic_version(void);

#ifdef __cplusplus
}
#endif
#endif /* FIC_H_ */
