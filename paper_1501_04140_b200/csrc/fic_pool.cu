// fic_pool.cu -- domain-pool construction kernels and the
// order-preserving compactions used by the pool (kept list) and the quadtree (a8).
//
//   entropy_keys_kernel  P:44-56 Eq. (4)-(5) + Abstract P:14: entropy of each raw 2B x 2B candidate
//                        as the exact fixed-point key  K = LUT[m] - sum_v LUT[h_v]  [R6]
//   select_*             row-major compaction (kept list, next-level ranges, accepted records)
//   pool_moments_kernel  SD = sum D', SDD = sum D'^2, C = n SDD - SD^2 (int64, exact)
#include <atomic>
#include <cfloat>
#include <cstdio>

#include <cub/device/device_radix_sort.cuh>

#include "fic_internal.cuh"

namespace fic {

// ------------------------------------------------------------------------------------ entropy

// Exact warp sum of int64 values in three 22-bit limbs (each limb sum < 2^27 over 32 lanes, the
// top limb signed): three single-instruction warp reductions instead of five 64-bit shuffle
// rounds.
__device__ __forceinline__ int64_t warp_sum_i64(int64_t v) {
    const int l0 = (int)(v & 0x3FFFFF), l1 = (int)((v >> 22) & 0x3FFFFF), l2 = (int)(v >> 44);
    const int s0 = __reduce_add_sync(0xffffffffu, l0);
    const int s1 = __reduce_add_sync(0xffffffffu, l1);
    const int s2 = __reduce_add_sync(0xffffffffu, l2);
    return (int64_t)s0 + ((int64_t)s1 << 22) + ((int64_t)s2 << 44);
}

// One warp per candidate (grid-stride).  Each warp owns a 256-bin histogram in shared memory.
// The key is accumulated while the histogram is built: inserting a pixel into a bin holding
// `old` pixels adds delta[old] = LUT[old+1] - LUT[old], so after all m insertions the sum is
// sum_v LUT[h_v] exactly, whatever the insertion order (integer telescoping).
__global__ void __launch_bounds__(256) entropy_keys_kernel(
    const uint8_t *__restrict__ img, int32_t N, int32_t side, int32_t L, int32_t A,
    const int64_t *__restrict__ g_delta, int64_t lut_m, int64_t T, int use_tau,
    int64_t *__restrict__ keys, uint8_t *__restrict__ keep) {
    extern __shared__ __align__(16) unsigned char sm[];
    const int m = side * side;
    int64_t *delta = reinterpret_cast<int64_t *>(sm);
    int32_t *hist_all = reinterpret_cast<int32_t *>(sm + sizeof(int64_t) * m);
    for (int i = threadIdx.x; i < m; i += blockDim.x) delta[i] = g_delta[i];
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    int32_t *hist = hist_all + warp * 256;
    const int lgs = __ffs(side) - 1;
    const int64_t n_c = (int64_t)A * A;
    const int64_t wstride = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t c = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp; c < n_c; c += wstride) {
        for (int v = lane; v < 256; v += 32) hist[v] = 0;
        __syncwarp();
        const int64_t x = (c % A) * L, y = (c / A) * L;
        const uint8_t *base = img + y * N + x;
        int64_t acc = 0;
        for (int idx = lane; idx < m; idx += 32) {  // side = 2B is a power of two
            const int i = idx >> lgs, j = idx & (side - 1);
            const int v = base[i * N + j];
            const int old = atomicAdd(&hist[v], 1);
            acc += delta[old];
        }
        acc = warp_sum_i64(acc);
        if (lane == 0) {
            const int64_t key = lut_m - acc;
            keys[c] = key;
            keep[c] = (uint8_t)(!use_tau || key > T);
        }
        __syncwarp();
    }
}

// Sliding-window form for large blocks (2B > 2L): one warp per run of kSlideSeg consecutive
// candidates of one candidate row.  The first histogram is built by m insertions; each step to
// the next candidate (L columns to the right) removes the L leaving columns and inserts the L
// entering ones (2 L side updates instead of m).  Removing a pixel from a bin holding `old`
// adds LUT[old-1] - LUT[old] = -delta[old-1]; per bin the contributions telescope to
// LUT[final] - LUT[initial] in any order (a removed pixel is always present, so no count goes
// negative), so every key is the same exact integer as the direct build.
#ifndef FIC_SLIDE_SEG
#define FIC_SLIDE_SEG 12
#endif
constexpr int kSlideSeg = FIC_SLIDE_SEG;
__global__ void __launch_bounds__(256) entropy_slide_kernel(
    const uint8_t *__restrict__ img, int32_t N, int32_t side, int32_t L, int32_t A,
    const int64_t *__restrict__ g_delta, int64_t lut_m, int64_t T, int use_tau,
    int64_t *__restrict__ keys, uint8_t *__restrict__ keep) {
    extern __shared__ __align__(16) unsigned char sm[];
    pdl_wait();
    pdl_trigger();
    const int m = side * side;
    int64_t *delta = reinterpret_cast<int64_t *>(sm);
    int32_t *hist_all = reinterpret_cast<int32_t *>(sm + sizeof(int64_t) * m);
    for (int i = threadIdx.x; i < m; i += blockDim.x) delta[i] = g_delta[i];
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    int32_t *hist = hist_all + warp * 256;
    const int segs = (A + kSlideSeg - 1) / kSlideSeg;
    const int64_t w = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp;
    if (w >= (int64_t)A * segs) return;
    const int b = (int)(w / segs), a0 = (int)(w % segs) * kSlideSeg, a1 = min(A, a0 + kSlideSeg);
    const int64_t y = (int64_t)b * L;
    const uint8_t *rowbase = img + y * N;  // the warp's band of rows
    for (int v = lane; v < 256; v += 32) hist[v] = 0;
    __syncwarp();
    int64_t acc = 0;
    {
        const uint8_t *base = rowbase + (int64_t)a0 * L;
        const int lgs = __ffs(side) - 1;  // side = 2B is a power of two
        for (int idx = lane; idx < m; idx += 32) {
            const int old = atomicAdd(&hist[base[(idx >> lgs) * N + (idx & (side - 1))]], 1);
            acc += delta[old];
        }
    }
    const int nu = L * side;  // pixels leaving (and entering) per step
    // this lane's pixels of a step are the same for every step (relative to x = a L): their
    // offsets (leaving columns x .. x + L - 1, entering x + side ..) are formed once, so the step
    // loop has no division by L and no 64-bit address arithmetic
    constexpr int kSlots = 8;
    int off[kSlots];
    unsigned leaving = 0, valid = 0;
#pragma unroll
    for (int t = 0; t < kSlots; ++t) {
        const int u = lane + 32 * t;
        const bool lv = u < nu;
        const int uu = lv ? u : u - nu;
        const int i = uu / L, j = uu - (uu / L) * L;
        off[t] = i * N + j + (lv ? 0 : side);
        if (u < 2 * nu) valid |= 1u << t;
        if (lv) leaving |= 1u << t;
    }
    const bool fits = 2 * nu <= 32 * kSlots;
    for (int a = a0;; ++a) {
        const int64_t tot = warp_sum_i64(acc);
        if (lane == 0) {
            const int64_t key = lut_m - tot;
            const int64_t c = (int64_t)b * A + a;
            keys[c] = key;
            keep[c] = (uint8_t)(!use_tau || key > T);
        }
        if (a + 1 >= a1) break;
        __syncwarp();
        const uint8_t *base = rowbase + (int64_t)a * L;
        if (fits) {
#pragma unroll
            for (int t = 0; t < kSlots; ++t) {
                if (!((valid >> t) & 1u)) continue;
                const int v = base[off[t]];
                if ((leaving >> t) & 1u) {  // leaving column x + j
                    const int old = atomicSub(&hist[v], 1);
                    acc -= delta[old - 1];
                } else {                    // entering column x + side + j
                    const int old = atomicAdd(&hist[v], 1);
                    acc += delta[old];
                }
            }
        } else {
            for (int u = lane; u < 2 * nu; u += 32) {
                const int uu = u < nu ? u : u - nu;
                const int i = uu / L, j = uu - i * L;
                if (u < nu) {
                    const int old = atomicSub(&hist[base[i * N + j]], 1);
                    acc -= delta[old - 1];
                } else {
                    const int old = atomicAdd(&hist[base[i * N + side + j]], 1);
                    acc += delta[old];
                }
            }
        }
        __syncwarp();
    }
}

cudaError_t launch_entropy_keys(const uint8_t *img, int32_t N, int32_t B, int32_t L, int32_t A,
                                const int64_t *d_delta, int64_t lut_m, int64_t T, int use_tau,
                                int64_t *keys, uint8_t *keep, cudaStream_t st) {
    const int side = 2 * B, m = side * side;
    if (B >= 8 && L < side / 2) {  // sliding windows pay off (>= 4x fewer histogram updates)
        const size_t smem = sizeof(int64_t) * m + 8 * 256 * sizeof(int32_t);
        static std::atomic<unsigned long long> attr2{0};
        if (cudaError_t e = ensure_smem_attr(entropy_slide_kernel, 64 * 1024, attr2)) return e;
        const int64_t warps = (int64_t)A * ((A + kSlideSeg - 1) / kSlideSeg);
        return launch_pdl(entropy_slide_kernel, dim3((unsigned)((warps + 7) / 8)), dim3(256), smem, st, img, N, side, L,
                          A, d_delta, lut_m, T, use_tau, keys, keep);
    }
    const size_t smem = sizeof(int64_t) * m + 8 * 256 * sizeof(int32_t);
    static std::atomic<unsigned long long> attr{0};
    if (cudaError_t e = ensure_smem_attr(entropy_keys_kernel, 64 * 1024, attr)) return e;
    const int64_t n_c = (int64_t)A * A;
    int64_t blocks = (n_c + 7) / 8;
    if (blocks > 148 * 8) blocks = 148 * 8;
    if (blocks < 1) blocks = 1;
    entropy_keys_kernel<<<(unsigned)blocks, 256, smem, st>>>(img, N, side, L, A, d_delta, lut_m, T,
                                                             use_tau, keys, keep);
    return cudaGetLastError();
}

// ------------------------------------------------------------------------- order-preserving select
constexpr int kSelBlock = 4096;  // flags per CTA (select_chain_kernel); one scratch word each

size_t select_blocksum_len(int64_t n) { return (size_t)((n + kSelBlock - 1) / kSelBlock) + 1; }

struct EmitIndex {
    static constexpr bool kClear = false, kBlockCopy = false;
    int32_t *out;
    __device__ void operator()(int64_t i, int64_t pos) const { out[pos] = (int32_t)i; }
};
struct EmitGrid {  // the child bitmap is cleared as it is consumed (ready for the next level)
    static constexpr bool kClear = true, kBlockCopy = false;
    int2 *out;
    int64_t G;
    int32_t B;
    __device__ void operator()(int64_t i, int64_t pos) const {  // (G * G < 2^31: 32-bit division)
        const int ii = (int)i, g = (int)G;
        out[pos] = make_int2((ii % g) * B, (ii / g) * B);
    }
};
// records are moved as five 8-byte words so padding bytes (zero) are preserved
__device__ __forceinline__ void copy_record(fic_record *dst, const fic_record *src) {
    const uint64_t *s = reinterpret_cast<const uint64_t *>(src);
    uint64_t *d = reinterpret_cast<uint64_t *>(dst);
#pragma unroll
    for (int q = 0; q < 5; ++q) d[q] = s[q];
}

// records: the CTA lists its selected indices in shared memory, then copies the records as
// consecutive 8-byte words (coalesced stores; one thread copying its own records wrote 40-byte
// strided words -- 21.7 us for the ~200k records of C3's B = 4 level)
struct EmitRecord {
    static constexpr bool kClear = false, kBlockCopy = true;
    const fic_record *in;
    fic_record *out;
    const unsigned long long *base;
    int64_t cap;
    // record j of the CTA's selection (index blk0 + idx[j]) to position *base + excl + j
    __device__ void block_copy(const int *idx, int cnt, int64_t blk0, int64_t excl, int t, int nt) const {
        const int64_t o0 = (int64_t)*base + excl;
        const uint64_t *src = reinterpret_cast<const uint64_t *>(in);
        uint64_t *dst = reinterpret_cast<uint64_t *>(out);
        constexpr int WPR = sizeof(fic_record) / 8;  // 8-byte words per record
        static_assert(sizeof(fic_record) % 8 == 0, "records move as 8-byte words");
        for (int wd = t; wd < cnt * WPR; wd += nt) {
            const int j = wd / WPR, k = wd - j * WPR;
            if (o0 + j < cap) dst[(o0 + j) * WPR + k] = src[(blk0 + idx[j]) * WPR + k];
        }
    }
};

// Single-pass order-preserving compaction (index / grid emits): 4096 flags per CTA, block scan,
// then a decoupled look-back over the predecessors' published (aggregate | inclusive prefix)
// words, then the scatter -- one launch, every SM.  A word is tag << 34 | status << 32 | count;
// the per-call tag makes the words of earlier calls (same scratch buffer) invisible, so the
// buffer is never cleared.  Predecessors have lower block indices, which are dispatched first.
constexpr int kChainItems = 16, kChainThreads = 256, kChainBlock = kChainItems * kChainThreads;
template <class Emit>
__global__ void __launch_bounds__(kChainThreads) select_chain_kernel(const uint8_t *flags, int64_t n,
                                                                     Emit emit, unsigned long long *state,
                                                                     uint32_t tag, unsigned long long *d_total,
                                                                     unsigned long long *d_total2) {
    __shared__ int wsum[kChainThreads / 32];
    __shared__ long long s_excl;
    __shared__ int s_tot;
    __shared__ int s_idx[Emit::kBlockCopy ? kChainBlock : 1];
    pdl_wait();
    pdl_trigger();
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const int64_t b0 = (int64_t)blockIdx.x * kChainBlock + (int64_t)t * kChainItems;
    uint32_t w[kChainItems / 4];
    if (b0 + kChainItems <= n && ((reinterpret_cast<uintptr_t>(flags) & 15) == 0)) {
        const uint4 v = *reinterpret_cast<const uint4 *>(flags + b0);
        w[0] = v.x; w[1] = v.y; w[2] = v.z; w[3] = v.w;
        if constexpr (Emit::kClear) *reinterpret_cast<uint4 *>(const_cast<uint8_t *>(flags) + b0) = make_uint4(0, 0, 0, 0);
    } else {
#pragma unroll
        for (int q = 0; q < kChainItems / 4; ++q) {
            uint32_t x = 0;
            for (int b = 0; b < 4; ++b) {
                const int64_t i = b0 + 4 * q + b;
                if (i < n) {
                    x |= (uint32_t)(flags[i] & 1) << (8 * b);
                    if constexpr (Emit::kClear) const_cast<uint8_t *>(flags)[i] = 0;
                }
            }
            w[q] = x;
        }
    }
    int cnt = 0;
#pragma unroll
    for (int q = 0; q < kChainItems / 4; ++q) {
        w[q] &= 0x01010101u;  // flags are 0/1 bytes
        cnt += __popc(w[q]);
    }
    int incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += v;
    }
    if (lane == 31) wsum[warp] = incl;
    __syncthreads();
    if (warp == 0) {
        // warp 0: the CTA's exclusive warp offsets and total, then a warp-wide look-back over 32
        // predecessors at a time (the nearest one holding an inclusive prefix ends it; the
        // aggregates before it are summed) -- one dependent round of loads per 32 predecessors
        // instead of one per predecessor
        long long tot = 0;
        if (lane == 0) {
            for (int i = 0; i < kChainThreads / 32; ++i) {
                const int ws = wsum[i];
                wsum[i] = (int)tot;
                tot += ws;
            }
        }
        tot = __shfl_sync(0xffffffffu, tot, 0);
        const unsigned long long T = (unsigned long long)tag << 34;
        volatile unsigned long long *vs = state;
        long long excl = 0;
        if (blockIdx.x == 0) {
            if (lane == 0) vs[0] = T | (2ull << 32) | (unsigned long long)tot;
        } else {
            if (lane == 0) {
                vs[blockIdx.x] = T | (1ull << 32) | (unsigned long long)tot;  // aggregate
                __threadfence();
            }
            __syncwarp();
            for (int j0 = (int)blockIdx.x - 1;;) {
                const int j = j0 - lane;
                unsigned long long v = 0;
                bool ready = true;
                if (j >= 0) {
                    v = vs[j];
                    ready = (v >> 34) == tag;  // published in this call
                }
                if (!__all_sync(0xffffffffu, ready)) continue;
                const bool inc = j < 0 || ((v >> 32) & 3ull) == 2ull;
                const unsigned im = __ballot_sync(0xffffffffu, inc);
                const int stop = im ? __ffs(im) - 1 : 31;  // nearest inclusive prefix (or the window)
                long long c = lane <= stop && j >= 0 ? (long long)(v & 0xffffffffull) : 0;
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
                excl += c;
                if (im) break;
                j0 -= 32;
            }
            if (lane == 0) {
                __threadfence();
                vs[blockIdx.x] = T | (2ull << 32) | (unsigned long long)(excl + tot);
            }
        }
        if (lane == 0) {
            s_excl = excl;
            s_tot = (int)tot;
            if (blockIdx.x == gridDim.x - 1) {
                *d_total = (unsigned long long)(excl + tot);
                if (d_total2) *d_total2 = (unsigned long long)(excl + tot);
            }
        }
    }
    __syncthreads();
    if constexpr (Emit::kBlockCopy) {
        int lp = wsum[warp] + incl - cnt;  // position within the CTA's selection
#pragma unroll
        for (int q = 0; q < kChainItems / 4; ++q) {
            uint32_t x = w[q];
            while (x) {
                const int bit = __ffs(x) - 1;
                s_idx[lp++] = (int)(t * kChainItems + 4 * q + (bit >> 3));
                x &= x - 1;
            }
        }
        __syncthreads();
        emit.block_copy(s_idx, s_tot, (int64_t)blockIdx.x * kChainBlock, s_excl, t, kChainThreads);
    } else {
        int64_t pos = s_excl + wsum[warp] + incl - cnt;
#pragma unroll
        for (int q = 0; q < kChainItems / 4; ++q) {
            uint32_t x = w[q];
            while (x) {
                const int bit = __ffs(x) - 1;  // lowest set flag byte first: index order
                emit(b0 + 4 * q + (bit >> 3), pos++);
                x &= x - 1;
            }
        }
    }
}

static uint32_t next_chain_tag() {
    static std::atomic<uint32_t> ctr{0};
    uint32_t t;
    do t = (ctr.fetch_add(1) + 1) & 0x3fffffffu; while (t == 0);
    return t;
}

template <class Emit>
static cudaError_t select_run(const uint8_t *flags, int64_t n, int64_t *blocksum, Emit emit,
                              unsigned long long *d_total, cudaStream_t st, unsigned long long *d_total2 = nullptr) {
    const int64_t nb = (n + kSelBlock - 1) / kSelBlock;
    if (nb == 0) {
        if (d_total2) {
            const cudaError_t e = cudaMemsetAsync(d_total2, 0, sizeof(unsigned long long), st);
            if (e != cudaSuccess) return e;
        }
        return cudaMemsetAsync(d_total, 0, sizeof(unsigned long long), st);
    }
    static_assert(kChainBlock == kSelBlock, "blocksum scratch holds one word per chain block");
    return launch_pdl(select_chain_kernel<Emit>, dim3((unsigned)nb), dim3(kChainThreads), 0, st, flags, n, emit,
                      reinterpret_cast<unsigned long long *>(blocksum), next_chain_tag(), d_total, d_total2);
}

cudaError_t launch_select_index(const uint8_t *flags, int64_t n, int64_t *blocksum, int32_t *out,
                                unsigned long long *d_total, cudaStream_t st, unsigned long long *d_total2) {
    return select_run(flags, n, blocksum, EmitIndex{out}, d_total, st, d_total2);
}
cudaError_t launch_select_grid(const uint8_t *flags, int64_t G, int32_t B, int64_t *blocksum,
                               int2 *out, unsigned long long *d_total, cudaStream_t st) {
    return select_run(flags, G * G, blocksum, EmitGrid{out, G, B}, d_total, st);
}
cudaError_t launch_select_records(const uint8_t *flags, int64_t n, int64_t *blocksum,
                                  const fic_record *in, fic_record *out, const unsigned long long *d_base,
                                  int64_t capacity, unsigned long long *d_total, cudaStream_t st) {
    return select_run(flags, n, blocksum, EmitRecord{in, out, d_base, capacity}, d_total, st);
}

__global__ void set_u64_kernel(unsigned long long *p, unsigned long long v) { *p = v; }

cudaError_t launch_set_u64(unsigned long long *d, unsigned long long v, cudaStream_t st) {
    set_u64_kernel<<<1, 1, 0, st>>>(d, v);
    return cudaGetLastError();
}

__global__ void accumulate_kernel(unsigned long long *acc, const unsigned long long *add) { *acc += *add; }

// The encode's counters straight into page-locked host memory (mapped under UVA): one tiny kernel
// after the join instead of a device -> host copy-engine transfer.
__global__ void copy_counts_kernel(const unsigned long long *__restrict__ src, unsigned long long *dst, int n) {
    const int i = threadIdx.x;
    if (i < n) dst[i] = src[i];
}

cudaError_t launch_copy_counts(const unsigned long long *d_src, unsigned long long *h_dst, int n, cudaStream_t st) {
    copy_counts_kernel<<<1, 64, 0, st>>>(d_src, h_dst, n);
    return cudaGetLastError();
}

cudaError_t launch_accumulate(unsigned long long *d_acc, const unsigned long long *d_add, cudaStream_t st) {
    accumulate_kernel<<<1, 1, 0, st>>>(d_acc, d_add);
    return cudaGetLastError();
}

__global__ void top_flags_kernel(uint8_t *flags, int64_t n, int32_t shard, int32_t n_shards) {
    pdl_wait();
    pdl_trigger();
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) flags[i] = (uint8_t)((i % n_shards) == shard);
}

cudaError_t launch_top_flags(uint8_t *flags, int64_t G, int32_t shard, int32_t n_shards,
                             cudaStream_t st) {
    const int64_t n = G * G;
    return launch_pdl(top_flags_kernel, dim3((unsigned)((n + 255) / 256)), dim3(256), 0, st, flags, n, shard, n_shards);
}

// Warp per domain slot: SD, SDD (int), C = n SDD - SD^2 (int64); pads get zeros.
__global__ void __launch_bounds__(256) pool_moments_kernel(const uint8_t *__restrict__ img, int32_t N,
                                                           int32_t B, int32_t L, int32_t A,
                                                           const int32_t *__restrict__ kept,
                                                           const unsigned long long *__restrict__ d_nk,
                                                           int64_t n_slots, int32_t *__restrict__ SD,
                                                           float *__restrict__ SDf,
                                                           int64_t *__restrict__ C,
                                                           unsigned long long *d_cmax) {
    const int64_t d = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    const int64_t n_k = (int64_t)*d_nk;
    const int64_t ntiles = (n_k + kTileD - 1) / kTileD;
    const bool live = d < n_slots && d < ntiles * kTileD;  // (no early return: block_max_atomic)
    const int n = B * B;
    int64_t sd = 0, sdd = 0;
    if (live && d < n_k) {
        const int32_t c = kept[d];
        const int64_t x = (int64_t)(c % A) * L, y = (int64_t)(c / A) * L;
        for (int p = lane; p < n; p += 32) {
            const int i = p / B, j = p - (p / B) * B;
            const uint8_t *q = img + (y + 2 * i) * N + x + 2 * j;
            const int v = (int)q[0] + (int)q[1] + (int)q[N] + (int)q[N + 1];
            sd += v;
            sdd += (int64_t)v * v;
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        sd += __shfl_xor_sync(0xffffffffu, sd, o);
        sdd += __shfl_xor_sync(0xffffffffu, sdd, o);
    }
    const int64_t cc = (int64_t)n * sdd - sd * sd;
    if (lane == 0 && live) {
        SD[d] = (int32_t)sd;
        SDf[d] = (float)sd;
        C[d] = cc;
    }
    block_max_atomic(live && d < n_k ? (unsigned long long)cc : 0ull, d_cmax);
}

cudaError_t launch_pool_moments(const uint8_t *img, int32_t N, int32_t B, int32_t L, int32_t A,
                                const int32_t *kept, const unsigned long long *d_nk,
                                int64_t n_slots, int32_t *SD, float *SDf, int64_t *C,
                                unsigned long long *d_cmax, cudaStream_t st) {
    if (n_slots == 0) return cudaSuccess;
    const int64_t threads = n_slots * 32;
    pool_moments_kernel<<<(unsigned)((threads + 255) / 256), 256, 0, st>>>(
        img, N, B, L, A, kept, d_nk, n_slots, SD, SDf, C, d_cmax);
    return cudaGetLastError();
}

// t2f[j][d] = fp32 of (s_j s_j)(C/16) for s_j > 0; +inf for pad slots (never admitted).
// univ (large s sets, the s-independent filter): t2f[0][d] = RN(1/C) (0 if C = 0), NaN on pads.
// fold > 0 (tcgen05 filter at B <= 8, one or two s): the table holds RN(t2 - nhs_j * 1.5 * 2^23)
// with nhs_j = -RN(s_j / 2) * fold, so the epilogue's g = fma(nhs, magic-converted Bq, t2') needs
// no subtraction of the magic constant (the extra rounding is in the filter margin)
__global__ void t2f_kernel(const int64_t *__restrict__ C, const unsigned long long *__restrict__ d_nk,
                           int64_t n_slots, const SList spos, int32_t nsp, float *__restrict__ t2f, int32_t univ,
                           float fold, float grid_h) {
    pdl_wait();
    pdl_trigger();
    const int64_t d = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (d >= n_slots) return;
    const int64_t n_k = (int64_t)*d_nk;
    if (d >= ((n_k + kTileD - 1) / kTileD) * kTileD) return;
    if (univ == 2) {  // uniform grid: RN(C / 16) (+inf on pads: never passes), RN(4 / (C h))
        t2f[d] = d < n_k ? __double2float_rn(__dmul_rn(0.0625, (double)C[d])) : INFINITY;
        t2f[n_slots + d] = (d < n_k && C[d] > 0) ? __double2float_rn(4.0 / ((double)C[d] * (double)grid_h)) : 0.f;
        return;
    }
    if (univ) {
        t2f[d] = d < n_k ? (C[d] > 0 ? __double2float_rn(1.0 / (double)C[d]) : 0.f) : __int_as_float(0x7fc00000);
        return;
    }
    const double c16 = __dmul_rn(0.0625, (double)C[d]);
    for (int j = 0; j < nsp; ++j) {
        const double s = spos.s[j];
        double t = __dmul_rn(__dmul_rn(s, s), c16);
        if (fold > 0.f) {
            const double nhs = -(double)__double2float_rn(0.5 * s) * (double)fold;  // as the epilogue
            t = __dsub_rn(t, nhs * 12582912.0);                                     // (product exact)
        }
        t2f[j * n_slots + d] = d < n_k ? __double2float_rn(t) : INFINITY;
    }
}

cudaError_t launch_t2f(const int64_t *C, const unsigned long long *d_nk, int64_t n_slots, const SList &spos,
                       int32_t nsp, float *t2f, int32_t univ, float fold, cudaStream_t st, float grid_h) {
    if (n_slots == 0 || nsp == 0) return cudaSuccess;
    return launch_pdl(t2f_kernel, dim3((unsigned)((n_slots + 255) / 256)), dim3(256), 0, st, C, d_nk, n_slots, spos,
                      nsp, t2f, univ, fold, grid_h);
}

// ----------------------------------------------------------------------------- shard merge
// Records of every shard are sorted by key (B desc, ry, rx) and the shards' range sets are
// disjoint, so a record's output slot is its index in its own list plus, for every other shard,
// the number of that shard's records with a smaller key (binary search).
__device__ __forceinline__ uint64_t rec_key(const fic_record &r) {
    const int lg = 31 - __clz(r.B);
    return ((uint64_t)(8 - lg) << 48) | ((uint64_t)(uint32_t)r.ry << 24) | (uint64_t)(uint32_t)r.rx;
}

__global__ void merge_shards_kernel(const fic_record *__restrict__ in,
                                    const int64_t *__restrict__ counts, int32_t n_shards,
                                    int64_t stride, fic_record *__restrict__ out) {
    const int32_t sh = blockIdx.y;
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= counts[sh]) return;
    const fic_record &r = in[sh * stride + i];
    const uint64_t k = rec_key(r);
    int64_t pos = i;
    for (int32_t o = 0; o < n_shards; ++o) {
        if (o == sh) continue;
        int64_t lo = 0, hi = counts[o];
        const fic_record *L = in + o * stride;
        while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if (rec_key(L[mid]) < k) lo = mid + 1; else hi = mid;
        }
        pos += lo;
    }
    copy_record(out + pos, &r);
}

cudaError_t launch_merge_shards(const fic_record *in, const int64_t *d_counts, int32_t n_shards,
                                int64_t stride, int64_t max_count, fic_record *out,
                                cudaStream_t st) {
    if (max_count == 0) return cudaSuccess;
    dim3 grid((unsigned)((max_count + 255) / 256), (unsigned)n_shards);
    merge_shards_kernel<<<grid, 256, 0, st>>>(in, d_counts, n_shards, stride, out);
    return cudaGetLastError();
}

// ----------------------------------------------------------------------------- top-K selection
// The paper's "pool size" (Tables 1-2, Fig. 4; reading R27): keep the K candidates
// with the largest entropy keys, ties to the lower row-major index.  A stable descending radix
// sort of (key, index) pairs (CUB; equal keys keep ascending index order) ranks them; the first
// K indices are flagged and the usual order-preserving compaction builds the row-major kept list.
__global__ void iota_kernel(int32_t *__restrict__ v, int64_t n) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) v[i] = (int32_t)i;
}
__global__ void topk_flag_kernel(const int32_t *__restrict__ order, int64_t n, int64_t K, uint8_t *__restrict__ keep) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) keep[order[i]] = (uint8_t)(i < K);
}

struct TopkLayout {
    size_t kout, vin, vout, tmp, tmp_bytes, total;
};
static TopkLayout topk_layout(int64_t n) {
    auto al = [](size_t x) { return (x + 255) & ~(size_t)255; };
    TopkLayout L;
    size_t o = 0;
    L.kout = o; o += al(sizeof(int64_t) * n);
    L.vin = o; o += al(sizeof(int32_t) * n);
    L.vout = o; o += al(sizeof(int32_t) * n);
    L.tmp_bytes = 0;
    cub::DeviceRadixSort::SortPairsDescending(nullptr, L.tmp_bytes, (const int64_t *)nullptr, (int64_t *)nullptr,
                                              (const int32_t *)nullptr, (int32_t *)nullptr, (int)n, 0, 50);
    L.tmp = o; o += al(L.tmp_bytes);
    L.total = o;
    return L;
}

size_t topk_scratch_bytes(int64_t n_c) { return topk_layout(n_c).total; }

cudaError_t launch_topk_select(const int64_t *keys, int64_t n_c, int64_t K, void *scratch, uint8_t *keep,
                               cudaStream_t st) {
    if (n_c == 0) return cudaSuccess;
    const TopkLayout Ly = topk_layout(n_c);
    char *b = static_cast<char *>(scratch);
    int64_t *kout = reinterpret_cast<int64_t *>(b + Ly.kout);
    int32_t *vin = reinterpret_cast<int32_t *>(b + Ly.vin), *vout = reinterpret_cast<int32_t *>(b + Ly.vout);
    const unsigned g = (unsigned)((n_c + 255) / 256);
    iota_kernel<<<g, 256, 0, st>>>(vin, n_c);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    size_t tb = Ly.tmp_bytes;
    // keys = lut[m] - sum lut[h] >= 0 and < 2^50 for m <= 4096 (lut[4096] < 2^48)
    e = cub::DeviceRadixSort::SortPairsDescending(b + Ly.tmp, tb, keys, kout, vin, vout, (int)n_c, 0, 50, st);
    if (e != cudaSuccess) return e;
    topk_flag_kernel<<<g, 256, 0, st>>>(vout, n_c, K, keep);
    return cudaGetLastError();
}

}  // namespace fic
