// fic_code.cu -- the FIC1 container body (NEXT-3, the paper fixes no format and
// only reports compression ratios): the depth-first quadtree walk with row-major child
// order, one split bit per visited range above min_range, and per leaf
// [dx / L, dy / L, isometry (3), s index, o code (8)], bit-packed MSB-first.
//
// Parallel form of the walk: with children in row-major order the depth-first order of the
// leaves is (top-level block row-major, Morton code of the leaf origin inside it, y bit above x
// bit), and an internal node's split bit (1) is emitted right before its top-left descendant
// leaf.  So every leaf owns one contiguous bit run: its "opened" ancestors (those whose origin is
// its origin), its own split bit (0, if B > B_min) and its payload.  Sort the leaves by that key,
// exclusive-scan the run lengths, and let each leaf OR its bits in.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include "fic_internal.cuh"

namespace fic {

__device__ __forceinline__ int ilog2(int v) { return 31 - __clz(v); }

// a record the container can hold: B a level in [B_min, B_max], the range inside the image on
// its quadtree grid, the domain origin a candidate position of its level (multiple of L,
// 2B x 2B block inside the image), iso < 8, s_idx below the level's s count
__device__ __forceinline__ bool leaf_valid(const fic_record &r, const CodeParams &P) {
    if (r.B < P.B_min || r.B > P.B_max || (r.B & (r.B - 1)) != 0) return false;
    const int li = ilog2(P.B_max) - ilog2(r.B);
    const int64_t N = P.N, B = r.B;
    if (r.rx < 0 || r.ry < 0 || (int64_t)r.rx > N - B || (int64_t)r.ry > N - B || r.rx % r.B || r.ry % r.B)
        return false;
    if (r.dx < 0 || r.dy < 0 || (int64_t)r.dx > N - 2 * B || (int64_t)r.dy > N - 2 * B || r.dx % P.L || r.dy % P.L)
        return false;
    return r.iso < 8 && (int)r.s_idx < P.n_s[li];
}

// bit run of one leaf: (value right-aligned, MSB first; length)
__device__ __forceinline__ void leaf_bits(const fic_record &r, const CodeParams &P, uint64_t &v, int &len) {
    v = 0;
    len = 0;
    auto put = [&](uint64_t x, int w) {
        v = (v << w) | (x & ((w == 64) ? ~0ull : ((1ull << w) - 1)));
        len += w;
    };
    const int li = ilog2(P.B_max) - ilog2(r.B);  // level index (0 = B_max)
    for (int Bp = P.B_max; Bp > r.B; Bp >>= 1)    // opened ancestors, outermost first
        if (r.rx % Bp == 0 && r.ry % Bp == 0) put(1, 1);
    if (r.B > P.B_min) put(0, 1);  // this range is a leaf
    const int pb = P.posbits[li];
    put((uint64_t)(r.dx / P.L), pb);
    put((uint64_t)(r.dy / P.L), pb);
    put(r.iso, 3);
    put(r.s_idx, P.sbits[li]);
    put(r.o_code, 8);
}

__global__ void code_key_kernel(const fic_record *__restrict__ rec, int64_t n, const CodeParams P,
                                unsigned long long *__restrict__ keys, int32_t *__restrict__ idx,
                                uint32_t *__restrict__ lens, int32_t *__restrict__ d_bad) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const fic_record r = rec[i];
    if (!leaf_valid(r, P)) {  // reported as FIC_ERR_ARG; contributes no bits
        *d_bad = 1;
        keys[i] = ~0ull;
        idx[i] = (int32_t)i;
        lens[i] = 0;
        return;
    }
    const int G = P.N / P.B_max;
    const unsigned long long top = (unsigned long long)(r.ry / P.B_max) * G + (r.rx / P.B_max);
    const int lx = (r.rx % P.B_max) / P.B_min, ly = (r.ry % P.B_max) / P.B_min;
    unsigned morton = 0;
    for (int k = 0; k < 16; ++k) morton |= (((ly >> k) & 1u) << (2 * k + 1)) | (((lx >> k) & 1u) << (2 * k));
    keys[i] = (top << 32) | morton;
    idx[i] = (int32_t)i;
    uint64_t v;
    int len;
    leaf_bits(r, P, v, len);
    lens[i] = (uint32_t)len;
}

__global__ void code_gather_len_kernel(const int32_t *__restrict__ idx, const uint32_t *__restrict__ lens, int64_t n,
                                       unsigned long long *__restrict__ lsorted) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) lsorted[i] = lens[idx[i]];
}

// stream bit p (MSB first within its byte) of a little-endian word array
__global__ void code_write_kernel(const fic_record *__restrict__ rec, const int32_t *__restrict__ idx,
                                  const unsigned long long *__restrict__ off, int64_t n, const CodeParams P,
                                  unsigned *__restrict__ words, unsigned long long *__restrict__ d_total) {
    const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n) return;
    uint64_t v = 0;
    int len = 0;
    const fic_record r = rec[idx[j]];
    if (leaf_valid(r, P)) leaf_bits(r, P, v, len);
    const unsigned long long p0 = off[j];
    if (j == n - 1) *d_total = p0 + (unsigned long long)len;
    unsigned long long cur_w = ~0ull;
    unsigned mask = 0;
    for (int b = 0; b < len; ++b) {
        if (!((v >> (len - 1 - b)) & 1ull)) continue;
        const unsigned long long p = p0 + b;
        const unsigned long long byte = p >> 3, w = byte >> 2;
        const unsigned bit = 8u * (unsigned)(byte & 3) + 7u - (unsigned)(p & 7);
        if (w != cur_w) {
            if (mask) atomicOr(&words[cur_w], mask);
            cur_w = w;
            mask = 0;
        }
        mask |= 1u << bit;
    }
    if (mask) atomicOr(&words[cur_w], mask);
}

size_t code_scratch_bytes(int64_t n) {
    auto al = [](size_t b) { return (b + 255) & ~(size_t)255; };
    size_t s0 = 0, s1 = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, s0, (const unsigned long long *)nullptr, (unsigned long long *)nullptr,
                                    (const int32_t *)nullptr, (int32_t *)nullptr, (int)n);
    cub::DeviceScan::ExclusiveSum(nullptr, s1, (const unsigned long long *)nullptr, (unsigned long long *)nullptr,
                                  (int)n);
    return 2 * al(8 * n) + 2 * al(4 * n) + al(4 * n) + 2 * al(8 * n) + al(8) + al(s0 > s1 ? s0 : s1);
}

cudaError_t launch_code_body(const fic_record *rec, int64_t n, const CodeParams &P, void *scratch,
                             unsigned *words, unsigned long long *d_total, int32_t *d_bad, cudaStream_t st) {
    if (n == 0) return cudaMemsetAsync(d_total, 0, sizeof(unsigned long long), st);
    auto al = [](size_t b) { return (b + 255) & ~(size_t)255; };
    char *b = static_cast<char *>(scratch);
    unsigned long long *keys = reinterpret_cast<unsigned long long *>(b); b += al(8 * n);
    unsigned long long *kout = reinterpret_cast<unsigned long long *>(b); b += al(8 * n);
    int32_t *idx = reinterpret_cast<int32_t *>(b); b += al(4 * n);
    int32_t *iout = reinterpret_cast<int32_t *>(b); b += al(4 * n);
    uint32_t *lens = reinterpret_cast<uint32_t *>(b); b += al(4 * n);
    unsigned long long *ls = reinterpret_cast<unsigned long long *>(b); b += al(8 * n);
    unsigned long long *off = reinterpret_cast<unsigned long long *>(b); b += al(8 * n);
    b += al(8);
    size_t tb = 0, s0 = 0, s1 = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, s0, keys, kout, idx, iout, (int)n);
    cub::DeviceScan::ExclusiveSum(nullptr, s1, ls, off, (int)n);
    tb = s0 > s1 ? s0 : s1;
    const unsigned g = (unsigned)((n + 255) / 256);
    code_key_kernel<<<g, 256, 0, st>>>(rec, n, P, keys, idx, lens, d_bad);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    e = cub::DeviceRadixSort::SortPairs(b, tb, keys, kout, idx, iout, (int)n, 0, 64, st);
    if (e != cudaSuccess) return e;
    code_gather_len_kernel<<<g, 256, 0, st>>>(iout, lens, n, ls);
    e = cub::DeviceScan::ExclusiveSum(b, tb, ls, off, (int)n, st);
    if (e != cudaSuccess) return e;
    code_write_kernel<<<g, 256, 0, st>>>(rec, iout, off, n, P, words, d_total);
    return cudaGetLastError();
}

}  // namespace fic
