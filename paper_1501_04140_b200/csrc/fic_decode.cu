// fic_decode.cu -- PIFS decoding and PSNR (the quality side of the paper's CR/time/PSNR
// triplet, §4).  The paper only encodes; the decoder is the standard
// iteration implied by §2 lines 28-30 ("an affine transformation that maps the selected domain
// block"), with readings R23-R26:
//   o^ = (code - 127.5) * 510/256 (centre of the R11 cell);
//   one Jacobi pass: out(R) = clamp(rint(s * d + o^), 0, 255), d = T_k(D'/4) of the 2B x 2B
//   block at (dx, dy) of the previous iterate, binary64, s * d then + o^ (no contraction);
//   start from the constant image 128 (or a caller image); a fixed number of passes.
// Layout: an owner map (record index per pixel, -1 = not covered: keeps its value) built once,
// then one thread per pixel per pass (ping-pong buffers).  Parity: tests/test_gpu_decode.py.
#include <algorithm>
#include <cmath>

#include "fic_internal.cuh"

namespace fic {

struct DecRec {     // per record, ready for the pass kernel
    double s, o;    // contrast and dequantised offset
    int32_t rx, ry, dx, dy;
    int32_t B, iso;
};

// validate records, build DecRec and the owner map; *d_bad = 1 on an invalid record
__global__ void dec_prep_kernel(const fic_record *__restrict__ rec, int64_t n_rec, int32_t N, int32_t B_max,
                                int32_t n_levels, DecSList sl, DecRec *__restrict__ par,
                                int32_t *__restrict__ owner, int32_t *__restrict__ d_bad) {
    const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= n_rec) return;
    const fic_record r = rec[q];
    int l = 0;
    while (l < n_levels && (B_max >> l) > r.B) ++l;
    const bool ok = l < n_levels && (B_max >> l) == r.B && r.B >= 1 && r.s_idx < sl.n_s[l] && r.iso < 8 &&
                    r.rx >= 0 && r.ry >= 0 && (int64_t)r.rx + r.B <= N && (int64_t)r.ry + r.B <= N && r.dx >= 0 &&
                    r.dy >= 0 && (int64_t)r.dx + 2 * (int64_t)r.B <= N && (int64_t)r.dy + 2 * (int64_t)r.B <= N;
    if (!ok) {
        *d_bad = 1;
        return;
    }
    DecRec p;
    p.s = sl.s[sl.off[l] + r.s_idx];
    p.o = ((double)r.o_code - 127.5) * 1.9921875;
    p.rx = r.rx; p.ry = r.ry; p.dx = r.dx; p.dy = r.dy; p.B = r.B; p.iso = r.iso;
    par[q] = p;
    for (int i = 0; i < r.B; ++i)
        for (int j = 0; j < r.B; ++j) owner[(int64_t)(r.ry + i) * N + r.rx + j] = (int32_t)q;
}

// one Jacobi pass, thread per pixel
__global__ void dec_pass_kernel(const uint8_t *__restrict__ prev, const int32_t *__restrict__ owner,
                                const DecRec *__restrict__ par, int32_t N, uint8_t *__restrict__ out) {
    const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= (int64_t)N * N) return;
    const int32_t q = owner[p];
    if (q < 0) {
        out[p] = prev[p];
        return;
    }
    const DecRec r = par[q];
    const int y = (int)(p / N), x = (int)(p % N);
    const int i = y - r.ry, j = x - r.rx, b = r.B - 1;
    int si = i, sj = j;  // f_k(i, j), reading R2
    switch (r.iso) {
    case 1: si = b - j; sj = i; break;
    case 2: si = b - i; sj = b - j; break;
    case 3: si = j; sj = b - i; break;
    case 4: si = i; sj = b - j; break;
    case 5: si = j; sj = i; break;
    case 6: si = b - i; sj = j; break;
    case 7: si = b - j; sj = b - i; break;
    default: break;
    }
    const uint8_t *c = prev + (int64_t)(r.dy + 2 * si) * N + r.dx + 2 * sj;
    const int dp = (int)c[0] + (int)c[1] + (int)c[N] + (int)c[N + 1];
    double v = rint(__dadd_rn(__dmul_rn(r.s, (double)dp / 4.0), r.o));
    v = fmin(fmax(v, 0.0), 255.0);
    out[p] = (uint8_t)v;
}

__global__ void sse_kernel(const uint8_t *__restrict__ a, const uint8_t *__restrict__ b, int64_t n,
                           unsigned long long *__restrict__ sse) {
    unsigned long long acc = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int d = (int)a[i] - (int)b[i];
        acc += (unsigned long long)(d * d);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0 && acc) atomicAdd(sse, acc);
}

cudaError_t launch_decode(const fic_record *rec, int64_t n_rec, int32_t N, int32_t B_max, int32_t n_levels,
                          const DecSList &sl, int32_t iterations, const uint8_t *init, uint8_t *out,
                          void *scratch, int32_t *d_bad, cudaStream_t st) {
    const int64_t np = (int64_t)N * N;
    int32_t *owner = static_cast<int32_t *>(scratch);
    uint8_t *tmp = reinterpret_cast<uint8_t *>(owner + np);
    DecRec *par = reinterpret_cast<DecRec *>(tmp + ((np + 255) & ~(int64_t)255));
    cudaError_t e = cudaMemsetAsync(owner, 0xff, sizeof(int32_t) * np, st);
    if (e != cudaSuccess) return e;
    if (n_rec > 0) {
        dec_prep_kernel<<<(unsigned)((n_rec + 255) / 256), 256, 0, st>>>(rec, n_rec, N, B_max, n_levels, sl, par,
                                                                          owner, d_bad);
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
    }
    // passes alternate tmp <-> out so that the last one lands in out
    const uint8_t *src = init;
    if (!src) {
        e = cudaMemsetAsync(iterations % 2 ? tmp : out, 128, np, st);
        if (e != cudaSuccess) return e;
        src = iterations % 2 ? tmp : out;
    } else if (iterations == 0) {
        return cudaMemcpyAsync(out, init, np, cudaMemcpyDeviceToDevice, st);
    } else if (iterations % 2 == 0) {
        e = cudaMemcpyAsync(out, init, np, cudaMemcpyDeviceToDevice, st);  // keep the caller's init intact
        if (e != cudaSuccess) return e;
        src = out;
    }
    const unsigned g = (unsigned)((np + 255) / 256);
    for (int32_t it = 0; it < iterations; ++it) {
        uint8_t *dst = ((iterations - it) % 2 == 1) ? out : tmp;
        dec_pass_kernel<<<g, 256, 0, st>>>(src, owner, par, N, dst);
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
        src = dst;
    }
    return cudaSuccess;
}

size_t decode_scratch_bytes(int32_t N, int64_t n_rec) {
    const int64_t np = (int64_t)N * N;
    return sizeof(int32_t) * np + ((np + 255) & ~(int64_t)255) + sizeof(DecRec) * (size_t)(n_rec > 0 ? n_rec : 1);
}

cudaError_t launch_sse(const uint8_t *a, const uint8_t *b, int64_t n, unsigned long long *d_sse, cudaStream_t st) {
    cudaError_t e = cudaMemsetAsync(d_sse, 0, sizeof(unsigned long long), st);
    if (e != cudaSuccess || n == 0) return e;
    const int64_t blocks = std::min<int64_t>((n + 255) / 256, 148 * 8);
    sse_kernel<<<(unsigned)blocks, 256, 0, st>>>(a, b, n, d_sse);
    return cudaGetLastError();
}

}  // namespace fic
