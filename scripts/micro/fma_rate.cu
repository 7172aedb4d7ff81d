// Microbenchmark: issue rate of FFMA / FFMA2 / FMUL2 / FMNMX3 forms on one SM (clock64 per op).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fma_rate fma_rate.cu && ./fma_rate
#include <cstdio>
#include <cuda_runtime.h>
constexpr int ITER = 4096, CH = 8;
template <int MODE>
__global__ void k(float *out, float sb, long long *cyc) {
    float2 a[CH];
    float s[CH];
    for (int i = 0; i < CH; ++i) { a[i] = make_float2(threadIdx.x * 1e-3f + i, i * 0.5f); s[i] = a[i].x; }
    const float2 b = make_float2(sb, sb * 0.5f), c = make_float2(0.25f, 0.125f);
    __syncthreads();
    long long t0 = clock64();
#pragma unroll 4
    for (int it = 0; it < ITER; ++it) {
#pragma unroll
        for (int i = 0; i < CH; ++i) {
            if (MODE == 0) s[i] = fmaf(s[i], sb, s[(i + 1) % CH]);                  // FFMA 3 regs
            if (MODE == 1) a[i] = __ffma2_rn(a[i], b, a[(i + 1) % CH]);               // FFMA2 3 pairs
            if (MODE == 2) a[i] = __ffma2_rn(a[i], make_float2(sb, sb), a[(i + 1) % CH]);  // FFMA2 scalar bcast
            if (MODE == 3) a[i] = __fmul2_rn(a[i], b);                                // FMUL2
            if (MODE == 4) s[i] = fminf(s[i], fminf(s[(i + 1) % CH], s[(i + 2) % CH]));  // FMNMX3
            if (MODE == 5) { a[i] = __ffma2_rn(a[i], b, a[(i + 1) % CH]); s[i] = fminf(s[i], fminf(a[i].x, s[(i + 2) % CH])); }
            if (MODE == 6) s[i] = fmaf(s[i], 1.0001f, 0.5f);                          // FFMA imm
        }
    }
    long long t1 = clock64();
    float acc = 0;
    for (int i = 0; i < CH; ++i) acc += a[i].x + a[i].y + s[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}
template <int MODE>
void run(const char *name, int warps) {
    float *o; long long *c, h;
    cudaMalloc(&o, 4 * 1024 * 148); cudaMalloc(&c, 8);
    k<MODE><<<1, 32 * warps>>>(o, 1.0001f, c);
    k<MODE><<<1, 32 * warps>>>(o, 1.0001f, c);
    cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    // per SMSP: warps/4 warps each issuing ITER*CH ops
    printf("%-22s warps/SM %2d: %.3f cycles per warp-op per SMSP\n", name, warps, (double)h / ((double)ITER * CH * warps / 4));
    cudaFree(o); cudaFree(c);
}
int main() {
    for (int w : {4, 8, 16}) {
        run<0>("FFMA 3reg", w); run<6>("FFMA imm", w); run<1>("FFMA2 3pair", w); run<2>("FFMA2 bcast", w);
        run<3>("FMUL2", w); run<4>("FMNMX3", w); run<5>("FFMA2+FMNMX3 (2 ops)", w);
    }
}
