// Microbenchmark: tcgen05.ld (TMEM -> registers) throughput on one SM, bytes per clock.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o bin/tmem_rate tmem_rate.cu && bin/tmem_rate
#include <cstdio>
#include <cuda_runtime.h>
constexpr int ITER = 2048;
__device__ __forceinline__ unsigned su32(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }
template <int X, int INFLIGHT>
__global__ void k(unsigned *out, long long *cyc) {
    __shared__ unsigned sT;
    const int warp = threadIdx.x >> 5;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&sT)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const unsigned tm = sT + ((unsigned)((warp & 3) * 32) << 16) + (unsigned)((warp >> 2) * X * INFLIGHT % 512);
    unsigned acc = 0;
    long long t0 = clock64();
    for (int it = 0; it < ITER; ++it) {
        unsigned v[128];
#pragma unroll
        for (int f = 0; f < INFLIGHT; ++f) {
            const unsigned a = tm + (unsigned)((f * X) % 512);
            if (X == 8)
                asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                             : "=r"(v[f*8+0]), "=r"(v[f*8+1]), "=r"(v[f*8+2]), "=r"(v[f*8+3]), "=r"(v[f*8+4]), "=r"(v[f*8+5]), "=r"(v[f*8+6]), "=r"(v[f*8+7]) : "r"(a));
            if (X == 32)
                asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                             : "=r"(v[f*32+0]), "=r"(v[f*32+1]), "=r"(v[f*32+2]), "=r"(v[f*32+3]), "=r"(v[f*32+4]), "=r"(v[f*32+5]), "=r"(v[f*32+6]), "=r"(v[f*32+7]),
                               "=r"(v[f*32+8]), "=r"(v[f*32+9]), "=r"(v[f*32+10]), "=r"(v[f*32+11]), "=r"(v[f*32+12]), "=r"(v[f*32+13]), "=r"(v[f*32+14]), "=r"(v[f*32+15]),
                               "=r"(v[f*32+16]), "=r"(v[f*32+17]), "=r"(v[f*32+18]), "=r"(v[f*32+19]), "=r"(v[f*32+20]), "=r"(v[f*32+21]), "=r"(v[f*32+22]), "=r"(v[f*32+23]),
                               "=r"(v[f*32+24]), "=r"(v[f*32+25]), "=r"(v[f*32+26]), "=r"(v[f*32+27]), "=r"(v[f*32+28]), "=r"(v[f*32+29]), "=r"(v[f*32+30]), "=r"(v[f*32+31]) : "r"(a));
        }
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int f = 0; f < INFLIGHT * X; ++f) acc ^= v[f];
    }
    long long t1 = clock64();
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(sT));
}
template <int X, int F>
void run(int warps) {
    unsigned *o; long long *c, h;
    cudaMalloc(&o, 4 * 1024 * 148); cudaMalloc(&c, 8);
    k<X, F><<<1, 32 * warps>>>(o, c);
    k<X, F><<<1, 32 * warps>>>(o, c);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    const double bytes = (double)ITER * warps * F * X * 32 * 4;
    printf("x%-3d inflight %d warps %2d: %.1f B/clk/SM  (%.2f clk per ld) %s\n", X, F, warps, bytes / h,
           (double)h / ((double)ITER * F * warps / 4), e ? cudaGetErrorString(e) : "");
    cudaFree(o); cudaFree(c);
}
int main() {
    for (int w : {4, 8, 16}) {
        run<8, 4>(w); run<32, 1>(w); run<32, 2>(w); run<32, 4>(w);
    }
}
