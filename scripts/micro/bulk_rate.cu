// Microbenchmark: cp.async.bulk (global -> shared, mbarrier completion) throughput per SM with
// S copies of C bytes in flight, all 148 SMs streaming a 32 MB (L2-resident) buffer.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o bin/bulk_rate bulk_rate.cu && bin/bulk_rate
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ unsigned su32(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }
// MT = 1: stage s is issued and waited by lane s (copies from different threads)
template <int MT>
__global__ void k(const unsigned char *src, size_t nbytes, int C, int S, int iters, long long *cyc) {
    extern __shared__ __align__(128) unsigned char sm[];
    __shared__ __align__(8) unsigned long long bar[16];
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[s])));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    if (MT ? threadIdx.x >= S : threadIdx.x != 0) return;
    const size_t nchunks = nbytes / C;
    size_t chunk = (size_t)blockIdx.x * 977 + (MT ? threadIdx.x * 148 : 0);
    long long t0 = clock64();
    for (int i = MT ? threadIdx.x : 0; i < iters + S; i += MT ? S : 1) {
        const int s = i % S;
        if (i >= S) {  // wait for the copy issued S iterations ago
            const unsigned par = ((i / S) - 1) & 1;
            unsigned done = 0;
            while (!done)
                asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                             : "=r"(done) : "r"(su32(&bar[s])), "r"(par) : "memory");
        }
        if (i < iters) {
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar[s])), "r"(C) : "memory");
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                         ::"r"(su32(sm + (size_t)s * C)), "l"(src + (chunk % nchunks) * C), "r"(C), "r"(su32(&bar[s])) : "memory");
            chunk += MT ? 148 * S : 148;
        }
    }
    long long t1 = clock64();
    if (blockIdx.x == 0 && threadIdx.x == 0) *cyc = t1 - t0;
}
int main() {
    const size_t nbytes = 32u << 20;
    unsigned char *src; long long *c, h;
    cudaMalloc(&src, nbytes); cudaMemset(src, 1, nbytes); cudaMalloc(&c, 8);
    cudaFuncSetAttribute(k<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(k<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    for (int mt : {0, 1})
    for (int C : {8192, 16384, 32768})
        for (int S : {1, 2, 4, 8}) {
            if ((size_t)C * S > 190 * 1024) continue;
            const int iters = 400;
            if (mt) { k<1><<<148, 32, C * S>>>(src, nbytes, C, S, iters, c); k<1><<<148, 32, C * S>>>(src, nbytes, C, S, iters, c); }
            else { k<0><<<148, 32, C * S>>>(src, nbytes, C, S, iters, c); k<0><<<148, 32, C * S>>>(src, nbytes, C, S, iters, c); }
            printf("mt %d ", mt);
            cudaError_t e = cudaDeviceSynchronize();
            cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
            printf("C %6d S %d: %6.1f B/clk/SM  (%.0f clk per copy, chip %.2f TB/s @1.965GHz) %s\n", C, S,
                   (double)C * iters / h, (double)h / iters * S, (double)C * iters / h * 148 * 1.965e9 / 1e12,
                   e ? cudaGetErrorString(e) : "");
        }
}
