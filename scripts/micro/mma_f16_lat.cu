// Microbenchmark: tcgen05.mma kind::f16 (M = 128, K = 16 per instruction, fp32 accumulator,
// SWIZZLE_NONE core matrices, the search kernel's B = 4 / 8 form) on one CTA per SM:
//   rate:    back-to-back MMAs, one commit at the end      -> cycles per MMA (throughput)
//   latency: one MMA, commit, wait on the mbarrier, repeat -> cycles from issue to observed completion
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o bin/mma_f16_lat mma_f16_lat.cu && bin/mma_f16_lat
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ unsigned su32(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
    d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
    d |= (uint64_t)1 << 46;
    return d;
}
__device__ __forceinline__ void wait_bar(uint32_t bar, uint32_t ph) {
    unsigned done = 0;
    while (!done)
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                     : "=r"(done) : "r"(bar), "r"(ph) : "memory");
}
template <int N, int KS>
__global__ void k(long long *cyc, int iters, int mode) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint32_t sT;
    __shared__ __align__(8) uint64_t bar;
    constexpr int KB = 32 * KS;  // K bytes per row (KS instructions of K = 16 fp16)
    uint8_t *A = sm, *B = sm + 128 * KB;
    for (int i = threadIdx.x; i < (128 + N) * KB; i += blockDim.x) sm[i] = (uint8_t)((i * 7) & 0x3F);
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(su32(&sT)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    asm volatile("fence.proxy.async.shared::cta;");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tm = sT;
    constexpr uint32_t idesc = (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    if (threadIdx.x == 0) {
        const uint32_t b = su32(&bar);
        uint32_t ph = 0;
        long long t0 = clock64();
        for (int it = 0; it < iters; ++it) {
#pragma unroll
            for (int kk = 0; kk < KS; ++kk) {
                const uint64_t ad = desc(su32(A) + kk * 256, 128, (KB / 16) * 128);
                const uint64_t bd = desc(su32(B) + kk * 256, 128, (KB / 16) * 128);
                const uint32_t acc = kk ? 1u : 0u;
                asm volatile("{ .reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p; }"
                             ::"r"(tm), "l"(ad), "l"(bd), "r"(idesc), "r"(acc) : "memory");
            }
            if (mode == 1) {
                asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(b) : "memory");
                wait_bar(b, ph);
                ph ^= 1u;
            }
        }
        if (mode == 0) {
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(b) : "memory");
            wait_bar(b, ph);
        }
        long long t1 = clock64();
        if (blockIdx.x == 0) *cyc = t1 - t0;
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tm));
}
template <int N, int KS>
void run() {
    long long *c, h[2];
    cudaMalloc(&c, 8);
    const int smem = (128 + N) * 32 * KS;
    cudaFuncSetAttribute(k<N, KS>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int iters = 2000;
    for (int mode = 0; mode < 2; ++mode) {
        k<N, KS><<<148, 128, smem>>>(c, iters, mode);
        k<N, KS><<<148, 128, smem>>>(c, iters, mode);
        cudaDeviceSynchronize();
        cudaMemcpy(&h[mode], c, 8, cudaMemcpyDeviceToHost);
    }
    const double macs = 128.0 * N * 16 * KS;
    printf("f16 M128 N%3d K%3d (%d instr): rate %.1f cycles/tile (%.0f MAC/clk/SM), issue->observed latency %.1f cycles %s\n",
           N, 16 * KS, KS, (double)h[0] / iters, macs * iters / h[0], (double)h[1] / iters,
           cudaGetErrorString(cudaGetLastError()));
    cudaFree(c);
}
int main() {
    run<64, 1>(); run<128, 1>(); run<192, 1>(); run<256, 1>();
    run<64, 2>(); run<256, 2>(); run<256, 4>();
}
