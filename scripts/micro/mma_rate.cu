// Microbenchmark: tcgen05.mma kind::i8 (M = 128, N, K = 32 per instruction, operands in smem)
// issue rate on one SM per CTA, SWIZZLE_NONE (8x16B core matrices) vs SWIZZLE_128B K-major.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o bin/mma_rate mma_rate.cu && bin/mma_rate
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ unsigned su32(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
    d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
    d |= (uint64_t)1 << 46;
    d |= (uint64_t)layout << 61;
    return d;
}
template <int N, int SW, int KBB>
__global__ void k(long long *cyc, int iters) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint32_t sT;
    __shared__ __align__(8) uint64_t bar;
    constexpr int KB = 128;  // K bytes resident per operand row
    uint8_t *A = sm, *B = sm + 128 * KB;  // B rows hold KBB bytes (the kernel's resident range operand)
    for (int i = threadIdx.x; i < 128 * KB + N * KBB; i += blockDim.x) sm[i] = (uint8_t)(i * 7);
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
    constexpr uint32_t idesc = (2u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    if (threadIdx.x == 0) {
        long long t0 = clock64();
        for (int it = 0; it < iters; ++it) {
#pragma unroll
            for (int kk = 0; kk < KB / 32; ++kk) {
                uint64_t ad, bd;
                if (SW == 0) {  // no swizzle: core matrices 8 rows x 16 B, K halves 128 B apart
                    const int ch = it % (KBB / KB);
                    ad = desc(su32(A) + kk * 256, 128, (KB / 16) * 128, 0);
                    bd = desc(su32(B) + ch * (KB / 16) * 128 + kk * 256, 128, (KBB / 16) * 128, 0);
                } else {        // 128B swizzle, K-major: 8-row atoms of 128 B rows (SBO 1024)
                    ad = desc(su32(A) + kk * 32, 16, 1024, 2);
                    bd = desc(su32(B) + kk * 32, 16, 1024, 2);
                }
                const uint32_t acc = (it | kk) ? 1u : 0u;
                asm volatile("{ .reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p; }"
                             ::"r"(tm), "l"(ad), "l"(bd), "r"(idesc), "r"(acc) : "memory");
            }
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)) : "memory");
        unsigned done = 0;
        while (!done)
            asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0, 1, 0, p; }"
                         : "=r"(done) : "r"(su32(&bar)) : "memory");
        long long t1 = clock64();
        if (blockIdx.x == 0) *cyc = t1 - t0;
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tm));
}
template <int N, int SW, int KBB = 128>
void run() {
    long long *c, h;
    cudaMalloc(&c, 8);
    const int smem = 128 * 128 + N * KBB;
    cudaFuncSetAttribute(k<N, SW, KBB>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int iters = 2000;
    k<N, SW, KBB><<<148, 128, smem>>>(c, iters);
    k<N, SW, KBB><<<148, 128, smem>>>(c, iters);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    const double macs = 128.0 * N * 32 * 4 * iters;
    printf("KBB %4d N %3d %s: %.1f cycles per MMA (K=32), %.0f int8 MAC/clk/SM %s\n", KBB, N, SW ? "SW128" : "none ",
           (double)h / (4.0 * iters), macs / h, e ? cudaGetErrorString(e) : "");
    cudaFree(c);
}
int main() {
    run<128, 0>(); run<128, 0, 1024>(); run<64, 0, 1024>();
}
