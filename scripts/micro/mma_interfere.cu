// Microbenchmark: does a warp issuing tcgen05.mma slow the other warps of its SM sub-partition?
// 14 warps: warp 1 issues kind::f16 M128 N192 K16 MMAs (the B = 4 search tile) into two
// alternating TMEM accumulators with a commit + mbarrier wait per MMA (mode 1), or sleeps (mode 0);
// warps 2..13 (three per SMSP, like the epilogue) each run the same fixed ALU loop.  Prints each
// worker warp's cycles, grouped by SMSP (warp % 4).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o bin/mma_interfere mma_interfere.cu
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
constexpr int N = 192;
__global__ void __launch_bounds__(448, 1) k(long long *cyc, int iters, int mode, int work) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint32_t sT;
    __shared__ __align__(8) uint64_t bar;
    __shared__ volatile int stop;
    constexpr int KB = 32;
    uint8_t *A = sm, *B = sm + 128 * KB;
    for (int i = threadIdx.x; i < (128 + N) * KB; i += blockDim.x) sm[i] = (uint8_t)((i * 7) & 0x3F);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&sT)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (threadIdx.x == 0) {
        stop = 0;
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    asm volatile("fence.proxy.async.shared::cta;");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tm = sT;
    constexpr uint32_t idesc = (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    if (warp == 1) {
        if (mode >= 1 && lane == 0) {
            const uint32_t b = su32(&bar);
            uint32_t ph = 0;
            for (int it = 0; stop < 12; ++it) {
                if (mode == 4) { __nanosleep(work); continue; }
                const uint64_t ad = desc(su32(A), 128, (KB / 16) * 128);
                const uint64_t bd = desc(su32(B), 128, (KB / 16) * 128);
                asm volatile("tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, 0;"
                             ::"r"(tm + (it & 1) * 256), "l"(ad), "l"(bd), "r"(idesc) : "memory");
                if (mode <= 2) {
                    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(b) : "memory");
                    if (mode == 1) wait_bar(b, ph);
                    else {  // probe + sleep
                        unsigned done = 0;
                        for (;;) {
                            asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                                         : "=r"(done) : "r"(b), "r"(ph) : "memory");
                            if (done) break;
                            __nanosleep(32);
                        }
                    }
                    ph ^= 1u;
                }
                if (work > 0) __nanosleep(work);  // pacing (one MMA per ~tile)
            }
        }
    } else if (warp >= 2) {
        float a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3;
        const long long t0 = clock64();
        for (int i = 0; i < iters; ++i) {
            a0 = fmaf(a0, 1.0001f, 0.5f); a1 = fmaf(a1, 1.0001f, 0.5f);
            a2 = fmaf(a2, 1.0001f, 0.5f); a3 = fmaf(a3, 1.0001f, 0.5f);
            int x = __float_as_int(a0) ^ __float_as_int(a2);
            a1 += (float)(x & 7);
        }
        const long long t1 = clock64();
        if (lane == 0) { cyc[blockIdx.x * 16 + warp] = t1 - t0; atomicAdd((int *)&stop, 1); }
        if (lane == 0 && (a0 + a1 + a2 + a3) == 12345.f) cyc[0] = 0;
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
}
int main() {
    long long *c, h[148 * 16];
    cudaMalloc(&c, sizeof(h));
    const int smem = (128 + N) * 32;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    for (int rep = 0; rep < 2; ++rep)
        for (int mode = 0; mode < 5; ++mode)
            for (int pace : {0, 200, 400}) {
                if (mode >= 3 && pace == 0) continue;
                if (mode == 0 && pace) continue;
                k<<<148, 448, smem>>>(c, 200000, mode, pace);
                cudaError_t e = cudaDeviceSynchronize();
                cudaMemcpy(h, c, sizeof(h), cudaMemcpyDeviceToHost);
                double s[4] = {0, 0, 0, 0};
                int n[4] = {0, 0, 0, 0};
                for (int b = 0; b < 148; ++b)
                    for (int w = 2; w < 14; ++w) { s[w % 4] += (double)h[b * 16 + w]; n[w % 4]++; }
                if (rep == 1)
                    printf("mode %d (MMA warp on SMSP 1%s, pace %d ns): worker kcycles by SMSP 0..3: %.1f %.1f %.1f %.1f %s\n",
                           mode, mode == 0 ? " idle" : mode == 1 ? " MMA+commit+spin" : mode == 2 ? " MMA+commit+sleepwait" : mode == 3 ? " MMA only" : " sleep loop only", pace, s[0] / n[0] / 1e3, s[1] / n[1] / 1e3, s[2] / n[2] / 1e3,
                           s[3] / n[3] / 1e3, e ? cudaGetErrorString(e) : "");
            }
}
