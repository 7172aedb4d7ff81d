// Chip-wide peak rates for the pair-kernel roofline (SURVEY.md §8(d) "Roofline definition":
// P_int8, P_int32, P_fp64 measured on the box).  Every kernel runs on all SMs at full occupancy
// and is timed with CUDA events (best of 5 after a warm-up); the result is one JSON object on
// stdout (written to profiles/peaks_r02.json by scripts/measure_peaks.sh).
//
//   int8  : tcgen05.mma.cta_group::1.kind::i8, M = 128, N = 256, K = 32, operands in shared
//           memory (no swizzle), one issuing thread per CTA, one CTA per SM -> int8 ops/s
//           (2 per MAC)
//   int32 : IMAD (fma pipe), VIMNMX3 / IADD3 (alu pipe) and an IMAD + VIMNMX3 mix (both pipes)
//           -> lane-ops/s (one op per lane per instruction)
//   fp64  : DFMA, DADD, DMUL -> lane-ops/s
//
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o bin/peaks peaks.cu && bin/peaks
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

constexpr int CH = 8;        // independent chains per thread
constexpr int ITER = 8192;   // loop trips

template <int MODE>
__global__ void __launch_bounds__(512) int_kernel(int *out, int a, int b) {
    int x[CH];
#pragma unroll
    for (int i = 0; i < CH; ++i) x[i] = threadIdx.x * 7 + i * a;
#pragma unroll 4
    for (int it = 0; it < ITER; ++it) {
#pragma unroll
        for (int i = 0; i < CH; ++i) {
            if (MODE == 0) x[i] = x[i] * a + x[(i + 1) % CH];                                // IMAD
            if (MODE == 1) x[i] = __vimax3_s32(x[i], x[(i + 1) % CH] - 0, x[(i + 3) % CH]);  // VIMNMX3
            if (MODE == 2) x[i] = x[i] + x[(i + 1) % CH] + b;                                // IADD3
            if (MODE == 3) {                                                                 // IMAD + VIMNMX3
                if (i & 1) x[i] = __vimax3_s32(x[i], x[(i + 1) % CH], x[(i + 3) % CH]);
                else x[i] = x[i] * a + x[(i + 1) % CH];
            }
        }
    }
    int acc = 0;
#pragma unroll
    for (int i = 0; i < CH; ++i) acc ^= x[i];
    if (acc == 0x12345678) out[0] = acc;  // keep the chains live
}

template <int MODE>
__global__ void __launch_bounds__(512) fp64_kernel(double *out, double a, double b) {
    double x[CH];
#pragma unroll
    for (int i = 0; i < CH; ++i) x[i] = threadIdx.x * 1e-3 + i;
#pragma unroll 4
    for (int it = 0; it < ITER; ++it) {
#pragma unroll
        for (int i = 0; i < CH; ++i) {
            if (MODE == 0) x[i] = __fma_rn(x[i], a, x[(i + 1) % CH]);  // DFMA
            if (MODE == 1) x[i] = __dadd_rn(x[i], x[(i + 1) % CH]);    // DADD
            if (MODE == 2) x[i] = __dmul_rn(x[i], a);                  // DMUL
        }
    }
    double acc = 0;
#pragma unroll
    for (int i = 0; i < CH; ++i) acc += x[i];
    if (acc == b) out[0] = acc;
}

__device__ __forceinline__ unsigned su32(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
    d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
    d |= (uint64_t)1 << 46;
    return d;
}

template <int N>
__global__ void __launch_bounds__(128, 1) mma_kernel(int iters, int *out) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint32_t sT;
    __shared__ __align__(8) uint64_t bar;
    constexpr int KB = 128;
    uint8_t *A = sm, *Bm = sm + 128 * KB;
    for (int i = threadIdx.x; i < (128 + N) * KB; i += blockDim.x) sm[i] = (uint8_t)(i * 7);
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&sT)));
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
        for (int it = 0; it < iters; ++it) {
#pragma unroll
            for (int kk = 0; kk < KB / 32; ++kk) {
                const uint64_t ad = desc(su32(A) + kk * 256, 128, (KB / 16) * 128);
                const uint64_t bd = desc(su32(Bm) + kk * 256, 128, (KB / 16) * 128);
                const uint32_t acc = (it | kk) ? 1u : 0u;
                const uint32_t col = (it & 1) * N;  // two accumulators (512 columns)
                asm volatile("{ .reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p; }"
                             ::"r"(tm + col), "l"(ad), "l"(bd), "r"(idesc), "r"(acc) : "memory");
            }
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)) : "memory");
        unsigned done = 0;
        while (!done)
            asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0, 1, 0, p; }"
                         : "=r"(done) : "r"(su32(&bar)) : "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
    if (threadIdx.x == 0 && iters < 0) out[0] = 1;
}

template <class F>
static float best_ms(F launch) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    launch();
    cudaDeviceSynchronize();
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
        cudaEventRecord(e0);
        launch();
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    return best;
}

int main() {
    int dev = 0, sms = 0, clk_khz = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, dev);
    int *io;
    double *dout;
    cudaMalloc(&io, 64);
    cudaMalloc(&dout, 64);
    const int blocks = sms * 4, threads = 512;  // 2048 threads per SM
    const double lane_ops = (double)blocks * threads * ITER * CH;
    auto rate = [&](float ms) { return lane_ops / (ms * 1e-3); };
    const double imad = rate(best_ms([&] { int_kernel<0><<<blocks, threads>>>(io, 3, 5); }));
    const double vmnmx = rate(best_ms([&] { int_kernel<1><<<blocks, threads>>>(io, 3, 5); }));
    const double iadd3 = rate(best_ms([&] { int_kernel<2><<<blocks, threads>>>(io, 3, 5); }));
    const double mix = rate(best_ms([&] { int_kernel<3><<<blocks, threads>>>(io, 3, 5); }));
    const double dfma = rate(best_ms([&] { fp64_kernel<0><<<blocks, threads>>>(dout, 1.0000001, 0.5); }));
    const double dadd = rate(best_ms([&] { fp64_kernel<1><<<blocks, threads>>>(dout, 1.0000001, 0.5); }));
    const double dmul = rate(best_ms([&] { fp64_kernel<2><<<blocks, threads>>>(dout, 1.0000001, 0.5); }));
    constexpr int N = 256;
    const int smem = (128 + N) * 128;
    cudaFuncSetAttribute(mma_kernel<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int iters = 20000;
    const float mma_ms = best_ms([&] { mma_kernel<N><<<sms, 128, smem>>>(iters, io); });
    const double i8 = 2.0 * 128 * N * 32 * 4 * (double)iters * sms / (mma_ms * 1e-3);
    cudaError_t e = cudaDeviceSynchronize();
    printf("{\"sms\": %d, \"clock_attr_mhz\": %.0f, \"error\": \"%s\",\n", sms, clk_khz / 1e3, cudaGetErrorString(e));
    printf(" \"int32_lane_ops_per_s\": {\"imad\": %.4e, \"vimnmx3\": %.4e, \"iadd3\": %.4e, \"imad_vimnmx3_mix\": %.4e},\n",
           imad, vmnmx, iadd3, mix);
    printf(" \"fp64_lane_ops_per_s\": {\"dfma\": %.4e, \"dadd\": %.4e, \"dmul\": %.4e},\n", dfma, dadd, dmul);
    printf(" \"int8_tc_ops_per_s\": %.4e, \"int8_mma_ms\": %.3f}\n", i8, mma_ms);
    return e == cudaSuccess ? 0 : 1;
}
