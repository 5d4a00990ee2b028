// Per-SM L2 -> SM read bandwidth when G CTAs (one per SM) each stream `per` bytes of an
// L2-resident buffer with 1-D bulk copies (cp.async.bulk) into a shared-memory ring, the way the
// fused CVAE kernel's TMA producer does.  Prints GB/s per SM and aggregate for several G.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__global__ void __launch_bounds__(128, 1) ingest(const unsigned char* buf, size_t per, int chunk, int stages,
                                                 unsigned long long* cycles) {
    extern __shared__ __align__(128) unsigned char sm[];
    uint64_t* bar = reinterpret_cast<uint64_t*>(sm + (size_t)stages * chunk);
    const unsigned char* src = buf + (size_t)blockIdx.x * per;
    const int nper = (int)(per / chunk), n = nper * 10;   // the region 10 times (L2 hits)
    if (threadIdx.x == 0) {
        for (int s = 0; s < stages; ++s)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(bar + s)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned long long t0 = clock64();
        for (int i = 0; i < n + stages; ++i) {
            if (i >= stages) {   // wait for chunk i - stages
                const int s = (i - stages) % stages;
                const uint32_t ph = ((i - stages) / stages) & 1;
                asm volatile("{\n.reg .pred P;\nW: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n@!P bra W;\n}\n" ::"r"(su32(bar + s)), "r"(ph) : "memory");
            }
            if (i < n) {
                const int s = i % stages;
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(bar + s)), "r"(chunk) : "memory");
                asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su32(sm + (size_t)s * chunk)),
                             "l"(src + (size_t)(i % nper) * chunk), "r"(chunk), "r"(su32(bar + s)) : "memory");
            }
        }
        cycles[blockIdx.x] = clock64() - t0;
    }
}
int main() {
    const size_t per = 384 * 1024, total = 148 * per;
    unsigned char* buf; cudaMalloc(&buf, total); cudaMemset(buf, 1, total);
    unsigned long long* cyc; cudaMalloc(&cyc, 148 * 8);
    int clk = 0; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    for (int stg : {2, 4}) for (int ch : {24576, 32768, 49152}) for (int G : {128, 148}) {
        const int chunk = ch, stages = stg; const size_t smem = (size_t)stages * chunk + 128;
        cudaFuncSetAttribute(ingest, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        printf("chunk %d stages %d ", chunk, stages);
        for (int rep = 0; rep < 3; ++rep) ingest<<<G, 128, smem>>>(buf, per, chunk, stages, cyc);   // warm L2
        cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
        cudaEventRecord(a);
        for (int rep = 0; rep < 10; ++rep) ingest<<<G, 128, smem>>>(buf, per, chunk, stages, cyc);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        const double us = ms * 100.0;   // per launch
        printf("G=%3d: %.2f us per launch, %.1f GB/s per SM, %.2f TB/s aggregate\n", G, us, 10 * per / us * 1e-3,
               10.0 * G * per / us * 1e-6);
    }
    printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
