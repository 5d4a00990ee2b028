#include <cstdio>
#include <cuda_runtime.h>
__global__ void mma_tf32(float* out, int iters) {
    unsigned a0 = __float_as_uint(1.0f + threadIdx.x), a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, b0 = a0 + 5, b1 = a0 + 7;
    float d[4][4] = {};
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int q = 0; q < 4; ++q)
            asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                         : "+f"(d[q][0]), "+f"(d[q][1]), "+f"(d[q][2]), "+f"(d[q][3]) : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
    }
    float s = 0; for (int q = 0; q < 4; ++q) s += d[q][0] + d[q][1] + d[q][2] + d[q][3];
    if (s == 1.2345f) out[0] = s;
}
__global__ void mixed(float* out, int iters) {   // mma + independent FFMA stream
    unsigned a0 = __float_as_uint(1.0f + threadIdx.x), a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, b0 = a0 + 5, b1 = a0 + 7;
    float d[4][4] = {};
    float f[8]; for (int k = 0; k < 8; ++k) f[k] = threadIdx.x + k;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int q = 0; q < 4; ++q)
            asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                         : "+f"(d[q][0]), "+f"(d[q][1]), "+f"(d[q][2]), "+f"(d[q][3]) : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
            for (int k = 0; k < 8; ++k) f[k] = fmaf(f[k], 0.999f, 0.001f);
    }
    float s = 0; for (int q = 0; q < 4; ++q) s += d[q][0] + d[q][1] + d[q][2] + d[q][3];
    for (int k = 0; k < 8; ++k) s += f[k];
    if (s == 1.2345f) out[0] = s;
}
int main() {
    float* o; cudaMalloc(&o, 4);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    int blocks = 148 * 8, th = 256, it = 4096;
    for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(e0); mma_tf32<<<blocks, th>>>(o, it); cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        double mmas = (double)blocks * (th / 32) * it * 4;
        printf("mma tf32: %.3f ms, %.3f T mma/s, %.1f TFLOP/s\n", ms, mmas / ms / 1e9, mmas * 16 * 8 * 8 * 2 / ms / 1e9);
        cudaEventRecord(e0); mixed<<<blocks, th>>>(o, it); cudaEventRecord(e1); cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        double ffma = (double)blocks * th * it * 32;
        printf("mixed: %.3f ms (ffma alone would take %.3f ms at 72 TF)\n", ms, ffma * 2 / 72e12 * 1e3);
    }
}
