// Dependent-chain latency of FFMA / DFMA / DDIV / DSQRT / DMUL on one warp (cycles per op).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* out, long long* cyc, double x0, float f0) {
    double x = x0 + threadIdx.x * 1e-9, y = 1.0000001;
    float f = f0 + threadIdx.x * 1e-6f, g = 1.0000001f;
    long long t0 = clock64();
    for (int i = 0; i < 1024; ++i) f = fmaf(f, g, 1e-7f);
    long long t1 = clock64();
    for (int i = 0; i < 1024; ++i) x = fma(x, y, 1e-9);
    long long t2 = clock64();
    for (int i = 0; i < 256; ++i) x = 1.0 / (x + 0.5);
    long long t3 = clock64();
    for (int i = 0; i < 256; ++i) x = sqrt(x + 0.25);
    long long t4 = clock64();
    for (int i = 0; i < 1024; ++i) x = x * y;
    long long t5 = clock64();
    for (int i = 0; i < 256; ++i) x = exp(-x);
    long long t6 = clock64();
    out[threadIdx.x] = x + f;
    if (threadIdx.x == 0) {
        cyc[0] = (t1 - t0) / 1024; cyc[1] = (t2 - t1) / 1024; cyc[2] = (t3 - t2) / 256; cyc[3] = (t4 - t3) / 256;
        cyc[4] = (t5 - t4) / 1024; cyc[5] = (t6 - t5) / 256;
    }
}
int main() {
    double* o; long long* c; cudaMalloc(&o, 256); cudaMallocManaged(&c, 64);
    k<<<1, 32>>>(o, c, 1.0, 1.0f); cudaDeviceSynchronize();
    k<<<1, 32>>>(o, c, 1.0, 1.0f); cudaDeviceSynchronize();
    printf("cycles/op: FFMA %lld DFMA %lld DDIV(+add) %lld DSQRT(+add) %lld DMUL %lld DEXP %lld\n", c[0], c[1], c[2], c[3], c[4], c[5]);
}
