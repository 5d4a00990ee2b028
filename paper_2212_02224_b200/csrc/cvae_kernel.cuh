// K5: CVAE warm-start decoder MLP (paper PAPER.md:715-746; not in the reference package).
//
// (obs 55 + z) -> 1024 -> 1024 -> 1024 -> 1024 -> 256 -> dim with BatchNorm folded into
// each Linear and ReLU between layers.  The observation part of layer 1 is shared by all
// samples of a scene and computed once per output neuron.  Hidden layers use a
// register-tiled fp32 SIMT GEMM with the bias + ReLU epilogue fused (parity is unpinned:
// the reference ships no decoder; tests pin it against a float64 numpy restatement).
#pragma once

#include "bd_common.cuh"

namespace bd {

constexpr int CVAE_OBS = 55;          // observe() vector length (pkg/highway.py:18,208-246)
constexpr int CVAE_BM = 64;           // samples per CTA tile
constexpr int CVAE_BN = 64;           // output neurons per CTA tile
constexpr int CVAE_BK = 16;
constexpr int CVAE_THREADS = 256;     // 16 x 16 threads, 4 x 4 outputs each

__global__ void cvae_first_layer(int count, int n_out, int zdim, const float* __restrict__ W,
                                 const float* __restrict__ b, const float* __restrict__ obs,
                                 const float* __restrict__ z, float* __restrict__ out) {
    const int n = blockIdx.x * blockDim.x + threadIdx.x;
    if (n >= n_out) return;
    const int k_in = CVAE_OBS + zdim;
    const float* wr = W + (size_t)n * k_in;
    float shared_part = b[n];
    for (int k = 0; k < CVAE_OBS; ++k) shared_part = fmaf(wr[k], obs[k], shared_part);
    const int s0 = blockIdx.y * 32;
    for (int s = s0; s < s0 + 32 && s < count; ++s) {
        float acc = shared_part;
        for (int k = 0; k < zdim; ++k) acc = fmaf(wr[CVAE_OBS + k], z[(size_t)s * zdim + k], acc);
        out[(size_t)s * n_out + n] = fmaxf(acc, 0.f);
    }
}

// out[count x N] = act(in[count x K] W^T + b), W row-major [N x K].
__global__ void __launch_bounds__(CVAE_THREADS) cvae_linear(int count, int K, int N, const float* __restrict__ in,
                                                          const float* __restrict__ W, const float* __restrict__ b,
                                                          float* __restrict__ out, int relu) {
    __shared__ float As[CVAE_BK][CVAE_BM + 4];
    __shared__ float Bs[CVAE_BK][CVAE_BN + 4];
    const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
    const int m0 = blockIdx.y * CVAE_BM, n0 = blockIdx.x * CVAE_BN;
    float acc[4][4] = {};
    for (int k0 = 0; k0 < K; k0 += CVAE_BK) {
        for (int i = threadIdx.x; i < CVAE_BM * CVAE_BK; i += CVAE_THREADS) {
            const int r = i / CVAE_BK, c = i % CVAE_BK;
            const int gm = m0 + r, gk = k0 + c;
            As[c][r] = (gm < count && gk < K) ? in[(size_t)gm * K + gk] : 0.f;
            const int gn = n0 + r;
            Bs[c][r] = (gn < N && gk < K) ? W[(size_t)gn * K + gk] : 0.f;
        }
        __syncthreads();
#pragma unroll
        for (int kk = 0; kk < CVAE_BK; ++kk) {
            float a[4], w[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) { a[i] = As[kk][ty * 4 + i]; w[i] = Bs[kk][tx * 4 + i]; }
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], w[j], acc[i][j]);
        }
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int gm = m0 + ty * 4 + i;
        if (gm >= count) continue;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int gn = n0 + tx * 4 + j;
            if (gn >= N) continue;
            const float v = acc[i][j] + b[gn];
            out[(size_t)gm * N + gn] = relu ? fmaxf(v, 0.f) : v;
        }
    }
}

__global__ void cvae_to_double(const float* __restrict__ in, double* __restrict__ out, size_t n) {
    const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = (double)in[i];
}

}  // namespace bd
