// K5 hidden layers on the 5th-generation tensor cores (sm_100a): bf16 x bf16 -> fp32 GEMM with
// tcgen05.mma (accumulator in TMEM), TMA (cp.async.bulk.tensor, 128B swizzle) operand staging
// through a 4-stage mbarrier pipeline, and a fused bias + ReLU epilogue read back with
// tcgen05.ld.  out[M x N] = act(in[M x K] W[N x K]^T + b), all row-major (K-major operands).
//
// Warp roles (128 threads): warp 0 lane 0 = TMA producer, warp 1 lane 0 = MMA issuer, warp 2 =
// TMEM allocator; after the K loop all four warps drain the 128 x 128 fp32 accumulator (warp w
// owns TMEM lanes 32w..32w+31 = output rows).
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>

#include "bd_common.cuh"

namespace bd {

constexpr int TC_BM = 128, TC_BN = 128, TC_BK = 64, TC_STAGES = 4;
constexpr int TC_TILE_BYTES = TC_BM * TC_BK * 2;   // 16 KB per operand tile (A and B alike: 128 rows)
constexpr int TC_SMEM = TC_STAGES * 2 * TC_TILE_BYTES + 1024 /*align*/ + 256 /*barriers*/;

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int x, int y, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
        ::"r"(smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(smem_u32(bar))
        : "memory");
}

// UMMA shared-memory descriptor, K-major tile with 128-byte swizzle: rows of 64 bf16 (128 B),
// 8-row swizzle atoms of 1024 B (SBO), version 1 (sm_100), layout type 2 = SWIZZLE_128B.
__device__ __forceinline__ uint64_t umma_desc_sw128(uint32_t smem_addr) {
    return (uint64_t)((smem_addr & 0x3FFFF) >> 4) | (1ull << 16) | (64ull << 32) | (1ull << 46) | (2ull << 61);
}

// kind::f16 instruction descriptor: fp32 accumulate, bf16 A/B, K-major both, N = 128, M = 128.
constexpr uint32_t TC_IDESC = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(TC_BN >> 3) << 17) |
                              ((uint32_t)(TC_BM >> 4) << 24);

__global__ void __launch_bounds__(128, 1) cvae_tc_linear(const __grid_constant__ CUtensorMap map_a,
                                                        const __grid_constant__ CUtensorMap map_b, int M, int N,
                                                        int K, const float* __restrict__ bias,
                                                        __nv_bfloat16* __restrict__ out, int relu) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    unsigned char* tiles_a = smem;
    unsigned char* tiles_b = smem + TC_STAGES * TC_TILE_BYTES;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + 2 * TC_STAGES * TC_TILE_BYTES);
    uint64_t* empty = full + TC_STAGES;
    uint64_t* done = empty + TC_STAGES;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 1);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int m0 = blockIdx.y * TC_BM, n0 = blockIdx.x * TC_BN;
    const int kblocks = (K + TC_BK - 1) / TC_BK;

    if (threadIdx.x == 0) {
        for (int s = 0; s < TC_STAGES; ++s) {
            mbar_init(full + s, 1);
            mbar_init(empty + s, 1);
        }
        mbar_init(done, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 2) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(TC_BN));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = *tmem_slot;

    if (warp == 0 && lane == 0) {
        // ---- TMA producer
        for (int kb = 0; kb < kblocks; ++kb) {
            const int s = kb % TC_STAGES;
            if (kb >= TC_STAGES) mbar_wait(empty + s, ((kb / TC_STAGES) + 1) & 1);
            mbar_expect_tx(full + s, 2 * TC_TILE_BYTES);
            tma_load_2d(tiles_a + s * TC_TILE_BYTES, &map_a, kb * TC_BK, m0, full + s);
            tma_load_2d(tiles_b + s * TC_TILE_BYTES, &map_b, kb * TC_BK, n0, full + s);
        }
    } else if (warp == 1 && lane == 0) {
        // ---- MMA issuer: 4 x (128x128x16) per 64-wide K block, accumulator in TMEM
        for (int kb = 0; kb < kblocks; ++kb) {
            const int s = kb % TC_STAGES;
            mbar_wait(full + s, (kb / TC_STAGES) & 1);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const uint64_t da = umma_desc_sw128(smem_u32(tiles_a + s * TC_TILE_BYTES));
            const uint64_t db = umma_desc_sw128(smem_u32(tiles_b + s * TC_TILE_BYTES));
#pragma unroll
            for (int k = 0; k < TC_BK / 16; ++k) {
                const uint32_t acc = (kb | k) != 0;
                asm volatile(
                    "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                    "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
                    "l"(da + (uint64_t)(k * 2)), "l"(db + (uint64_t)(k * 2)), "r"(TC_IDESC), "r"(acc));
            }
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                             smem_u32(empty + s))
                         : "memory");
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                         smem_u32(done))
                     : "memory");
    }
    __syncwarp();
    // ---- epilogue: TMEM -> registers -> bias + ReLU -> bf16 rows
    mbar_wait(done, 0);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const int row = m0 + warp * 32 + lane;
#pragma unroll 1
    for (int c0 = 0; c0 < TC_BN; c0 += 32) {
        uint32_t r[32];
        const uint32_t taddr = tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)c0;
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
            "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
            : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
              "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
              "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]),
              "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]),
              "=r"(r[30]), "=r"(r[31])
            : "r"(taddr));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        if (row < M && n0 + c0 < N) {
            uint32_t packed[16];
#pragma unroll
            for (int j = 0; j < 16; ++j) {
                float a0 = __uint_as_float(r[2 * j]) + bias[n0 + c0 + 2 * j];
                float a1 = __uint_as_float(r[2 * j + 1]) + bias[n0 + c0 + 2 * j + 1];
                if (relu) { a0 = fmaxf(a0, 0.f); a1 = fmaxf(a1, 0.f); }
                const __nv_bfloat162 h = __floats2bfloat162_rn(a0, a1);
                packed[j] = *reinterpret_cast<const uint32_t*>(&h);
            }
            uint4* dst = reinterpret_cast<uint4*>(out + (size_t)row * N + n0 + c0);
#pragma unroll
            for (int q = 0; q < 4; ++q)
                dst[q] = make_uint4(packed[4 * q], packed[4 * q + 1], packed[4 * q + 2], packed[4 * q + 3]);
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 2)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TC_BN));
}

// First layer (obs part shared by the scene) and last layer (256 -> dim) stay SIMT: K = 57 and N = 8
// are below the tensor-core tile.  bf16 activations in/out.
__global__ void cvae_first_layer_bf16(int count, int n_out, int zdim, const float* __restrict__ W,
                                      const float* __restrict__ b, const float* __restrict__ obs,
                                      const float* __restrict__ z, __nv_bfloat16* __restrict__ out) {
    const int n = blockIdx.x * blockDim.x + threadIdx.x;
    if (n >= n_out) return;
    const int k_in = 55 + zdim;
    const float* wr = W + (size_t)n * k_in;
    float shared_part = b[n];
    for (int k = 0; k < 55; ++k) shared_part = fmaf(wr[k], obs[k], shared_part);
    const int s0 = blockIdx.y * 32;
    for (int s = s0; s < s0 + 32 && s < count; ++s) {
        float acc = shared_part;
        for (int k = 0; k < zdim; ++k) acc = fmaf(wr[55 + k], z[(size_t)s * zdim + k], acc);
        out[(size_t)s * n_out + n] = __float2bfloat16_rn(fmaxf(acc, 0.f));
    }
}

__global__ void cvae_last_layer_bf16(int count, int K, int N, const __nv_bfloat16* __restrict__ in,
                                     const float* __restrict__ W, const float* __restrict__ b, double* out) {
    // one warp per sample: lanes stride over K, shuffle-reduce per output
    const int s = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (s >= count) return;
    for (int n = 0; n < N; ++n) {
        float acc = 0.f;
        for (int k = lane; k < K; k += 32) acc = fmaf(__bfloat162float(in[(size_t)s * K + k]), W[(size_t)n * K + k], acc);
        for (int o = 16; o >= 1; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (lane == 0) out[(size_t)s * N + n] = (double)(acc + b[n]);
    }
}

}  // namespace bd
