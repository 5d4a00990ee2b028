// K5 fused: the whole CVAE warm-start decoder ((55+2) -> 1024 -> 1024 -> 1024 ->
// 1024 -> 256 -> dim, BatchNorm folded, ReLU between layers) in ONE persistent cooperative launch.
//
// Every layer is cut into 128-row x 64-column output tiles (128 tiles per 1024-wide layer at
// 1000 samples: one per SM).  CTA c takes tiles c, c + grid, ... of every layer in turn; a tile
// of layer l waits only for its 128-row block of layer l-1 (a per-(layer, row block) arrival
// counter in global memory), so row blocks flow through the layers without a grid-wide barrier.
//   layer 0            SIMT (K = 57): the observation part of each output is shared by all rows
//   hidden layers      tcgen05.mma kind::f16 (bf16 operands, fp32 accumulator in TMEM), operands
//                      TMA-staged through a 4-stage mbarrier ring (128-byte swizzle), bias + ReLU +
//                      bf16 epilogue from tcgen05.ld; activations go to L2-resident global buffers
//   last layer         fused into the last hidden layer's epilogue: each 64-column tile adds its
//                      partial dot products, the tile that completes a row block sums them in a
//                      fixed order (deterministic) and writes the fp64 outputs
// Activations cross CTAs through global memory: the producer's generic-proxy stores are fenced to
// the async proxy (fence.proxy.async.global) before the release, the consumer fences after its
// acquire and only then issues the TMA loads.
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>

#include "bd_common.cuh"
#include "cvae_tc.cuh"

namespace bd {

// A ring stage holds FZ_KG 64-wide K blocks, each operand loaded by ONE 3-D tensor copy
// ([K block][row][64]): the per-SM ingest of bulk copies grows with the bytes per copy (8 / 16 /
// 24 / >= 32 KB: 32 / 62 / 91 / ~120 GB/s, tools/probes/l2_ingest.cu), and the tiles are
// ingest-bound.  Kernel time at 1000 samples (ncu, warm L2): FZ_KG 1 (6 stages of 24 KB) 50.5 us,
// 2 (4 x 48 KB) 46.1 us, 4 (2 x 96 KB) 44.8 us
#ifndef FZ_KG_DEF
#define FZ_KG_DEF 4
#endif
constexpr int FZ_KG = FZ_KG_DEF;
constexpr int FZ_BM = 128, FZ_BN = 64, FZ_BK = 64, FZ_STAGES = FZ_KG == 1 ? 6 : (FZ_KG == 2 ? 4 : 2);
constexpr int FZ_MAXH = 6;                            // hidden tensor-core layers supported
constexpr int FZ_MAXOUT = 16;                         // last-layer outputs
constexpr int FZ_A_BYTES = FZ_KG * FZ_BM * FZ_BK * 2;         // 16 KB per K block
constexpr int FZ_B_BYTES = FZ_KG * FZ_BN * FZ_BK * 2;         // 8 KB per K block
constexpr int FZ_MAXZ = 16;                           // latent dimension
constexpr int FZ_SMEM = FZ_STAGES * (FZ_A_BYTES + FZ_B_BYTES) + 1024 /*align*/ + 256 /*barriers*/ +
                        FZ_MAXOUT * FZ_BN * 4 /*last-layer weight slice*/ + FZ_BM * FZ_MAXZ * 4 /*latent rows*/ +
                        FZ_BN * FZ_MAXZ * 4 /*layer-0 latent weights*/;

// kind::f16 instruction descriptor: fp32 accumulate, bf16 A/B, K-major both, N = 64, M = 128.
constexpr uint32_t FZ_IDESC = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(FZ_BN >> 3) << 17) |
                              ((uint32_t)(FZ_BM >> 4) << 24);

struct FusedMaps {
    CUtensorMap a[FZ_MAXH];   // activations entering hidden layer h (rows = count, box 128 x 64)
    CUtensorMap b[FZ_MAXH];   // bf16 weights of hidden layer h (rows = outputs, box 64 x 64)
};

struct FusedArgs {
    int count, nh, zdim;                    // nh = hidden tensor-core layers (Linear layers - 2)
    int dims[FZ_MAXH + 3];                  // dims[0] = 55 + zdim, ..., dims[nh + 2] = outputs
    const float* W0;                        // first layer fp32 [dims[1] x dims[0]]
    const float* bias[FZ_MAXH + 2];         // every layer's bias (fp32)
    const float* Wlast;                     // last layer fp32 [dims[nh+2] x dims[nh+1]]
    const float* obs;                       // 55
    const float* z;                         // count x zdim
    __nv_bfloat16* act[FZ_MAXH + 1];        // act[l]: output of Linear layer l (count x dims[l+1]), l <= nh
    float* partial;                         // [dims[nh+1] / 64][count][outputs]
    double* out;                            // count x outputs
    unsigned* ready;                        // [nh + 1][row blocks] arrival counters, never reset between
    unsigned epoch;                         // launches: launch e waits for e x (tiles per row block)
};

__device__ __forceinline__ void fence_proxy_async_global() {
    asm volatile("fence.proxy.async.global;" ::: "memory");
}

// 3-D box [FZ_KG K blocks][rows][64] at (K block kb, row y): FZ_KG consecutive 128-byte-swizzled
// K-major tiles in shared memory, the layout FZ_KG 2-D copies would produce
__device__ __forceinline__ void tma_load_3d_fz(void* dst, const CUtensorMap* map, int y, int kb, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
        ::"r"(smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(map)), "r"(0), "r"(y), "r"(kb), "r"(smem_u32(bar))
        : "memory");
}

// mbarrier wait that traps after ~2 s instead of spinning forever (a lost arrival must fail the
// launch, not hang the GPU)
__device__ __forceinline__ void mbar_wait_fz(uint64_t* bar, uint32_t parity) {
    const long long t0 = clock64();
    uint32_t ok = 0;
    while (true) {
        asm volatile(
            "{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(ok) : "r"(smem_u32(bar)), "r"(parity) : "memory");
        if (ok) return;
        if (clock64() - t0 > (4ll << 30)) __trap();
    }
}

__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

#ifndef FZ_POLL_NS
#define FZ_POLL_NS 16   // A/B (ncu warm, median): 64 ns 40.0 us, 16 ns 39.7 us, 0 ns 39.7 us
#endif
// Block until `need` tiles of a row block arrived (thread 0 polls; bounded, then gives up).
__device__ __forceinline__ void fz_wait(const unsigned* ctr, unsigned need) {
    if (threadIdx.x == 0) {
        long long spins = 0;
        while (ld_acquire_u32(ctr) < need && ++spins < (1ll << 27)) __nanosleep(FZ_POLL_NS);
        fence_proxy_async_global();
    }
    __syncthreads();
}

// Publish this CTA's tile: every thread fences its generic stores to the async proxy, then one
// release increment.  Returns the counter value before the increment (all threads).
// acquire: the caller reads other CTAs' data if it was the last to arrive (fence after the add).
__device__ __forceinline__ unsigned fz_arrive(unsigned* ctr, bool acquire = true) {
    __shared__ unsigned s_old;
    fence_proxy_async_global();
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        s_old = atomicAdd(ctr, 1u);
        if (acquire) __threadfence();
    }
    __syncthreads();
    return s_old;
}

__global__ void __launch_bounds__(128, 1) cvae_fused_kernel(const __grid_constant__ FusedMaps maps,
                                                           const FusedArgs a) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* smem =
        reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    unsigned char* tiles_a = smem;
    unsigned char* tiles_b = smem + FZ_STAGES * FZ_A_BYTES;
    uint64_t* full = reinterpret_cast<uint64_t*>(tiles_b + FZ_STAGES * FZ_B_BYTES);
    uint64_t* empty = full + FZ_STAGES;
    uint64_t* done = empty + FZ_STAGES;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 1);
    float* wl_s = reinterpret_cast<float*>(reinterpret_cast<unsigned char*>(full) + 256);   // [out][64]
    float* zs = wl_s + FZ_MAXOUT * FZ_BN;                                                  // [128][zdim]
    float* w0z = zs + FZ_BM * FZ_MAXZ;                                                     // [64][zdim]

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int count = a.count, mblocks = (count + FZ_BM - 1) / FZ_BM;
    const int nout = a.dims[a.nh + 2];

    if (threadIdx.x == 0) {
        for (int s = 0; s < FZ_STAGES; ++s) {
            mbar_init(full + s, 1);
            mbar_init(empty + s, 1);
        }
        mbar_init(done, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 2) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(FZ_BN));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = *tmem_slot;
#ifdef BD_PHASE_TIMING
    unsigned long long fzt[24];
    int nfz = 0;
    auto fzstamp = [&]() { unsigned long long t_; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t_)); if (nfz < 24) fzt[nfz++] = t_; };
    fzstamp();
#define FZ_STAMP() fzstamp()
#else
#define FZ_STAMP()
#endif

    // ---------------- layer 0 (SIMT): relu(W0 [obs; z] + b0) -> bf16
    {
        const int N = a.dims[1], K = a.dims[0], nb = N / FZ_BN;
        const int zd = a.zdim;
        for (int t = blockIdx.x; t < mblocks * nb; t += gridDim.x) {
            const int m = t / nb, n = t % nb;
            // every global load of the tile is issued before any is used (one L2 round trip): the
            // block's latent rows, the observation terms of its 64 outputs (two threads per output,
            // 28 / 27 terms each) and the latent weights
            const int cl = threadIdx.x & 63, half = threadIdx.x >> 6;
            const int c = n * FZ_BN + cl;
            const float* wr = a.W0 + (size_t)c * K;
            constexpr int OT = (CVAE_OBS + 1) / 2;
            float wv[OT], ov[OT];
#pragma unroll
            for (int j = 0; j < OT; ++j) {
                const int k = half + 2 * j;
                wv[j] = k < CVAE_OBS ? __ldg(wr + k) : 0.f;
                ov[j] = k < CVAE_OBS ? __ldg(a.obs + k) : 0.f;
            }
            for (int i = threadIdx.x; i < FZ_BM * zd; i += blockDim.x) {
                const int r = m * FZ_BM + i / zd;
                zs[i] = r < count ? a.z[(size_t)m * FZ_BM * zd + i] : 0.f;
            }
            for (int i = threadIdx.x; i < FZ_BN * zd; i += blockDim.x)
                w0z[i] = __ldg(a.W0 + (size_t)(n * FZ_BN + i / zd) * K + CVAE_OBS + i % zd);
            FZ_STAMP();
            float sp = 0.f;
#pragma unroll
            for (int j = 0; j < OT; ++j) sp = fmaf(wv[j], ov[j], sp);
            float* sps = zs + FZ_BM * FZ_MAXZ / 2;                        // [2][64] halves, then [64] sums
            sps[half * FZ_BN + cl] = sp;
            __syncthreads();
            if (threadIdx.x < FZ_BN) sps[2 * FZ_BN + cl] = a.bias[0][c] + (sps[cl] + sps[FZ_BN + cl]);
            __syncthreads();
            FZ_STAMP();
            // eight threads per row, each one 16-byte chunk (8 outputs) of the row's 128-byte
            // segment: a warp stores four whole segments per instruction (coalesced)
            const int q = threadIdx.x & 7;
            if (zd <= 2) {
                // the paper's latent size: this thread's 8 outputs' observation sums and latent
                // weights stay in registers across its rows (same arithmetic order as below)
                float bo[8], wa[8], wb[8];
#pragma unroll
                for (int e = 0; e < 8; ++e) {
                    const int cc = q * 8 + e;
                    bo[e] = sps[2 * FZ_BN + cc];
                    wa[e] = w0z[cc * zd];
                    wb[e] = zd > 1 ? w0z[cc * zd + 1] : 0.f;
                }
#pragma unroll 4
                for (int rl = threadIdx.x >> 3; rl < FZ_BM; rl += 128 / 8) {
                    const int r = m * FZ_BM + rl;
                    const float z0 = zs[rl * zd], z1 = zd > 1 ? zs[rl * zd + 1] : 0.f;
                    uint32_t pk[4];
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        float v2[2];
#pragma unroll
                        for (int e = 0; e < 2; ++e) {
                            float acc = fmaf(wa[2 * j + e], z0, bo[2 * j + e]);
                            if (zd > 1) acc = fmaf(wb[2 * j + e], z1, acc);
                            v2[e] = fmaxf(acc, 0.f);
                        }
                        const __nv_bfloat162 hv = __floats2bfloat162_rn(v2[0], v2[1]);
                        pk[j] = *reinterpret_cast<const uint32_t*>(&hv);
                    }
                    if (r < count)
                        reinterpret_cast<uint4*>(a.act[0] + (size_t)r * N + n * FZ_BN)[q] =
                            make_uint4(pk[0], pk[1], pk[2], pk[3]);
                }
            } else
#pragma unroll 2
            for (int rl = threadIdx.x >> 3; rl < FZ_BM; rl += 128 / 8) {
                const int r = m * FZ_BM + rl;
                float zr[FZ_MAXZ / 2];
#pragma unroll
                for (int k = 0; k < FZ_MAXZ / 2; ++k) zr[k] = k < zd ? zs[rl * zd + k] : 0.f;
                uint32_t pk[4];
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    float v2[2];
#pragma unroll
                    for (int e = 0; e < 2; ++e) {
                        const int cc = q * 8 + 2 * j + e;
                        float acc = sps[2 * FZ_BN + cc];
#pragma unroll
                        for (int k = 0; k < FZ_MAXZ / 2; ++k)
                            if (k < zd) acc = fmaf(w0z[cc * zd + k], zr[k], acc);
                        v2[e] = fmaxf(acc, 0.f);
                    }
                    const __nv_bfloat162 hv = __floats2bfloat162_rn(v2[0], v2[1]);
                    pk[j] = *reinterpret_cast<const uint32_t*>(&hv);
                }
                if (r < count)
                    reinterpret_cast<uint4*>(a.act[0] + (size_t)r * N + n * FZ_BN)[q] =
                        make_uint4(pk[0], pk[1], pk[2], pk[3]);
            }
            FZ_STAMP();
            fz_arrive(a.ready + m, false);
        }
    }
    FZ_STAMP();

    // ---------------- hidden layers on tcgen05
    uint32_t gk = 0, tiles = 0;                  // ring position / done-barrier parity, across tiles
    for (int h = 0; h < a.nh; ++h) {
        const int l = h + 1;                      // Linear layer index
        const int K = a.dims[l], N = a.dims[l + 1], nb = N / FZ_BN, kblocks = K / (FZ_BK * FZ_KG);
        const int nb_prev = a.dims[l] / FZ_BN;
        const bool last_hidden = (h == a.nh - 1);
        for (int t = blockIdx.x; t < mblocks * nb; t += gridDim.x) {
            const int m = t / nb, n = t % nb;
            if (last_hidden)        // this tile's slice of the last layer's weights
                for (int i = threadIdx.x; i < nout * FZ_BN; i += blockDim.x)
                    wl_s[i] = a.Wlast[(size_t)(i / FZ_BN) * N + n * FZ_BN + i % FZ_BN];
            fz_wait(a.ready + (size_t)(l - 1) * mblocks + m, a.epoch * (unsigned)nb_prev);
            FZ_STAMP();
            if (warp == 0 && lane == 0) {
                // ---- TMA producer
                for (int kb = 0; kb < kblocks; ++kb) {
                    const uint32_t g = gk + kb, s = g % FZ_STAGES;
                    if (g >= FZ_STAGES) mbar_wait_fz(empty + s, ((g / FZ_STAGES) + 1) & 1);
                    mbar_expect_tx(full + s, FZ_A_BYTES + FZ_B_BYTES);
                    tma_load_3d_fz(tiles_a + s * FZ_A_BYTES, &maps.a[h], m * FZ_BM, kb * FZ_KG, full + s);
                    tma_load_3d_fz(tiles_b + s * FZ_B_BYTES, &maps.b[h], n * FZ_BN, kb * FZ_KG, full + s);
                }
            } else if (warp == 1 && lane == 0) {
                // ---- MMA issuer: 4 x (128 x 64 x 16) per 64-wide K block, FZ_KG blocks per stage
                for (int kb = 0; kb < kblocks; ++kb) {
                    const uint32_t g = gk + kb, s = g % FZ_STAGES;
                    mbar_wait_fz(full + s, (g / FZ_STAGES) & 1);
                    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
                    for (int k = 0; k < FZ_KG * FZ_BK / 16; ++k) {
                        const int u = k / (FZ_BK / 16), kk = k % (FZ_BK / 16);   // K block of the stage, step in it
                        const uint64_t da =
                            umma_desc_sw128(smem_u32(tiles_a + s * FZ_A_BYTES + u * (FZ_A_BYTES / FZ_KG)));
                        const uint64_t db =
                            umma_desc_sw128(smem_u32(tiles_b + s * FZ_B_BYTES + u * (FZ_B_BYTES / FZ_KG)));
                        const uint32_t acc = (kb | k) != 0;
                        asm volatile(
                            "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                            "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
                            "l"(da + (uint64_t)(kk * 2)), "l"(db + (uint64_t)(kk * 2)), "r"(FZ_IDESC), "r"(acc));
                    }
                    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                                     smem_u32(empty + s))
                                 : "memory");
                }
                asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                                 smem_u32(done))
                             : "memory");
            }
            gk += kblocks;
            __syncwarp();
            mbar_wait_fz(done, tiles & 1);
            FZ_STAMP();
            ++tiles;
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            // ---- epilogue: TMEM -> bias + ReLU -> bf16 (warp w owns rows 32w..32w+31 of the tile)
            const int row = m * FZ_BM + warp * 32 + lane;
            const float* bias = a.bias[l] + n * FZ_BN;
            float pout[FZ_MAXOUT];
#pragma unroll
            for (int o = 0; o < FZ_MAXOUT; ++o) pout[o] = 0.f;
#pragma unroll
            for (int c0 = 0; c0 < FZ_BN; c0 += 32) {
                uint32_t r[32];
                const uint32_t taddr = tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)c0;
                asm volatile(
                    "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
                    "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                    : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                      "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
                      "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]),
                      "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]),
                      "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
                    : "r"(taddr));
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                uint32_t packed[16];
#pragma unroll
                for (int j = 0; j < 16; ++j) {
                    const float a0 = fmaxf(__uint_as_float(r[2 * j]) + bias[c0 + 2 * j], 0.f);
                    const float a1 = fmaxf(__uint_as_float(r[2 * j + 1]) + bias[c0 + 2 * j + 1], 0.f);
                    const __nv_bfloat162 hv = __floats2bfloat162_rn(a0, a1);
                    packed[j] = *reinterpret_cast<const uint32_t*>(&hv);
                    if (last_hidden) {
                        // last layer (fp32 weights on the bf16 activations): this tile's partial dots,
                        // weights from the staged slice (broadcast shared-memory loads)
                        const float h0 = __low2float(hv), h1 = __high2float(hv);
#pragma unroll
                        for (int o = 0; o < FZ_MAXOUT; ++o)
                            if (o < nout) {
                                const float2 wo = *reinterpret_cast<const float2*>(wl_s + o * FZ_BN + c0 + 2 * j);
                                pout[o] = fmaf(h1, wo.y, fmaf(h0, wo.x, pout[o]));
                            }
                    }
                }
                if (!last_hidden) {
                    // stage the row's 16-byte chunks in the (idle) ring, XOR-swizzled by row, so the
                    // warp can store whole 128-byte row segments below
                    uint4* st = reinterpret_cast<uint4*>(tiles_a) + (size_t)(warp * 32 + lane) * 8;
#pragma unroll
                    for (int q = 0; q < 4; ++q)
                        st[((c0 >> 3) + q) ^ (lane & 7)] =
                            make_uint4(packed[4 * q], packed[4 * q + 1], packed[4 * q + 2], packed[4 * q + 3]);
                }
            }
            if (!last_hidden) {
                // the warp's 32 rows x 128 bytes: lane l stores chunk l % 8 of row 4 i + l / 8
                __syncwarp();
                const uint4* st = reinterpret_cast<const uint4*>(tiles_a) + (size_t)warp * 32 * 8;
                const int ch = lane & 7;
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    const int rr = 4 * i + (lane >> 3), grow = m * FZ_BM + warp * 32 + rr;
                    if (grow < count)
                        reinterpret_cast<uint4*>(a.act[l] + (size_t)grow * N + n * FZ_BN)[ch] = st[rr * 8 + (ch ^ (rr & 7))];
                }
            }
            if (last_hidden && row < count)
#pragma unroll
                for (int o = 0; o < FZ_MAXOUT; ++o)
                    if (o < nout) a.partial[((size_t)n * count + row) * nout + o] = pout[o];
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            const unsigned prev = fz_arrive(a.ready + (size_t)l * mblocks + m, last_hidden);
            if (last_hidden && prev == a.epoch * (unsigned)nb - 1 && row < count) {
                // this tile completed the row block: sum the nb partials in column-block order + bias
                // (loads of all outputs first: one L2 round trip per column block, not per output)
                float acc[FZ_MAXOUT];
#pragma unroll
                for (int o = 0; o < FZ_MAXOUT; ++o) acc[o] = 0.f;
                for (int q = 0; q < nb; ++q) {
                    const float* pp = a.partial + ((size_t)q * count + row) * nout;
                    float pv[FZ_MAXOUT];
#pragma unroll
                    for (int o = 0; o < FZ_MAXOUT; ++o) pv[o] = o < nout ? __ldcg(pp + o) : 0.f;
#pragma unroll
                    for (int o = 0; o < FZ_MAXOUT; ++o) acc[o] += pv[o];
                }
                for (int o = 0; o < nout; ++o) a.out[(size_t)row * nout + o] = (double)(acc[o] + a.bias[a.nh + 1][o]);
            }
        }
    }
#ifdef BD_PHASE_TIMING
    FZ_STAMP();
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        printf("FZ cta %d:", blockIdx.x);
        for (int i = 1; i < nfz; ++i) printf(" %.2f", (fzt[i] - fzt[0]) * 1e-3);
        printf("\n");
    }
#endif
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 2) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(FZ_BN));
}

}  // namespace bd
