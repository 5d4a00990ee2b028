// Shared definitions for the sm_100a kernels of the bi-level planner hot path.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <cfloat>
#include <cstdio>

// Device-side bounds / invariant checks (build with -DBD_CHECKS=1; tools/build_variant.sh checks
// "-DBD_CHECKS=1").  Off in the product build.
#ifndef BD_CHECKS
#define BD_CHECKS 0
#endif
#define BD_CHECK(cond)                                                                     \
    do {                                                                                   \
        if (BD_CHECKS && !(cond)) {                                                        \
            printf("BD_CHECK failed %s:%d: %s\n", __FILE__, __LINE__, #cond);             \
            __trap();                                                                      \
        }                                                                                  \
    } while (0)

namespace bd {

constexpr int NC = 11;             // coefficients per axis: Bernstein order 10 (pkg/basis.py:156-179)
constexpr int NX = 2 * NC;         // stacked xi = (c_x, c_y)
constexpr int WROW = 36;           // one timestep of [W | Wd | Wdd] in fp32, padded to 9 x float4
constexpr int KROW = 12;           // fp64 row stride of the per-axis u vectors in the AM scratch (6 x double2)
constexpr int KSTR = 14;           // fp64 row stride of the aug-KKT inverse rows in shared memory: rows are
                                   // stored by value index (2 kk + axis), the 8 consecutive rows a lane
                                   // group reads sit 7 x 16 B apart -> conflict-free LDS.128
constexpr int MAX_NEQ = 9;         // 6 initial-state rows (+3 goal rows), pkg/batch_qp.py:181-193
constexpr int MAX_DIM = 16;        // behaviour vector length (2*m_seg [+2])
constexpr int ITMAX_SLOTS = 32;    // spread slots for the per-iteration batch max (early exit)

// Error bits of the device error word.
constexpr int ERR_NONFINITE = 1;   // NumericalFailure: non-finite iterate (pkg/projection.py:290-291)
constexpr int ERR_KKT_RESID = 2;   // NumericalFailure: stage-1 KKT residual (pkg/batch_qp.py:272-279)
constexpr int ERR_BAD_RHS = 4;     // ValueError: non-finite right-hand side (pkg/batch_qp.py:105-106)
constexpr int ERR_P2P_TIMEOUT = 16; // RuntimeError: a peer never signalled (sharded exchange)

// Per-scene scalars in the form the AM kernel consumes (ConstraintSpec, pkg/constraints.py:31-42).
struct SceneLim {
    float a, b, inv_a, inv_b;
    float v_min, v_max, a_max, k_max, inv_k_max, c_max, y_lb, y_ub;
};

__device__ __forceinline__ unsigned float_key(float r) {
    // residuals are >= 0 (sums of max(0, .)), so their IEEE bits order like the values; NaN sorts last.
    return __float_as_uint(r);
}

__host__ __device__ __forceinline__ size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

// Packed fp32x2 arithmetic (sm_100a FFMA2 / FADD2 / FMUL2): one issue slot for two lanes of
// work; a scalar first operand is broadcast by the hardware operand selector (no extra moves).
__device__ __forceinline__ unsigned long long f2u(float2 v) { return *reinterpret_cast<unsigned long long*>(&v); }
__device__ __forceinline__ float2 u2f(unsigned long long v) { return *reinterpret_cast<float2*>(&v); }
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
    unsigned long long r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(f2u(a)), "l"(f2u(b)), "l"(f2u(c)));
    return u2f(r);
}
__device__ __forceinline__ float2 ffma2(float a, float2 b, float2 c) { return ffma2(make_float2(a, a), b, c); }
__device__ __forceinline__ float2 fadd2(float2 a, float2 b) {
    unsigned long long r;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(f2u(a)), "l"(f2u(b)));
    return u2f(r);
}
__device__ __forceinline__ float2 fmul2(float2 a, float2 b) {
    unsigned long long r;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(f2u(a)), "l"(f2u(b)));
    return u2f(r);
}

// ---- mbarrier + bulk-copy (TMA) helpers shared by the kernels
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

// 1-D TMA bulk copy global -> shared (bytes and both addresses multiples of 16), completing on bar.
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

}  // namespace bd
