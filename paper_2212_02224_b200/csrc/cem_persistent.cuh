// Single-scene CEM cycle as ONE persistent cooperative kernel (the config-2 latency shape).
//
// Replaces the per-iteration launch chain of bd_cem_cycle -- sample + stage 1, AM pass, replay
// guard, rank count, rank + refit -- for solve_bilevel's loop (pkg/bilevel.py:249-292) when the
// batch fills every SM with one CTA of 3-8 one-warp samples (B ~ 300-1200).  All CTAs are
// co-resident (cooperative launch), so the batch-global steps are grid barriers instead of kernel
// boundaries, and the serial work of each barrier is done by a dedicated control CTA:
//
//   per CEM iteration (worker CTAs: one CTA of 3-8 one-warp samples per SM, + the remainder warp at
//   3-8; one control CTA)
//     S   every warp: draw its set-point (p = mu + z L^T, pkg/bilevel.py:51-57) and solve its
//         stage-1 QP (pkg/batch_qp.py:209-280), constants staged in shared memory once per launch
//     A   every warp: the AM projection of its sample (am_samples, the latency instance of K2)
//     --- barrier; the control CTA scans the per-iteration batch maxima (early exit,
//         pkg/projection.py:329).  If an exit fired, every worker replays its samples for exactly
//         that many iterations and a second barrier follows.
//     R   every warp: the stable rank of its residual among the batch (np.argsort(kind="stable"),
//         pkg/bilevel.py:131) by counting over the keys staged in shared memory; scatter
//     --- barrier; the control CTA runs rank_refit_block: elites by augmented cost, weights,
//         mean / covariance refit, Cholesky factor, IterationStats, best record
//         (pkg/bilevel.py:129-194, 272-292)
//
// The arithmetic of every phase is the same device code as the multi-launch path, so the two
// paths give identical results (tests/test_gpu_cem.py compares them bit for bit).
#pragma once

#include "aux_kernels.cuh"
#include "am_kernel.cuh"
#include "cem_kernels.cuh"

namespace bd {

#ifdef BD_PHASE_TIMING   // diagnostic build: per-phase %globaltimer stamps printed by every worker CTA
__device__ __forceinline__ unsigned __smid() {
    unsigned r;
    asm volatile("mov.u32 %0, %smid;" : "=r"(r));
    return r;
}
__device__ __forceinline__ unsigned long long gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
#define BD_STAMP(k) if (threadIdx.x == 0) stamp[k] = gtime()
#else
#define BD_STAMP(k)
#endif

struct CemPersistArgs {
    AmArgs am;              // full pass (replay == nullptr); iters_used / replay_out / itmax per scene 0
    CemState cs;
    S1Args s1;
    const double* z;        // (it1 - it0) x B x dim caller normals, or nullptr (device Philox)
    const double* warm;     // B x dim warm-start rows for iteration 0, or nullptr
    uint64_t seed;
    int scene_offset, it0, it1, am_iters;
    double* params;         // B x dim set-points of the current iteration
    int* order;             // B   stable residual order
    unsigned* bar;          // 4 words: arrival count, generation, stop flag, replay flag (zero at launch)
    size_t s1_off, key_off; // dynamic shared-memory offsets of the stage-1 constants / rank keys
};

__device__ __forceinline__ unsigned ld_acquire_gpu(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_gpu(unsigned* p, unsigned v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Barrier words (p.bar): [0] arrivals of the worker CTAs, [1] generation released by the control
// CTA, [2] the control CTA's stop verdict (scene frozen after a failed iteration), [3] its
// early-exit verdict (replay, then rank again).  A worker reads the generation before arriving, so a release is never missed; every wait
// gives up after ~10 s (a CTA that never arrives) and flags ERR_P2P_TIMEOUT instead of hanging.
#ifndef BD_POLL_NS
#define BD_POLL_NS 32
#endif
#ifndef BD_CTL_POLL_NS
#define BD_CTL_POLL_NS 32
#endif
__device__ __forceinline__ void worker_arrive_wait(unsigned* bar, int* err) {
    __shared__ unsigned s_gen;
    __syncthreads();
    if (threadIdx.x == 0) {
        s_gen = ld_acquire_gpu(bar + 1);
        __threadfence();
        atomicAdd(bar, 1u);
        long long spins = 0;
        while (ld_acquire_gpu(bar + 1) == s_gen) {
            if (BD_POLL_NS) __nanosleep(BD_POLL_NS);
            if (++spins > (1ll << 28)) { atomicOr(err, ERR_P2P_TIMEOUT); break; }
        }
        __threadfence();
    }
    __syncthreads();       // thread 0's acquire + the CTA barrier publish the other CTAs' writes
}

// Control CTA: wait until every worker arrived, reset the count (the caller then does the serial
// step and calls control_release).
__device__ __forceinline__ void control_gather(unsigned* bar, int* err, unsigned workers) {
    __syncthreads();
    if (threadIdx.x == 0) {
        long long spins = 0;
        while (ld_acquire_gpu(bar) < workers) {
            if (BD_CTL_POLL_NS) __nanosleep(BD_CTL_POLL_NS);
            if (++spins > (1ll << 28)) { atomicOr(err, ERR_P2P_TIMEOUT); break; }
        }
        bar[0] = 0u;
        __threadfence();
    }
    __syncthreads();
}

__device__ __forceinline__ void control_release(unsigned* bar) {
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        st_release_gpu(bar + 1, ld_acquire_gpu(bar + 1) + 1u);
    }
}

// Grid = workers + 1.  Workers (one CTA of SPC one-warp samples per SM) run S, A and R; the last
// CTA is the control CTA: it never runs the AM loop, so the code of the serial steps (exit scan,
// elite ranking, refit, Cholesky) stays warm in its SM's instruction cache -- run by whichever
// worker arrived last, the refit took ~20 us, mostly instruction-fetch misses after the AM loop.
template <int TPB, int HELP>
__global__ void __launch_bounds__(TPB, 1) cem_persistent_kernel(const CemPersistArgs p) {
    // HELP > 0: the last warp of a worker CTA is the AM remainder warp (am_helper), no sample
    constexpr int P = 32, SPC = TPB / 32 - (HELP > 0 ? 1 : 0);
    extern __shared__ __align__(16) unsigned char smem[];
    const CemState& cs = p.cs;
    const S1Args& a1 = p.s1;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int B = cs.B, d = cs.dim;
    const unsigned workers = gridDim.x - 1;
    unsigned long long* keys = reinterpret_cast<unsigned long long*>(smem + p.key_off);

    // The error word is only read where no CTA can be writing it (S / A set its bits): at kernel
    // start, and by the control CTA after every worker has ranked; its verdict reaches the workers
    // as bar[2] together with the release.
    if (cs.err[0] != 0) return;                              // frozen by an earlier iteration range
    if (blockIdx.x == workers) {
        // ---------------- control CTA
        __shared__ int s_rep, s_stop;
        for (int it = p.it0; it < p.it1; ++it) {
            control_gather(p.bar, cs.err, workers);            // every worker finished its AM pass
            control_release(p.bar);                            // workers rank while the exit scan runs
            exit_scan_block(p.am.itmax, p.am.max_iters, p.am.tol, 0, p.am.iters_used, p.am.replay_out, nullptr);
            __syncthreads();
            if (threadIdx.x == 0) s_rep = p.am.replay_out[0];
            __syncthreads();
            control_gather(p.bar, cs.err, workers);            // every worker ranked its sample
            if (s_rep > 0) {
                // early exit: the ranking used the full pass; workers replay for the exit
                // iteration count and rank again (bar[3] carries the verdict with the release)
                if (threadIdx.x == 0) p.bar[3] = 1u;
                control_release(p.bar);
                control_gather(p.bar, cs.err, workers);        // replayed
                control_release(p.bar);
                control_gather(p.bar, cs.err, workers);        // ranked again
                if (threadIdx.x == 0) p.bar[3] = 0u;
            }
            rank_refit_block(cs, it, p.order, 0, reinterpret_cast<unsigned char*>(keys));
            __syncthreads();
            if (threadIdx.x == 0) {
                s_stop = cs.err[0] != 0;                        // failed iteration: the scene freezes
                p.bar[2] = (unsigned)s_stop;
            }
            control_release(p.bar);
            __syncthreads();
            if (s_stop) break;
        }
        return;
    }

    // ---------------- worker CTAs
    const int i = blockIdx.x * SPC + wid;                // this warp's sample
    const bool active = wid < SPC && i < B;
    // constants staged once per launch: AM (basis rows, obstacle tile, K blocks), stage 1
    __shared__ __align__(8) uint64_t stage_bar;
    am_stage<P, false>(p.am, 0, smem, &stage_bar);
    double* kinv = reinterpret_cast<double*>(smem + p.s1_off);
    double* kkt = kinv + a1.nr * s1_ld(a1.nr);
    double* qm = kkt + a1.nr * s1_ld(a1.nr);
    double* pw = qm + 2 * NC * a1.m_seg;                 // one behaviour vector per warp
    double* vw = pw + SPC * MAX_DIM;                     // per-warp stage-1 vectors
    stage1_load(a1, kinv, kkt, qm);
    __syncthreads();

#ifdef BD_PHASE_TIMING
    __shared__ unsigned long long stamp[8];
#endif
    for (int it = p.it0; it < p.it1; ++it) {
        BD_STAMP(0);
        // ---- S: set-point draw + stage 1 (sample_stage1_kernel's per-warp body)
        if (active) {
            double* pr = pw + wid * MAX_DIM;
            const double* warm = it == 0 ? p.warm : nullptr;
            if (warm != nullptr) {
                if (lane < d) pr[lane] = warm[(size_t)i * d + lane];
            } else {
                double zz[MAX_DIM];
                if (p.z != nullptr) {
                    const double* zi = p.z + ((size_t)(it - p.it0) * B + i) * d;
                    for (int q = 0; q < d; ++q) zz[q] = zi[q];
                } else {
                    philox_normals_warp(p.seed, p.scene_offset, it, i, zz, d, lane);
                }
                if (lane < d) {
                    double acc = 0.0;
                    for (int q = 0; q < d; ++q) acc = fma(zz[q], cs.L[lane * d + q], acc);
                    pr[lane] = cs.mean[lane] + acc;
                }
            }
            __syncwarp();
            if (lane < d) p.params[(size_t)i * d + lane] = pr[lane];
            stage1_body<true>(a1, i, pr, kinv, kkt, qm, vw + wid * S1_VEC);
        }
        __syncwarp();
        BD_STAMP(1);
        // ---- A: the AM projection of this CTA's samples
        am_samples<P, false, 100, 5, TPB, true, HELP>(p.am, 0, blockIdx.x, p.am_iters, smem);
        BD_STAMP(2);
        worker_arrive_wait(p.bar, cs.err);               // every worker's residuals are final
        BD_STAMP(3);
        // ---- R: stable residual rank of this warp's sample, scattered into the order (the control
        //      CTA scans for a batch-global early exit meanwhile)
        auto rank_phase = [&]() {
            for (int j = threadIdx.x; j < B; j += TPB) keys[j] = ordered_bits(cs.resid[j]);
            __syncthreads();
            if (active) {
                const unsigned long long ki = keys[i];
                int cnt = 0;
#pragma unroll 4
                for (int j = lane; j < B; j += 32) {
                    const unsigned long long kj = keys[j];
                    cnt += (int)(kj < ki) | ((int)(kj == ki) & (int)(j < i));
                }
                for (int o = 16; o >= 1; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
                BD_CHECK(cnt >= 0 && cnt < B);
                if (lane == 0) p.order[cnt] = i;
            }
        };
        rank_phase();
        worker_arrive_wait(p.bar, cs.err);               // control: exit verdict (or refit)
        if (ld_acquire_gpu(p.bar + 3) != 0u) {           // early exit: replay for exactly that many
            const int rep = p.am.replay_out[0];          // iterations, then rank the final batch
            AmArgs ar = p.am;
            ar.replay = p.am.replay_out;
            am_samples<P, false, 100, 5, TPB, true, HELP>(ar, 0, blockIdx.x, rep, smem);
            worker_arrive_wait(p.bar, cs.err);
            rank_phase();
            worker_arrive_wait(p.bar, cs.err);
        }
        BD_STAMP(4);
        BD_STAMP(7);
        if (ld_acquire_gpu(p.bar + 2) != 0u) break;      // the control CTA froze the scene
#ifdef BD_PHASE_TIMING
        if (threadIdx.x == 0)
            printf("PH it %d cta %d smid %d: S %.2f A %.2f bar1 %.2f R %.2f bar2 %.2f Aend %.2f\n", it, blockIdx.x,
                   __smid(), (stamp[1] - stamp[0]) * 1e-3, (stamp[2] - stamp[1]) * 1e-3, (stamp[3] - stamp[2]) * 1e-3,
                   (stamp[4] - stamp[3]) * 1e-3, (stamp[7] - stamp[4]) * 1e-3, (stamp[2] % 1000000000ull) * 1e-3);
#endif
    }
}

}  // namespace bd
