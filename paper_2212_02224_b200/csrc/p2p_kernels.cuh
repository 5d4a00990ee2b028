// Sharded-batch exchange over NVLink peer memory, sm_100a.
//
// Every rank owns one symmetric buffer (torch symmetric memory: the same layout on every GPU,
// peer-mapped) holding the gathered residuals and costs of the whole batch, each rank's
// per-iteration residual maxima and one coefficient row per rank, plus a signal pad of uint32
// epoch slots.  The AM kernel's epilogue stores each sample's (residual, cost) into every rank's
// buffer directly (the all-gather fused into the compute); the small kernels below publish the
// iteration maxima / the best row and signal with system-scope release stores, and wait on the
// local pad with acquire loads.  Epochs only grow, so no slot is ever reset.
#pragma once

#include "bd_common.cuh"

namespace bd {

struct P2PArgs {
    int world, rank, iters_cap;
    void* const* bufs;          // world symmetric buffers
    unsigned* const* sigs;      // world signal pads
    size_t res_off, cost_off, itmax_off, xi_off;
    int* err;                   // local error word (ERR_P2P_TIMEOUT)
};

__device__ __forceinline__ void st_release_sys(unsigned* p, unsigned v) {
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned ld_acquire_sys(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
template <class T>
__device__ __forceinline__ T* at(void* base, size_t off) { return reinterpret_cast<T*>(static_cast<char*>(base) + off); }

// Copy this rank's iteration maxima into every rank's table (optional), then signal `slot`.
__global__ void p2p_publish_kernel(const P2PArgs p, const float* itmax_local, int iters, unsigned epoch, int slot) {
    if (itmax_local)
        for (int g = 0; g < p.world; ++g)
            for (int i = threadIdx.x; i < iters; i += blockDim.x)
                at<float>(p.bufs[g], p.itmax_off)[p.rank * p.iters_cap + i] = itmax_local[i];
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence_system();       // this kernel's and (stream-ordered) earlier kernels' peer stores
        for (int g = 0; g < p.world; ++g) st_release_sys(p.sigs[g] + slot * p.world + p.rank, epoch);
    }
}

// Wait until every rank has signalled `slot` with `epoch` (bounded: ~10 s, then ERR_P2P_TIMEOUT).
__global__ void p2p_wait_kernel(const P2PArgs p, unsigned epoch, int slot) {
    for (int g = threadIdx.x; g < p.world; g += blockDim.x) {
        const unsigned* s = p.sigs[p.rank] + slot * p.world + g;
        long long spins = 0;
        while (ld_acquire_sys(s) < epoch) {
            __nanosleep(200);
            if (++spins > (1ll << 25)) { atomicOr(p.err, ERR_P2P_TIMEOUT); break; }
        }
    }
    __syncthreads();
}

// Batch-global exit (pkg/projection.py:329) from all ranks' maxima: used = first k with the
// max over ranks <= tol (else iters); replay = used if it is < iters, else 0.
__global__ void p2p_exit_kernel(const P2PArgs p, int iters, double tol, int* replay, int* used) {
    __shared__ int first;
    if (threadIdx.x == 0) first = iters;
    __syncthreads();
    const float* tab = at<float>(p.bufs[p.rank], p.itmax_off);
    for (int i = threadIdx.x; i < iters; i += blockDim.x) {
        float mx = 0.f;
        for (int g = 0; g < p.world; ++g) mx = fmaxf(mx, __ldcg(tab + g * p.iters_cap + i));
        if (static_cast<double>(mx) <= tol) atomicMin(&first, i + 1);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        *replay = first < iters ? first : 0;
        if (used) *used = first;
    }
}

// Best elite row to every rank: the owner of global row j stores its coefficients, the others
// zeros, into slot `rank` of every rank's row table; then signal.
__global__ void p2p_share_row_kernel(const P2PArgs p, const long long* best, long long row0, int b_shard,
                                     const double* xi_shard, unsigned epoch, int slot) {
    const long long j = *best;
    const bool mine = j >= row0 && j < row0 + b_shard;
    for (int g = 0; g < p.world; ++g)
        for (int k = threadIdx.x; k < NX; k += blockDim.x)
            at<double>(p.bufs[g], p.xi_off)[p.rank * NX + k] = mine ? xi_shard[(j - row0) * NX + k] : 0.0;
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence_system();
        for (int g = 0; g < p.world; ++g) st_release_sys(p.sigs[g] + slot * p.world + p.rank, epoch);
    }
}

__global__ void p2p_sum_rows_kernel(const P2PArgs p, double* out) {
    const double* tab = at<double>(p.bufs[p.rank], p.xi_off);
    for (int k = threadIdx.x; k < NX; k += blockDim.x) {
        double s = 0.0;
        for (int g = 0; g < p.world; ++g) s += __ldcg(tab + g * NX + k);   // one non-zero row: exact
        out[k] = s;
    }
}

}  // namespace bd
