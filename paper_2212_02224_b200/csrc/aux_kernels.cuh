// K1 stage-1 batch QP, trajectory evaluation and the fp64 residual evaluator (sm_100a).
#pragma once

#include "bd_common.cuh"

namespace bd {

// ---------------------------------------------------------------- K1: stage-1 QP
// build_rhs_batch + solve_batch (pkg/batch_qp.py:209-280): one warp per sample,
// lane i owns KKT row i.  sol = KKT^{-1} [-q; b] with the host-factorised inverse,
// then the reference's residual check |KKT sol - rhs|_inf <= 1e-8 (1 + |rhs|_inf).
struct S1Args {
    int total, B, dim, neq, m_seg, with_goal, nr, nvar;
    const double* rhs_in;   // generic mode: total x nr right-hand sides (params unused)
    double* sol_out;        // generic mode: total x nr solutions
    const double* qmx;      // NC x m_seg
    const double* qmy;      // NC x m_seg
    const double* kkt;      // nr x nr
    const double* kinv;     // nr x nr
    const double* params;   // total x dim
    const double* bscene;   // S x neq
    double* xi_bar;         // total x NX  (nullable)
    double* mu;             // total x neq (nullable)
    double* b_out;          // total x neq (nullable)
    int* err;
};

// Shared-memory row stride of the staged KKT blocks (doubles): even, so rows are 16-byte aligned
// for double2 loads, and an odd number of 16-byte units, so the lanes of a warp -- each reading
// its own row at the same column -- hit distinct banks (an unpadded stride of 28 makes 8 lanes
// collide on every load).
__host__ __device__ __forceinline__ int s1_ld(int nr) {
    const int ld = (nr + 1) & ~1;
    return (ld / 2) % 2 ? ld : ld + 2;
}
// per-warp staging of the right-hand side / solution vector (broadcast reads in the mat-vecs)
constexpr int S1_VEC = 32;

__device__ __forceinline__ void stage1_load(const S1Args& a, double* kinv, double* kkt, double* qm) {
    // a warp per row, a lane per column (no index division; coalesced row reads)
    const int ld = s1_ld(a.nr), lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    for (int r = threadIdx.x >> 5; r < a.nr; r += nw)
        for (int c = lane; c < ld; c += 32) {
            kinv[r * ld + c] = c < a.nr ? a.kinv[r * a.nr + c] : 0.0;
            kkt[r * ld + c] = c < a.nr ? a.kkt[r * a.nr + c] : 0.0;
        }
    if (!a.rhs_in)
        for (int i = threadIdx.x; i < NC * a.m_seg; i += blockDim.x) { qm[i] = a.qmx[i]; qm[NC * a.m_seg + i] = a.qmy[i]; }
}

// One sample per warp; pr points at its behaviour vector (global or shared memory).
// Row i of M (staged with stride ld) times the warp's vector v, summed in column order.
__device__ __forceinline__ double s1_rowdot(const double* M, const double* v, int i, int nr, int ld) {
    const double2* m2 = reinterpret_cast<const double2*>(M + (size_t)i * ld);
    const double2* v2 = reinterpret_cast<const double2*>(v);
    double s = 0.0;
    int j = 0;
    for (; j + 1 < nr; j += 2) {
        const double2 m = m2[j >> 1], x = v2[j >> 1];
        s = fma(m.x, x.x, s);
        s = fma(m.y, x.y, s);
    }
    if (j < nr) s = fma(M[(size_t)i * ld + j], v[j], s);
    return s;
}

// DEF: the default layout (28 KKT rows = 22 coefficients + 6 equalities, 4 segments, no goal rows,
// behaviour vector of 8) as compile-time constants, so the row loops unroll without bounds checks.
constexpr int S1_DEF_NR = NX + 6, S1_DEF_MS = 4, S1_DEF_DIM = 8;
template <bool DEF = false>
__device__ __forceinline__ void stage1_body(const S1Args& a, int row, const double* pr, const double* kinv,
                                            const double* kkt, const double* qm, double* vec) {
    const int lane = threadIdx.x & 31;
    const int i = lane;
    const int nr = DEF ? S1_DEF_NR : a.nr;
    double rhs = 0.0;
    if (!DEF && a.rhs_in) {
        if (i < nr) rhs = a.rhs_in[(size_t)row * nr + i];
    } else {
    const int scene = row / a.B;
    const int ms = DEF ? S1_DEF_MS : a.m_seg;
    if (i < NC) {
        double s = 0.0;
        for (int k = 0; k < ms; ++k) s = fma(qm[i * ms + k], pr[ms + k], s);
        rhs = -s;
    } else if (i < NX) {
        double s = 0.0;
        for (int k = 0; k < ms; ++k) s = fma(qm[NC * ms + (i - NC) * ms + k], pr[k], s);
        rhs = -s;
    } else if (i < nr) {
        const int e = i - NX;
        if (!DEF && a.with_goal && e >= 6) rhs = (e == 6) ? pr[2 * ms] : (e == 7) ? pr[2 * ms + 1] : 0.0;
        else rhs = a.bscene[(size_t)scene * a.neq + e];
    }
    }
    const int ld = s1_ld(nr);
    if (i < nr) vec[i] = rhs;
    __syncwarp();
    const double sol = i < nr ? s1_rowdot(kinv, vec, i, nr, ld) : 0.0;
    __syncwarp();
    if (i < nr) vec[i] = sol;
    __syncwarp();
    double res = i < nr ? s1_rowdot(kkt, vec, i, nr, ld) : 0.0;
    __syncwarp();
    res = fabs(res - rhs);
    double scale = fabs(rhs);
    for (int o = 16; o >= 1; o >>= 1) {
        res = fmax(res, __shfl_xor_sync(0xffffffffu, res, o));
        scale = fmax(scale, __shfl_xor_sync(0xffffffffu, scale, o));
    }
    const bool finite_rhs = __all_sync(0xffffffffu, isfinite(rhs));
    if (lane == 0 && !finite_rhs) atomicOr(a.err + (!DEF && a.rhs_in ? 0 : row / a.B), ERR_BAD_RHS);
    else if (lane == 0 && !(res <= 1e-8 * (1.0 + scale)))
        atomicOr(a.err + (!DEF && a.rhs_in ? 0 : row / a.B), ERR_KKT_RESID);
    if (!DEF && a.rhs_in) {
        if (i < nr) a.sol_out[(size_t)row * nr + i] = sol;
        return;
    }
    if (i < NX) {
        if (a.xi_bar) a.xi_bar[(size_t)row * NX + i] = sol;
    } else if (i < nr) {
        const int e = i - NX;
        if (a.mu) a.mu[(size_t)row * a.neq + e] = sol;
        if (a.b_out) a.b_out[(size_t)row * a.neq + e] = rhs;
    }
}

__global__ void __launch_bounds__(256) stage1_kernel(const S1Args a) {
    extern __shared__ __align__(16) unsigned char smem[];
    double* kinv = reinterpret_cast<double*>(smem);
    double* kkt = kinv + a.nr * s1_ld(a.nr);
    double* qm = kkt + a.nr * s1_ld(a.nr);                       // qmx | qmy
    double* vw = qm + 2 * NC * a.m_seg;                          // per-warp vectors
    stage1_load(a, kinv, kkt, qm);
    __syncthreads();
    const int row = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (row >= a.total) return;
    stage1_body(a, row, a.rhs_in ? nullptr : a.params + (size_t)row * a.dim, kinv, kkt, qm,
                vw + (threadIdx.x >> 5) * S1_VEC);
}

// K4 + K1 fused for the CEM cycle: p = mean + z L^T (pkg/bilevel.py:51-57; z from the caller
// or device Philox; the warm-start tile on iteration 1) written to params, then stage 1.
template <bool DEF>
__global__ void __launch_bounds__(256) sample_stage1_kernel(CemState cs, int it, const double* z, const double* warm,
                                                           uint64_t seed, int scene_offset, double* params,
                                                           const S1Args a) {
    extern __shared__ __align__(16) unsigned char smem[];
    double* kinv = reinterpret_cast<double*>(smem);
    double* kkt = kinv + a.nr * s1_ld(a.nr);
    double* qm = kkt + a.nr * s1_ld(a.nr);
    double* pw = qm + 2 * NC * a.m_seg;                  // one behaviour vector per warp
    double* vw = pw + (blockDim.x >> 5) * MAX_DIM;       // per-warp mat-vec vectors
    stage1_load(a, kinv, kkt, qm);
    __syncthreads();
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int row = blockIdx.x * (blockDim.x >> 5) + wid;
    if (row >= a.total) return;
    const int scene = row / a.B, j = row % a.B;
    if (cs.err[scene]) return;                          // failed scene: frozen until the cycle ends
    const int d = DEF ? S1_DEF_DIM : cs.dim;
    double* pr = pw + wid * MAX_DIM;
    if (warm != nullptr) {
        if (lane < d) pr[lane] = warm[(size_t)row * d + lane];
    } else {
        double zz[MAX_DIM];
        if (z != nullptr) {
            for (int q = 0; q < d; ++q) zz[q] = z[(size_t)row * d + q];
        } else {
            philox_normals_warp(seed, scene + scene_offset, it, j, zz, d, lane);
        }
        if (lane < d) {
            const double* L = cs.L + scene * d * d;
            double acc = 0.0;
            for (int q = 0; q < d; ++q) acc = fma(zz[q], L[lane * d + q], acc);
            pr[lane] = cs.mean[scene * d + lane] + acc;
        }
    }
    __syncwarp();
    if (lane < d) params[(size_t)row * d + lane] = pr[lane];
    stage1_body<DEF>(a, row, pr, kinv, kkt, qm, vw + wid * S1_VEC);
}

// SamplingDistribution.sample (pkg/bilevel.py:51-57) for one distribution: the factor is
// computed by warp 0 (chol, 1e-5 I fallback), then p = mean + z L^T per sample.
__global__ void sample_one_kernel(int d, int count, const double* mean, const double* cov, const double* z,
                                  double* out) {
    __shared__ double L[MAX_DIM * MAX_DIM], csh[MAX_DIM * MAX_DIM], lsh[MAX_DIM * MAX_DIM];
    __shared__ double mu[MAX_DIM];
    for (int i = threadIdx.x; i < d * d; i += blockDim.x) csh[i] = cov[i];
    if (threadIdx.x < d) mu[threadIdx.x] = mean[threadIdx.x];
    __syncthreads();
    if (threadIdx.x < 32) warp_sampling_factor(csh, lsh, L, d, threadIdx.x);
    __syncthreads();
    for (int s = blockIdx.x * blockDim.x + threadIdx.x; s < count; s += gridDim.x * blockDim.x) {
        for (int r = 0; r < d; ++r) {
            double acc = 0.0;
            for (int q = 0; q < d; ++q) acc = fma(z[(size_t)s * d + q], L[r * d + q], acc);
            out[(size_t)s * d + r] = mu[r] + acc;
        }
    }
}

// Philox-keyed variant of the above (bd_sample_philox).
__global__ void sample_philox_kernel(int d, int count, const double* mean, const double* cov, uint64_t seed,
                                     int scene, int iteration, int first_index, double* out) {
    __shared__ double L[MAX_DIM * MAX_DIM], csh[MAX_DIM * MAX_DIM], lsh[MAX_DIM * MAX_DIM];
    __shared__ double mu[MAX_DIM];
    for (int i = threadIdx.x; i < d * d; i += blockDim.x) csh[i] = cov[i];
    if (threadIdx.x < d) mu[threadIdx.x] = mean[threadIdx.x];
    __syncthreads();
    if (threadIdx.x < 32) warp_sampling_factor(csh, lsh, L, d, threadIdx.x);
    __syncthreads();
    for (int s = blockIdx.x * blockDim.x + threadIdx.x; s < count; s += gridDim.x * blockDim.x) {
        double z[MAX_DIM];
        philox_normals(seed, scene, iteration, first_index + s, z, d);
        for (int r = 0; r < d; ++r) {
            double acc = 0.0;
            for (int q = 0; q < d; ++q) acc = fma(z[q], L[r * d + q], acc);
            out[(size_t)s * d + r] = mu[r] + acc;
        }
    }
}

// Per-iteration maximum over the spread slots of the early-exit buffer (one scene).
__global__ void itmax_reduce_kernel(const unsigned* itmax, int iters, float* out) {
    for (int it = blockIdx.x * blockDim.x + threadIdx.x; it < iters; it += gridDim.x * blockDim.x) {
        unsigned mx = 0;
        for (int s = 0; s < ITMAX_SLOTS; ++s) mx = max(mx, itmax[(size_t)it * ITMAX_SLOTS + s]);
        out[it] = __uint_as_float(mx);
    }
}

// ---------------------------------------------------------------- trajectory evaluation
// eval_trajectory (pkg/basis.py:182-195) in fp64: one thread per (sample, timestep).
__global__ void eval_kernel(int count, int m, const double* __restrict__ W, const double* __restrict__ Wd,
                            const double* __restrict__ Wdd, const double* __restrict__ xi, double* x, double* y,
                            double* xd, double* yd, double* xdd, double* ydd) {
    const size_t id = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (id >= (size_t)count * m) return;
    const int s = (int)(id / m), t = (int)(id % m);
    const double* c = xi + (size_t)s * NX;
    double v[6] = {0, 0, 0, 0, 0, 0};
    for (int k = 0; k < NC; ++k) {
        const double w = W[t * NC + k], wd = Wd[t * NC + k], wdd = Wdd[t * NC + k];
        v[0] = fma(w, c[k], v[0]);
        v[1] = fma(w, c[NC + k], v[1]);
        v[2] = fma(wd, c[k], v[2]);
        v[3] = fma(wd, c[NC + k], v[3]);
        v[4] = fma(wdd, c[k], v[4]);
        v[5] = fma(wdd, c[NC + k], v[5]);
    }
    double* outs[6] = {x, y, xd, yd, xdd, ydd};
    for (int q = 0; q < 6; ++q)
        if (outs[q]) outs[q][id] = v[q];
}

// ---------------------------------------------------------------- fp64 residual evaluator
// batch_residuals (pkg/constraints.py:95-153) directly in fp64: one warp per sample.
struct ResArgs {
    int total, B, m, n_obs, n_curv;
    const double* W; const double* Wd; const double* Wdd;
    const double* ox; const double* oy;     // S x n_obs x m (unscaled)
    const double* lim;                      // S x 9: a b vmin vmax amax kmax cmax ylb yub
    const double* curv;                     // S x 2 x n_curv
    const double* xi; double* out;
};

__device__ __forceinline__ double interp_d(double x, const double* xs, const double* ks, int n) {
    if (x != x) return x;
    if (x <= xs[0]) return ks[0];
    if (x >= xs[n - 1]) return ks[n - 1];
    int lo = 0, hi = n - 1;
    while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (xs[mid] <= x) lo = mid; else hi = mid;
    }
    const double slope = (ks[lo + 1] - ks[lo]) / (xs[lo + 1] - xs[lo]);
    return ks[lo] + slope * (x - xs[lo]);
}

__global__ void residual_kernel(const ResArgs a) {
    const int lane = threadIdx.x & 31;
    const int row = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (row >= a.total) return;
    const int scene = row / a.B;
    const double* L = a.lim + (size_t)scene * 9;
    const double ea = L[0], eb = L[1], vmin = L[2], vmax = L[3], amax = L[4], kmax = L[5], cmax = L[6];
    const double ylb = L[7], yub = L[8];
    const double* c = a.xi + (size_t)row * NX;
    const double* ox = a.ox + (size_t)scene * a.n_obs * a.m;
    const double* oy = a.oy + (size_t)scene * a.n_obs * a.m;
    const double* cx = a.curv + (size_t)scene * 2 * a.n_curv;
    double coll = 0, vel = 0, acc = 0, cur = 0, cen = 0, lan = 0;
    for (int t = lane; t < a.m; t += 32) {
        double X = 0, Y = 0, XD = 0, YD = 0, XDD = 0, YDD = 0;
        for (int k = 0; k < NC; ++k) {
            const double w = a.W[t * NC + k], wd = a.Wd[t * NC + k], wdd = a.Wdd[t * NC + k];
            X = fma(w, c[k], X); Y = fma(w, c[NC + k], Y);
            XD = fma(wd, c[k], XD); YD = fma(wd, c[NC + k], YD);
            XDD = fma(wdd, c[k], XDD); YDD = fma(wdd, c[NC + k], YDD);
        }
        for (int o = 0; o < a.n_obs; ++o) {
            const double dx = (X - ox[o * a.m + t]) / ea, dy = (Y - oy[o * a.m + t]) / eb;
            coll += fmax(1.0 - dx * dx - dy * dy, 0.0);
        }
        const double sp = hypot(XD, YD);
        vel += fmax(sp - vmax, 0.0) + fmax(vmin - sp, 0.0);
        acc += fmax(hypot(XDD, YDD) - amax, 0.0);
        const double s3 = fmax(sp, 1e-6);
        cur += fmax(fabs(YDD * XD - XDD * YD) / (s3 * s3 * s3) - kmax, 0.0);
        if (a.n_curv > 0) cen += fmax(XD * XD * fabs(interp_d(X, cx, cx + a.n_curv, a.n_curv)) - cmax, 0.0);
        lan += fmax(Y - yub, 0.0) + fmax(ylb - Y, 0.0);
    }
    for (int o = 16; o >= 1; o >>= 1) {
        coll += __shfl_xor_sync(0xffffffffu, coll, o);
        vel += __shfl_xor_sync(0xffffffffu, vel, o);
        acc += __shfl_xor_sync(0xffffffffu, acc, o);
        cur += __shfl_xor_sync(0xffffffffu, cur, o);
        cen += __shfl_xor_sync(0xffffffffu, cen, o);
        lan += __shfl_xor_sync(0xffffffffu, lan, o);
    }
    // summed in the reference's dict order (pkg/constraints.py:153)
    if (lane == 0) a.out[row] = ((((coll + vel) + acc) + cur) + cen) + lan;
}

}  // namespace bd
