// K3 select + refit and K4 sampler of the CEM upper level (sm_100a).
//
// rank_samples (pkg/bilevel.py:129-137), _elite_weights / update_distribution
// (:163-194), IterationStats (:100-108, :282-292), the best EliteRecord
// (:272-280) and SamplingDistribution.sample (:51-57).
#pragma once

#include "bd_common.cuh"

namespace bd {

// Order-preserving map of a double onto uint64 (numpy: -0 == +0, NaN last).
__device__ __forceinline__ unsigned long long ordered_bits(double x) {
    if (x != x) return 0xFFFFFFFFFFFFFFFEull;          // every NaN sorts after all numbers, before padding
    if (x == 0.0) return 0x8000000000000000ull;       // -0 == +0
    const unsigned long long b = (unsigned long long)__double_as_longlong(x);
    return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

// aug = c + w r with numpy's rounding (no FMA contraction), so near-ties order as in
// rank_samples (pkg/bilevel.py:134-135).
__device__ __forceinline__ double aug_cost(double c, double w, double r) { return __dadd_rn(c, __dmul_rn(w, r)); }

// Warp-cooperative Cholesky of a dim x dim SPD matrix held in shared memory (row-major, fp64).
// Lane r < dim keeps row r of L in registers; column j is formed by every lane from row j of L
// (broadcast by shuffles), lane j's value being the pivot: the same operations in the same order
// as the textbook column loop (pivot a_jj - sum_k l_jk^2, entries (a_ij - sum_k l_ik l_jk) / l_jj),
// without shared-memory round trips on the dependency chain.  D is the compile-time size (every
// loop unrolled, L in registers: 8 x 8 ~2.7k cycles against ~6k for a shared-memory column loop).
// Returns false (in every lane) if the matrix is not positive definite; L is then unspecified.
template <int D>
__device__ __forceinline__ bool warp_chol_fixed(const double* A, double* L, int lane) {
    // one lane, every entry in registers, no warp-synchronous step on the chain: column j costs the
    // j-deep FMA chains of its entries (independent) plus one sqrt and one reciprocal.  Inside the
    // persistent CEM kernel every shuffle / warp barrier on this chain cost ~400 cycles (22k cycles
    // for the lane-parallel form); this form takes ~2k.
    bool ok = true;
    if (lane == 0) {
        double Lm[D][D];
#pragma unroll
        for (int i = 0; i < D; ++i)
#pragma unroll
            for (int k = 0; k <= i; ++k) Lm[i][k] = A[i * D + k];
#pragma unroll
        for (int j = 0; j < D; ++j) {
            double piv = Lm[j][j];
#pragma unroll
            for (int k = 0; k < j; ++k) piv -= Lm[j][k] * Lm[j][k];
            ok = ok && piv > 0.0;
            const double ljj = sqrt(piv);
            const double rinv = 1.0 / ljj;          // LAPACK dpotf2 scales the column by 1 / l_jj
            Lm[j][j] = ljj;
#pragma unroll
            for (int i = j + 1; i < D; ++i) {
                double t = Lm[i][j];
#pragma unroll
                for (int k = 0; k < j; ++k) t -= Lm[i][k] * Lm[j][k];
                Lm[i][j] = t * rinv;
            }
        }
#pragma unroll
        for (int i = 0; i < D; ++i)
#pragma unroll
            for (int k = 0; k < D; ++k) L[i * D + k] = k <= i ? Lm[i][k] : 0.0;
    }
    ok = __shfl_sync(0xffffffffu, ok, 0);
    __syncwarp();
    return ok;
}

// Any size <= MAX_DIM: lane 0 forms the pivot of column j, lanes i > j the sub-diagonal entries.
__device__ bool warp_chol(const double* A, double* L, int d, int lane) {
    if (d == 8) return warp_chol_fixed<8>(A, L, lane);
    for (int i = lane; i < d * d; i += 32) L[i] = 0.0;
    __syncwarp();
    bool ok = true;
    for (int j = 0; j < d; ++j) {
        double piv = 0.0;
        if (lane == 0) {
            double s = A[j * d + j];
            for (int k = 0; k < j; ++k) s -= L[j * d + k] * L[j * d + k];
            piv = s;
            L[j * d + j] = s > 0.0 ? sqrt(s) : 0.0;
        }
        piv = __shfl_sync(0xffffffffu, piv, 0);
        __syncwarp();
        if (!(piv > 0.0)) { ok = false; break; }
        const double ljj = L[j * d + j];
        const int i = j + 1 + lane;
        if (i < d) {
            double t = A[i * d + j];
            for (int k = 0; k < j; ++k) t -= L[i * d + k] * L[j * d + k];
            L[i * d + j] = t / ljj;
        }
        __syncwarp();
    }
    return ok;
}

// SamplingDistribution.sample's factor (pkg/bilevel.py:52-55): chol(cov), falling back to
// chol(cov + 1e-5 I); a failing fallback leaves NaN (numpy would raise).  One warp; cov_sh and
// L_sh are shared-memory scratch (cov_sh is modified by the fallback); Lout receives the factor.
__device__ void warp_sampling_factor(double* cov_sh, double* L_sh, double* Lout, int d, int lane) {
    if (!warp_chol(cov_sh, L_sh, d, lane)) {
        if (lane < d) cov_sh[lane * d + lane] += 1e-5;
        __syncwarp();
        if (!warp_chol(cov_sh, L_sh, d, lane))
            for (int i = lane; i < d * d; i += 32) L_sh[i] = __longlong_as_double(0x7ff8000000000000ll);
        __syncwarp();
    }
    for (int i = lane; i < d * d; i += 32) Lout[i] = L_sh[i];
}

// ---------------------------------------------------------------- Philox4x32-10 normals
__device__ __forceinline__ void philox_round(uint32_t (&c)[4], uint32_t (&k)[2]) {
    const uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u;
    const uint32_t hi0 = __umulhi(M0, c[0]), lo0 = M0 * c[0];
    const uint32_t hi1 = __umulhi(M1, c[2]), lo1 = M1 * c[2];
    const uint32_t n0 = hi1 ^ c[1] ^ k[0], n2 = hi0 ^ c[3] ^ k[1];
    c[0] = n0; c[1] = lo1; c[2] = n2; c[3] = lo0;
    k[0] += 0x9E3779B9u; k[1] += 0xBB67AE85u;
}

__device__ __forceinline__ void philox4(uint32_t (&c)[4], uint64_t seed) {
    uint32_t k[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
#pragma unroll
    for (int r = 0; r < 10; ++r) philox_round(c, k);
}

// Standard normals keyed by (seed, scene, CEM iteration, sample index): identical for any GPU count.
__device__ void philox_normals(uint64_t seed, uint32_t scene, uint32_t it, uint32_t sample, double* z, int d) {
    for (int base = 0; base < d; base += 4) {
        uint32_t c[4] = {sample, it, scene, (uint32_t)(base / 4)};
        philox4(c, seed);
        for (int q = 0; q < 4 && base + q < d; q += 2) {
            const double u1 = ((double)c[q] + 0.5) * 2.3283064365386963e-10;     // (0, 1)
            const double u2 = ((double)c[q + 1] + 0.5) * 2.3283064365386963e-10;
            const double r = sqrt(-2.0 * log(u1));
            double s, co;
            sincospi(2.0 * u2, &s, &co);
            z[base + q] = r * co;
            if (base + q + 1 < d) z[base + q + 1] = r * s;
        }
    }
}

// Warp-cooperative form for one sample per warp: lane l draws Box-Muller pair l (the same
// counter block and arithmetic as philox_normals, so bit-identical values) and the d normals are
// broadcast to every lane.  Must be called by all 32 lanes.
__device__ __forceinline__ void philox_normals_warp(uint64_t seed, uint32_t scene, uint32_t it, uint32_t sample,
                                                    double* z, int d, int lane) {
    double a = 0.0, b = 0.0;
    if (lane < (d + 1) / 2) {
        uint32_t c[4] = {sample, it, scene, (uint32_t)(lane / 2)};
        philox4(c, seed);
        const int q = (2 * lane) & 3;
        const double u1 = ((double)c[q] + 0.5) * 2.3283064365386963e-10;
        const double u2 = ((double)c[q + 1] + 0.5) * 2.3283064365386963e-10;
        const double r = sqrt(-2.0 * log(u1));
        double sn, co;
        sincospi(2.0 * u2, &sn, &co);
        a = r * co;
        b = r * sn;
    }
    for (int k = 0; k < d; ++k) z[k] = __shfl_sync(0xffffffffu, (k & 1) ? b : a, k >> 1);
}

// ---------------------------------------------------------------- CEM state
struct CemState {
    int S, B, dim, n_cons, n_elite, iters;
    double eta, gamma, w_res;
    double* mean;       // S x dim
    double* cov;        // S x dim x dim
    double* L;          // S x dim x dim   sampling factor of cov
    int* err;           // S   sticky error bits (stage-1 / AM)
    int* done;          // S   completed CEM iterations (-1 = failed in iteration 1)
    // per-iteration data
    const double* resid;   // S*B
    const double* cost;    // S*B
    const double* params;  // S*B x dim
    const double* xi;      // S*B x NX
    // outputs
    long long* cons_idx;   // S x n_cons   (nullable)
    long long* elite_idx;  // S x n_elite  (nullable)
    double* elite_aug;     // S x n_elite  (nullable)
    double* stats;         // S x iters x 6 (nullable)
    long long* best_index; // S
    double* best_params;   // S x dim
    double* best_xi;       // S x NX
    double* best_scal;     // S x 3: cost, residual, aug
};

// Initial factor of the configured Gaussian (pkg/bilevel.py:244).
__global__ void cem_init_kernel(CemState s, const double* mean0, const double* cov0) {
    const int scene = blockIdx.x;
    const int d = s.dim;
    __shared__ double csh[MAX_DIM * MAX_DIM], lsh[MAX_DIM * MAX_DIM];
    for (int i = threadIdx.x; i < d; i += blockDim.x) s.mean[scene * d + i] = mean0[scene * d + i];
    for (int i = threadIdx.x; i < d * d; i += blockDim.x) {
        const double v = cov0[scene * d * d + i];
        s.cov[scene * d * d + i] = v;
        csh[i] = v;
    }
    __syncthreads();
    if (threadIdx.x < 32) warp_sampling_factor(csh, lsh, s.L + scene * d * d, d, threadIdx.x);
    if (threadIdx.x == 0) {
        s.err[scene] = 0;
        s.done[scene] = 0;
    }
}

// Two block-wide sums in one pass (each in block_sum's order; results valid in every thread).
// red holds 64 doubles.
__device__ __forceinline__ double block_sum2(double v, double u, double* red, double& usum) {
    for (int o = 16; o >= 1; o >>= 1) {
        v += __shfl_xor_sync(0xffffffffu, v, o);
        u += __shfl_xor_sync(0xffffffffu, u, o);
    }
    __syncthreads();
    if ((threadIdx.x & 31) == 0) {
        red[threadIdx.x >> 5] = v;
        red[32 + (threadIdx.x >> 5)] = u;
    }
    __syncthreads();
    const int nw = blockDim.x >> 5, ln = threadIdx.x & 31;
    double t = ln < nw ? red[ln] : 0.0, r = ln < nw ? red[32 + ln] : 0.0;
    for (int o = 16; o >= 1; o >>= 1) {
        t += __shfl_xor_sync(0xffffffffu, t, o);
        r += __shfl_xor_sync(0xffffffffu, r, o);
    }
    usum = r;
    return t;
}

// Stable residual order by counting (np.argsort(kind="stable"), pkg/bilevel.py:131): one warp per
// sample counts the keys that precede it, (key, index) lexicographic, and scatters the sample to
// its rank.  O(B^2) comparisons, but spread over the whole GPU instead of a single CTA's sort.
__global__ void __launch_bounds__(256) rank_count_kernel(const double* resid, const int* err, int S, int B,
                                                         int* order) {
    const int lane = threadIdx.x & 31;
    const long gi = (long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (gi >= (long)S * B) return;
    const int scene = (int)(gi / B), i = (int)(gi % B);
    if (err && err[scene]) return;
    const double* r = resid + (size_t)scene * B;
    const unsigned long long ki = ordered_bits(r[i]);
    int cnt = 0;
    for (int j = lane; j < B; j += 32) {
        const unsigned long long kj = ordered_bits(__ldg(r + j));
        cnt += (kj < ki) || (kj == ki && j < i);
    }
    for (int o = 16; o >= 1; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
    BD_CHECK(cnt >= 0 && cnt < B);
    if (lane == 0) order[(size_t)scene * B + cnt] = i;
}

// Same ranking with the scene's keys staged once per CTA in shared memory (B <= RANK_SMEM_MAX):
// grid (ceil(B / 32), S), 8 warps x 4 samples per CTA.  Cuts the L2 traffic of the per-warp
// scans from B doubles per sample to B keys per 32 samples.
constexpr int RANK_SMEM_MAX = 12288;
__global__ void __launch_bounds__(256) rank_count_smem_kernel(const double* resid, const int* err, int B, int* order) {
    extern __shared__ __align__(16) unsigned char smem[];
    unsigned long long* keys = reinterpret_cast<unsigned long long*>(smem);
    const int scene = blockIdx.y;
    if (err && err[scene]) return;
    const double* r = resid + (size_t)scene * B;
    for (int j = threadIdx.x; j < B; j += blockDim.x) keys[j] = ordered_bits(__ldg(r + j));
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int q = 0; q < 4; ++q) {
        const int i = blockIdx.x * 32 + warp * 4 + q;
        if (i >= B) break;
        const unsigned long long ki = keys[i];
        int cnt = 0;
        for (int j = lane; j < B; j += 32) {
            const unsigned long long kj = keys[j];
            cnt += (kj < ki) || (kj == ki && j < i);
        }
        for (int o = 16; o >= 1; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
        BD_CHECK(cnt >= 0 && cnt < B);
        if (lane == 0) order[(size_t)scene * B + cnt] = i;
    }
}

// Dynamic shared memory of rank_refit_kernel (bytes).
__host__ __device__ inline size_t rank_refit_smem(int n_cons, int n_elite, int dim) {
    const int staged = n_elite <= 128 ? n_elite : 0;
    return (size_t)n_cons * (8 + 8 + 8 + 4 + 4 + 8) + (size_t)staged * dim * 8;   // key2 augc aug2 cidx idx2 w
}

constexpr int RANK_REFIT_THREADS = 1024;
constexpr int REFIT_SUM_THREADS = 224;   // threads that take part in the refit sums (see rank_refit_block)

// rank_samples + update_distribution + IterationStats + best record for one CEM
// iteration, one CTA (1024 threads) per scene, on the residual order produced by
// rank_count_kernel.  The n constraint elites are ranked by augmented cost (ties by sample
// index, np.lexsort((idx, aug))) by counting in shared memory, the q elite set-point vectors
// staged in shared memory and the weighted mean / covariance reduced warp-parallel in fp64; the
// tail (Cholesky factor, IterationStats, best record) runs on separate warps concurrently.
// The body runs on any CTA of <= 1024 threads (>= 4 warps): rank_refit_kernel (one CTA per scene)
// and the single-scene persistent CEM kernel, whose last CTA to finish ranking runs it.
#ifdef BD_PHASE_TIMING
#define RR_STAMP(k) if (threadIdx.x == 0) { unsigned long long t_; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t_)); rr_t[k] = t_; }
#else
#define RR_STAMP(k)
#endif
__device__ __forceinline__ void rank_refit_block(const CemState& s, int it, const int* order, int scene,
                                                 unsigned char* smem) {
#ifdef BD_PHASE_TIMING
    __shared__ unsigned long long rr_t[12];
#endif
    RR_STAMP(0);
    const int d = s.dim;
    if (s.err[scene] != 0) {            // this iteration (or an earlier one) failed: freeze
        if (threadIdx.x == 0 && s.done[scene] == it) s.done[scene] = (it == 0) ? -1 : it;
        return;
    }
    const int n = s.n_cons, q = s.n_elite;
    // dynamic layout (rank_refit_smem): key2 | aug | aug2 | cidx | idx2 | w | staged elite set-points
    unsigned long long* key2 = reinterpret_cast<unsigned long long*>(smem);
    double* augc = reinterpret_cast<double*>(key2 + n);      // aug of constraint elite i (residual order)
    double* aug2 = augc + n;                                  // aug by elite rank
    int* cidx = reinterpret_cast<int*>(aug2 + n);
    int* idx2 = cidx + n;
    double* w = reinterpret_cast<double*>(idx2 + n);          // n ints + n ints: 8-byte aligned
    double* pe = w + n;                                       // q <= 128 staged; larger q read from global
    __shared__ double red[64];
    __shared__ double mu_new[MAX_DIM];
    __shared__ double cnew[MAX_DIM * MAX_DIM];
    __shared__ double csym[MAX_DIM * MAX_DIM], lsh[MAX_DIM * MAX_DIM];
    const size_t base = (size_t)scene * s.B;
    const int* ord = order + base;
    // constraint elites: first n of the stable residual order; aug = cost + w r
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const int j = ord[i];
        BD_CHECK(j >= 0 && j < s.B);
        const double a = aug_cost(s.cost[base + j], s.w_res, s.resid[base + j]);
        augc[i] = a;
        key2[i] = ordered_bits(a);
        cidx[i] = j;
        if (s.cons_idx) s.cons_idx[(size_t)scene * n + i] = j;
    }
    __syncthreads();
    RR_STAMP(1);
    // rank among the constraint elites by (aug, sample index), scatter index and aug: G threads per
    // elite (G = 4, 2 or 1: one round whenever the CTA has G n threads), each counting, branch-free,
    // the keys that precede it in a 1/G share of the list; the G counts meet by shuffles (the group
    // is G aligned lanes of one warp)
    {
        const int G = (int)blockDim.x >= 4 * n ? 4 : ((int)blockDim.x >= 2 * n ? 2 : 1);
        const int share = (n + G - 1) / G;
        for (int t0 = 0; t0 < G * n; t0 += blockDim.x) {
            const int t = t0 + threadIdx.x;
            const int i = t / G, g = t % G;
            int rk = 0;
            if (i < n) {
                const unsigned long long ki = key2[i];
                const int ji = cidx[i];
                const int k0 = g * share, k1 = min(n, (g + 1) * share);
                // eight keys per step, four independent counts (the loads of a step overlap)
                int c4[4] = {0, 0, 0, 0};
                int k = k0;
                for (; k + 8 <= k1; k += 8) {
#pragma unroll
                    for (int u = 0; u < 8; ++u) {
                        const unsigned long long kk = key2[k + u];
                        const int ck = cidx[k + u];
                        c4[u & 3] += (int)(kk < ki) | ((int)(kk == ki) & (int)(ck < ji));
                    }
                }
                for (; k < k1; ++k) {
                    const unsigned long long kk = key2[k];
                    c4[0] += (int)(kk < ki) | ((int)(kk == ki) & (int)(cidx[k] < ji));
                }
                rk = (c4[0] + c4[1]) + (c4[2] + c4[3]);
            }
            if (G >= 2) rk += __shfl_xor_sync(0xffffffffu, rk, 1);
            if (G == 4) rk += __shfl_xor_sync(0xffffffffu, rk, 2);
            if (i < n && g == 0) {
                BD_CHECK(rk >= 0 && rk < n);
                idx2[rk] = cidx[i];
                aug2[rk] = augc[i];
            }
        }
    }
    __syncthreads();
    RR_STAMP(2);
    // elite weights exp(-(aug - min aug)/gamma), uniform fallback (pkg/bilevel.py:163-172)
    const int j0 = idx2[0];
    const double amin = aug2[0];
    double part = 0.0, cpart = 0.0;
    const bool staged = q <= 128;
    // the elite set-points are staged first so their L2 loads overlap the exp() below
    if (staged) {
        const int nq = q * d;
#pragma unroll 4
        for (int e = threadIdx.x; e < nq; e += blockDim.x) pe[e] = s.params[(base + idx2[e / d]) * d + e % d];
    }
    for (int i = threadIdx.x; i < q; i += blockDim.x) {
        const int j = idx2[i];
        const double aug = aug2[i];
        const double wi = exp(-(aug - amin) / s.gamma);
        w[i] = wi;
        part += wi;
        cpart += s.cost[base + j];
        if (s.elite_idx) s.elite_idx[(size_t)scene * q + i] = j;
        if (s.elite_aug) s.elite_aug[(size_t)scene * q + i] = aug;
    }
    double csum;
    const double total = block_sum2(part, cpart, red, csum);
    RR_STAMP(3);
    const bool uniform = !(isfinite(total) && total > 0.0);
    for (int i = threadIdx.x; i < q; i += blockDim.x) w[i] = uniform ? 1.0 / q : w[i] / total;
    __syncthreads();
    RR_STAMP(4);
    // weighted mean / covariance refit (pkg/bilevel.py:175-194): warp per output entry
    const double eta = s.eta;
    double* mean = s.mean + scene * d;
    double* cov = s.cov + scene * d * d;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    auto P = [&](int i, int r) -> double {
        return staged ? pe[i * d + r] : __ldg(s.params + (base + idx2[i]) * d + r);
    };
    // every thread takes one entry and a strided chunk of the elites; the chunk partials are
    // folded in a fixed order (deterministic).  The chunking uses at most REFIT_SUM_THREADS
    // threads whatever the CTA size, so the 1024-thread kernel and the 224/256-thread persistent
    // CEM kernel sum in the same order (bit-identical refits).
    __shared__ double partial[RANK_REFIT_THREADS];
    const int nsum = min((int)blockDim.x, REFIT_SUM_THREADS);
    // each chunk sum runs as four interleaved partial sums (elites i, i + 4 chunks, ...), added
    // pairwise at the end: four independent fp64 chains instead of one
    {
        const int chunks = max(1, min(8, nsum / d)), e = threadIdx.x % d, ch = threadIdx.x / d;
        double a4[4] = {0.0, 0.0, 0.0, 0.0};
        if (ch < chunks) {                  // element k of the chunk's sequence -> a4[k & 3]
            int i = ch;
            for (; i + 3 * chunks < q; i += 4 * chunks) {
#pragma unroll
                for (int u = 0; u < 4; ++u) a4[u] = fma(w[i + u * chunks], P(i + u * chunks, e), a4[u]);
            }
#pragma unroll
            for (int u = 0; u < 3; ++u)
                if (i + u * chunks < q) a4[u] = fma(w[i + u * chunks], P(i + u * chunks, e), a4[u]);
        }
        const double acc = (a4[0] + a4[1]) + (a4[2] + a4[3]);
        partial[threadIdx.x] = acc;
        __syncthreads();
        if (threadIdx.x < d) {
            double t = 0.0;
            for (int k = 0; k < chunks; ++k) t += partial[k * d + threadIdx.x];
            mu_new[threadIdx.x] = (1.0 - eta) * mean[threadIdx.x] + eta * t;
        }
        __syncthreads();
    RR_STAMP(5);
    }
    {
        const int dd = d * d, chunks = max(1, nsum / dd), e = threadIdx.x % dd, ch = threadIdx.x / dd;
        const int r = e / d, c = e % d;
        double a4[4] = {0.0, 0.0, 0.0, 0.0};
        if (ch < chunks) {
            const double mr = mu_new[r], mc = mu_new[c];
            int i = ch;
            for (; i + 3 * chunks < q; i += 4 * chunks) {
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int iu = i + u * chunks;
                    a4[u] = fma(w[iu] * (P(iu, r) - mr), P(iu, c) - mc, a4[u]);
                }
            }
#pragma unroll
            for (int u = 0; u < 3; ++u) {
                const int iu = i + u * chunks;
                if (iu < q) a4[u] = fma(w[iu] * (P(iu, r) - mr), P(iu, c) - mc, a4[u]);
            }
        }
        const double acc = (a4[0] + a4[1]) + (a4[2] + a4[3]);
        partial[threadIdx.x] = acc;
        __syncthreads();
        if (threadIdx.x < dd) {
            double t = 0.0;
            for (int k = 0; k < chunks; ++k) t += partial[k * dd + threadIdx.x];
            cnew[threadIdx.x] = (1.0 - eta) * cov[threadIdx.x] + eta * t + (r == c ? 1e-6 : 0.0);
        }
        __syncthreads();
    RR_STAMP(6);
    }
    for (int e = threadIdx.x; e < d * d; e += blockDim.x) {
        const int r = e / d, c = e % d;
        const double v = 0.5 * (cnew[r * d + c] + cnew[c * d + r]);
        cov[e] = v;
        csym[e] = v;
    }
    if (threadIdx.x < d) mean[threadIdx.x] = mu_new[threadIdx.x];
    __syncthreads();
    RR_STAMP(7);
    if (warp == 0) {
        warp_sampling_factor(csym, lsh, s.L + scene * d * d, d, lane);
        if (lane == 0) { RR_STAMP(9); }
    } else if (warp == 1) {
        if (lane == 0) {
            // IterationStats (pkg/bilevel.py:282-292)
            const int B = s.B;
            const double rmin = s.resid[base + ord[0]], rmax = s.resid[base + ord[B - 1]];
            const double rmed = (B & 1) ? s.resid[base + ord[B / 2]]
                                        : 0.5 * (s.resid[base + ord[B / 2 - 1]] + s.resid[base + ord[B / 2]]);
            double tr = 0.0;
            for (int i = 0; i < d; ++i) tr += cnew[i * d + i];   // symmetrisation keeps the diagonal
            if (s.stats) {
                double* st = s.stats + ((size_t)scene * s.iters + it) * 6;
                st[0] = csum / q; st[1] = amin; st[2] = tr; st[3] = rmin; st[4] = rmed; st[5] = rmax;
            }
            // best EliteRecord = elite[0] (pkg/bilevel.py:272-280)
            s.best_index[scene] = j0;
            s.best_scal[scene * 3 + 0] = s.cost[base + j0];
            s.best_scal[scene * 3 + 1] = s.resid[base + j0];
            s.best_scal[scene * 3 + 2] = amin;
            s.done[scene] = it + 1;
        }
    } else if (warp == 2) {
        if (lane < d) s.best_params[scene * d + lane] = s.params[(base + j0) * d + lane];
    } else if (warp == 3) {
        if (lane < NX && s.xi) s.best_xi[scene * NX + lane] = s.xi[(base + j0) * NX + lane];
    }
#ifdef BD_PHASE_TIMING
    __syncthreads();
    RR_STAMP(8);
    if (threadIdx.x == 0)
        printf("refit phases (us): chol %.2f; ", (rr_t[9] - rr_t[7]) * 1e-3);
    if (threadIdx.x == 0)
        printf("refit phases (us): load %.2f rank %.2f weights %.2f norm %.2f mean %.2f cov %.2f sym %.2f tail %.2f\n",
               (rr_t[1] - rr_t[0]) * 1e-3, (rr_t[2] - rr_t[1]) * 1e-3, (rr_t[3] - rr_t[2]) * 1e-3,
               (rr_t[4] - rr_t[3]) * 1e-3, (rr_t[5] - rr_t[4]) * 1e-3, (rr_t[6] - rr_t[5]) * 1e-3,
               (rr_t[7] - rr_t[6]) * 1e-3, (rr_t[8] - rr_t[7]) * 1e-3);
#endif
}

__global__ void __launch_bounds__(RANK_REFIT_THREADS) rank_refit_kernel(CemState s, int it, const int* order) {
    extern __shared__ __align__(16) unsigned char smem[];
    rank_refit_block(s, it, order, blockIdx.x, smem);
}

}  // namespace bd
