// K2: persistent alternating-minimisation projection kernel (sm_100a).
//
// Replaces ProjectionOperator.project (pkg/projection.py:216-339) together with
// polar_decompose (:100-135), _clip_magnitudes (:138-169), the per-iteration
// augmented KKT solve (:286-292), the direct residual evaluator
// (pkg/constraints.py:95-153) and the upper cost (pkg/bilevel.py:125-126).
//
// Mapping.  A sample is owned by a group of P lanes inside one warp; lane p of
// the group handles timesteps t = p, p+P, p+2P, ...  The basis rows, the
// scene's obstacle tile and the aug-KKT inverse blocks are staged once per CTA
// in shared memory; everything per (sample, obstacle, timestep) lives in
// registers and never returns to HBM between iterations.
//
// Algebra (verified against the reference in fp64):
//   * polar step in trig-free residual form: with w = (X-x_o)/a, (Y-y_o)/b and
//     q = |w|^2, the clipped back-projection residual is w (1 - q^-1/2) for
//     0 < q < 1, (-1, 0) for q == 0 and 0 otherwise (scaled by a, b);
//     velocity/acceleration residuals are v (|v| - clip|v|)/|v|.
//   * the KKT identity K Q~ + K_b A = I turns the per-iteration solve into the
//     increment  c <- c + K (l - c - rho g)  with l = xi_bar + lambda, where g is
//     the back-projected residual F^T(F c - h) and K the per-axis 11x11 block of
//     the aug-KKT inverse; lambda <- lambda - rho/2 g.  The first step adds
//     K_b (b - A xi_bar) so a xi_bar that does not satisfy A xi = b is handled
//     exactly as the reference's direct solve would.
//   * precision recipe: per-(o,t) and per-t work plus the W mat-vecs in fp32;
//     the per-sample state (c, lambda, the K apply) in fp64.
#pragma once

#include "bd_common.cuh"

namespace bd {

struct AmArgs {
    int m, neq, n_obs, n_curv, B, s_cta, max_iters;
    double rho;
    int sorted;                 // 1: scene tiles hold each timestep's obstacles sorted by -x/a (float2)
    const float* wrow;          // m x WROW        [W | Wd | Wdd] rows, fp32
    const double* kblk;         // NX x KSTR       aug-KKT inverse rows by value index (2 kk + axis)
    const double* kb;           // NX x neq        xi-b block of the aug-KKT inverse
    const double* aeq;          // neq x NX
    const float4* obs;          // S x m x n_obs/2 pairs (-x0/a, -x1/a, -y0/b, -y1/b), n_obs padded to even
    const SceneLim* lim;        // S
    const double* bscene;       // S x neq         shared b per scene (b0, zero goal rows)
    const float* curv;          // S x 2 x n_curv  (xs then ks)
    const double* xi_bar;       // (S*B) x NX
    const double* b;            // (S*B) x neq or nullptr (use bscene)
    double* xi_out;             // (S*B) x NX
    double* resid_out;          // S*B
    double* cost_out;           // S*B or nullptr
    float* hist_out;            // S x max_iters x B or nullptr
    unsigned* itmax;            // S x max_iters x ITMAX_SLOTS (float bits, atomicMax)
    unsigned long long* conflicts;  // S
    int* err;
    const int* replay;          // nullptr, or per-scene iteration count of a replay launch (0 = skip)
    // full pass only (replay == nullptr): the last CTA of each scene runs the batch-global exit scan
    double tol;
    int* iters_used;            // S (nullptr: no in-kernel scan)
    int* replay_out;            // S
    unsigned* done_ctr;         // S, zero before the launch, re-armed to zero by the last CTA
    // sharded batch over NVLink peer memory (nullptr: off): every (residual, cost) is also stored
    // straight into each rank's gathered arrays at global row p2p_row0 + local (the all-gather
    // fused into the epilogue, overlapping the remaining CTAs' math)
    void* const* p2p_bufs;      // world device pointers (symmetric buffers, peer-mapped)
    int p2p_world;
    long long p2p_row0;
    size_t p2p_res_off, p2p_cost_off;
};

// Batch-global early exit (pkg/projection.py:329): the first iteration whose batch maximum
// residual is <= tol sets iterations_used and, if that is before max_iters, the replay count.
// Out of line: run by one CTA per scene, kept away from the main loop's register allocation.
__device__ __noinline__ void exit_scan_block(unsigned* base, int max_iters, double tol, int scene,
                                                int* iters_used, int* replay, unsigned long long* conflicts) {
    // the slots of iteration it are 8 uint4 chunks held by 8 consecutive lanes; every chunk is
    // loaded (coalesced, up to 4 per thread in flight) before any is re-armed with zeros, so the
    // scan costs a few L2 round trips instead of one per slot
    static_assert(ITMAX_SLOTS == 32, "8 uint4 chunks per iteration");
    __shared__ int red[32];
    int first = max_iters;
    const int chunks = max_iters * (ITMAX_SLOTS / 4), T = blockDim.x;
    uint4* b4 = reinterpret_cast<uint4*>(base);
    const uint4 zero = make_uint4(0u, 0u, 0u, 0u);
    for (int c0 = 0; c0 < chunks; c0 += 4 * T) {
        uint4 v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int c = c0 + u * T + (int)threadIdx.x;
            v[u] = c < chunks ? __ldcg(b4 + c) : zero;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int c = c0 + u * T + (int)threadIdx.x;
            if (c < chunks) __stcg(b4 + c, zero);   // re-arm for the next launch (no memset needed)
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int c = c0 + u * T + (int)threadIdx.x;
            unsigned mx = max(max(v[u].x, v[u].y), max(v[u].z, v[u].w));
            mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
            mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
            mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, 4));
            const int it = c >> 3;
            if (c < chunks && (c & 7) == 0 && static_cast<double>(__uint_as_float(mx)) <= tol && it < first) first = it;
        }
    }
    for (int o = 16; o >= 1; o >>= 1) first = min(first, __shfl_xor_sync(0xffffffffu, first, o));
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = first;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < (int)(blockDim.x + 31) / 32; ++w) first = min(first, red[w]);
        const int used = first < max_iters ? first + 1 : max_iters;
        iters_used[scene] = used;
        const int rep = used < max_iters ? used : 0;
        if (replay) replay[scene] = rep;
        if (rep && conflicts) conflicts[scene] = 0ull;
    }
}

#ifndef BD_SORT_MIN_PAIRS
#define BD_SORT_MIN_PAIRS 8
#endif
constexpr int SORT_MIN_PAIRS = BD_SORT_MIN_PAIRS;   // >= 16 obstacles: sorted-window obstacle pass (dense scenes)

// Shared-memory carve-up, identical on host and device.
struct AmSmem {
    size_t w, obs, k, kb, a, curv, scr, dap, kap, kix, itm, hlp, red, total;
    // help > 0: the remainder warp's per-(sample, timestep) partial sums (am_helper), HSTR floats each
    static constexpr int HSTR = 28;
    static constexpr int RSTR = 28;     // row stride of the column-reduction buffer (conflict-free STS.128)
    __host__ __device__ AmSmem(int m, int n_obs, int neq, int n_curv, int s_cta, int threads, int P, bool curv_on,
                               int max_iters, int help = 0) {
        const int J = (m + P - 1) / P;
        size_t o = 0;
        w = o;    o = align_up(o + (size_t)m * WROW * 4, 16);
        obs = o;  o = align_up(o + (size_t)n_obs * m * 8, 16);          // n_obs already padded to even
        k = o;    o = align_up(o + (size_t)NX * KSTR * 8, 16);
        kb = o;   o = align_up(o + (size_t)NX * neq * 8, 16);
        a = o;    o = align_up(o + (size_t)neq * NX * 8, 16);
        curv = o; o = align_up(o + (size_t)2 * n_curv * 4, 16);
        scr = o;  o = align_up(o + (size_t)s_cta * SCR_BYTES, 16);
        dap = o;  o = align_up(o + (size_t)J * threads * 4, 16);
        kap = o;  o = align_up(o + (curv_on ? (size_t)J * threads * 4 : 0), 16);
        // dense scenes: each (timestep slot, thread)'s window start of the previous iteration
        kix = o;  o = align_up(o + (n_obs >= 2 * SORT_MIN_PAIRS ? (size_t)J * threads * 2 : 0), 16);
        // the CTA's per-iteration residual maxima (float bits), flushed to the global table once
        itm = o;  o = align_up(o + (size_t)max_iters * 4, 16);
        hlp = o;  o = align_up(o + (help > 0 ? (size_t)32 * HSTR * 4 : 0), 16);   // one slot per helper lane
        // help > 0: each sample warp's 32 x 24 partial sums for the shared-memory column reduction
        red = o;  o = align_up(o + (help > 0 ? (size_t)s_cta * 32 * RSTR * 4 : 0), 16);
        total = o;
    }
    // per-sample scratch: u (24 doubles) | c32 (24 floats) | lambda-state l (24 doubles) | first-step
    // correction (24 doubles) | pad -> 196 words (== 4 mod 32 banks: conflict-free LDS.128 across samples)
    static constexpr int SCR_BYTES = 784;
};

__device__ __forceinline__ float interp_table(float x, const float* xs, const float* ks, int n) {
    // np.interp semantics (pkg/constraints.py:67-72): clamp to the end values outside [xs0, xs_{n-1}].
    if (x != x) return x;
    if (x <= xs[0]) return ks[0];
    if (x >= xs[n - 1]) return ks[n - 1];
    int lo = 0, hi = n - 1;
    while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (xs[mid] <= x) lo = mid; else hi = mid;
    }
    const float slope = (ks[lo + 1] - ks[lo]) / (xs[lo + 1] - xs[lo]);
    return ks[lo] + slope * (x - xs[lo]);
}

// Recursive-halving reduce-scatter over the P lanes of a group: afterwards slot
// P*j of lane p holds the group sum of value index p + P*j.
template <int P, int NV>
__device__ __forceinline__ void group_reduce_scatter(float (&v)[NV], int lane) {
#pragma unroll
    for (int o = P / 2; o >= 1; o >>= 1) {
        const bool hi = (lane & o) != 0;
#pragma unroll
        for (int k = 0; k < NV; ++k) {
            if ((k & (P - 1) & ~(o - 1)) != 0) continue;
            const float keep = hi ? v[k | o] : v[k];
            const float send = hi ? v[k] : v[k | o];
            v[k] = keep + __shfl_xor_sync(0xffffffffu, send, o);
        }
    }
}

// One sweep over this lane's timesteps at the current coefficients cxy[k] = (c_x[k], c_y[k]):
// forward evaluation, polar split + coupled clips, back-projection of the residuals
// (v[2k] = g_x[k], v[2k+1] = g_y[k]), the direct residual (v[22]) and the upper cost (v[23]).
// The x/y pairs run as packed fp32x2 (FFMA2 with the basis value broadcast).
constexpr int SORT_MAX_OBS = 256;     // the 4-ary window search reaches k <= 255
constexpr int SCAN_W = 2;             // sorted-window scan: candidates loaded per step

#ifndef BD_AM_OBS_EARLY
#define BD_AM_OBS_EARLY 1
#endif


template <int P, bool CURV, bool INIT, int NV, int MT, int NPT, int TPB>
__device__ __forceinline__ void sweep(const float* __restrict__ wsm, const float4* __restrict__ osm,
                                      const float* __restrict__ csm, const float2 (&cxy)[NC], float (&v)[NV],
                                      float* dap, float* kap, unsigned short* kix, int dstride_rt, int p, int m_rt,
                                      int npair_rt,
                                      int n_curv, const SceneLim& L, int& conf, bool sorted_rt,
                                      bool want_cost = true) {
    // MT / NPT / TPB > 0: timesteps, obstacle pairs and CTA size fixed at compile time (the
    // BASELINE shapes), so the tile addressing folds into immediates and the pair loop unrolls.
    const int m = MT ? MT : m_rt;
    const int npair = NPT ? NPT : npair_rt;
    const int dstride = TPB ? TPB : dstride_rt;
    // dense scenes: obstacles of a timestep sorted by -x/a, only the window |X/a - x_o/a| < 1 is
    // visited (binary search + short scan) instead of every obstacle
    const bool sorted = NPT ? (NPT >= SORT_MIN_PAIRS) : sorted_rt;
#pragma unroll
    for (int k = 0; k < NV; ++k) v[k] = 0.f;
    int j = 0;
    for (int t = p; t < m; t += P, ++j) {
        float w[WROW];
        const float4* wr = reinterpret_cast<const float4*>(wsm + t * WROW);
#pragma unroll
        for (int q = 0; q < WROW / 4; ++q) {
            const float4 f = wr[q];
            w[4 * q] = f.x; w[4 * q + 1] = f.y; w[4 * q + 2] = f.z; w[4 * q + 3] = f.w;
        }
        // forward (X, Y) = W c, (Xd, Yd) = Wd c, (Xdd, Ydd) = Wdd c (pkg/projection.py:295)
        float2 P0 = make_float2(0.f, 0.f), P1 = P0, P2 = P0;
        const float4* op = osm + t * npair;          // (-x0, -x1, -y0, -y1) / (a, a, b, b)
        float qmin = 3.0e38f;
#if BD_AM_OBS_EARLY
        if (NPT > 0 && NPT < SORT_MIN_PAIRS) {
            // position first, then the obstacle-distance pass interleaved with the derivative
            // chains so the tile's shared-memory latency hides behind them
#pragma unroll
            for (int k = 0; k < NC; ++k) P0 = ffma2(w[k], cxy[k], P0);
            float4 ob[NPT > 0 ? NPT : 1];
#pragma unroll
            for (int o = 0; o < NPT; ++o) ob[o] = op[o];
#pragma unroll
            for (int k = 0; k < NC; ++k) {
                P1 = ffma2(w[NC + k], cxy[k], P1);
                P2 = ffma2(w[2 * NC + k], cxy[k], P2);
            }
            const float xs0 = P0.x * L.inv_a, ys0 = P0.y * L.inv_b;
#pragma unroll
            for (int o = 0; o < NPT; ++o) {
                const float2 wc = fadd2(make_float2(xs0, xs0), make_float2(ob[o].x, ob[o].y));
                const float2 ws = fadd2(make_float2(ys0, ys0), make_float2(ob[o].z, ob[o].w));
                const float2 q = ffma2(wc, wc, fmul2(ws, ws));
                qmin = fminf(qmin, fminf(q.x, q.y));
            }
        } else
#endif
        {
#pragma unroll
            for (int k = 0; k < NC; ++k) {
                P0 = ffma2(w[k], cxy[k], P0);
                P1 = ffma2(w[NC + k], cxy[k], P1);
                P2 = ffma2(w[2 * NC + k], cxy[k], P2);
            }
        }
        const float X = P0.x, Y = P0.y, XD = P1.x, YD = P1.y, XDD = P2.x, YDD = P2.y;
        // velocity / acceleration polar split (pkg/projection.py:119-122) in unit-vector form
        const float dv2 = fmaf(XD, XD, YD * YD);
        const float da2 = fmaf(XDD, XDD, YDD * YDD);
        const float iv = dv2 > 0.f ? rsqrtf(dv2) : 0.f;
        const float ia = da2 > 0.f ? rsqrtf(da2) : 0.f;
        const float dv = dv2 * iv, da = da2 * ia;
        // |sin(alpha_a - alpha_v)| = |a x v| / (|a| |v|); a zero vector has angle 0 (atan2(0, 0)),
        // i.e. unit vector (1, 0): |sin| = |y| / |.| of the other vector.  The cross product is
        // shared with the curvature residual below.
        const float cross = fabsf(fmaf(YDD, XD, -XDD * YD));
        // written as selects (a nested ternary compiled to a divergent branch): da2 == 0 makes
        // cross == 0, dv2 == 0 makes iv == 0
        const float gv = (da2 > 0.f ? cross : fabsf(YD)) * iv;
        const float gva = gv * ia;
        const float gap = dv2 > 0.f ? (da2 > 0.f ? gva : gv) : fabsf(YDD) * ia;
        const float cv = dv2 > 0.f ? XD * iv : 1.f;                   // cos(alpha_v), curvature bound only
        // coupled clip window (pkg/projection.py:138-169)
        const int di = j * dstride;
        BD_CHECK(j < (m + P - 1) / P && t < m);
        const float da_prev = INIT ? fminf(fmaxf(da, 0.f), L.a_max) : dap[di];
        float vhi = L.v_max;
        float kcur = 0.f;
        if (CURV) {
            kcur = fabsf(interp_table(X, csm, csm + n_curv, n_curv));
            const float kuse = INIT ? kcur : kap[di];
            const float cent = kuse * cv * cv;
            if (cent > 1e-12f) vhi = fminf(L.v_max, sqrtf(L.c_max / cent));
            kap[di] = kcur;
        }
        const float vlo = fmaxf(L.v_min, sqrtf(da_prev * gap * L.inv_k_max));
        conf += (vlo > vhi) ? 1 : 0;
        const float dvc = fminf(fmaxf(dv, fminf(vlo, vhi)), vhi);
        const float ahi = fminf(L.a_max, __fdividef(dvc * dvc * L.k_max, fmaxf(gap, 1e-8f)));
        const float dac = fminf(fmaxf(da, 0.f), ahi);
        dap[di] = dac;
        // residuals F c - h of the velocity / acceleration blocks (pkg/projection.py:312-315)
        float2 rv, ra;
        if (dv2 > 0.f) rv = fmul2(make_float2((dv - dvc) * iv, (dv - dvc) * iv), P1);
        else rv = make_float2(-dvc, 0.f);
        if (da2 > 0.f) ra = fmul2(make_float2((da - dac) * ia, (da - dac) * ia), P2);
        else ra = make_float2(-dac, 0.f);
        // obstacle block (pkg/projection.py:316-322) + clearance violation (pkg/constraints.py:116-120).
        // Common path: branch-free min of the normalised squared distances over this timestep's
        // tile row, two obstacles per LDS.128 / FADD2 / FFMA2; only a lane inside some ellipse
        // (q < 1) takes the exact per-obstacle path.
        const float xs = X * L.inv_a, ys = Y * L.inv_b;
        float rox = 0.f, roy = 0.f, coll = 0.f;
#pragma unroll 5
        for (int o = 0; o < ((BD_AM_OBS_EARLY && NPT > 0) || sorted ? 0 : npair); ++o) {
            const float4 ob = op[o];
            const float2 wc = fadd2(make_float2(xs, xs), make_float2(ob.x, ob.y));
            const float2 ws = fadd2(make_float2(ys, ys), make_float2(ob.z, ob.w));
            const float2 q = ffma2(wc, wc, fmul2(ws, ws));
            qmin = fminf(qmin, fminf(q.x, q.y));
        }
        if (sorted) {
            const float2* row = reinterpret_cast<const float2*>(osm) + (size_t)t * 2 * npair;
            const int nob = 2 * npair;
            // rounding-safe window: every obstacle with |fl(xs + ox')| < 1 lies strictly inside
            const float win = 1.0f + fmaf(4e-6f, fabsf(xs), 1e-5f);
            const float lo_key = -xs - win, hi_key = -xs + win;
            int k = 0;
            bool hit = false;
            if (!INIT) {
                // last iteration's window start is usually still right: two independent checks
                const int k0 = kix[di];
                const bool okl = k0 == 0 || row[max(k0 - 1, 0)].x <= lo_key;
                const bool okr = k0 >= nob || row[min(k0, nob - 1)].x > lo_key;
                hit = okl && okr;
                k = hit ? k0 : 0;
            }
            if (!hit) {
                // 4-ary search: k = #keys <= lo_key, three independent loads per level (strides 64,
                // 16, 4, 1 reach k <= 255); a binary search waited on one dependent load per level
#pragma unroll
                for (int stride = 64; stride > 0; stride >>= 2) {
                    int cnt = 0;
#pragma unroll
                    for (int u = 1; u < 4; ++u) {
                        const int idx = k + u * stride - 1;
                        cnt += (idx < nob && row[min(idx, nob - 1)].x <= lo_key) ? 1 : 0;
                    }
                    k += cnt * stride;
                }
            }
            kix[di] = (unsigned short)k;
            // SCAN_W candidates per step, loaded together (rows are sorted, so "inside the window"
            // holds for a prefix of them); same obstacle order as a one-by-one scan, which waited
            // on one dependent load per obstacle (2 per step: dense launch 2.31 -> 2.09 ms)
            for (; k < nob; k += SCAN_W) {
                float2 ob[SCAN_W];
#pragma unroll
                for (int u = 0; u < SCAN_W; ++u) ob[u] = row[min(k + u, nob - 1)];
                bool inside = true;
#pragma unroll
                for (int u = 0; u < SCAN_W; ++u) {
                    inside = inside && (k + u < nob) && (ob[u].x < hi_key);
                    const float wc = xs + ob[u].x, ws = ys + ob[u].y;
                    const float q = fmaf(wc, wc, ws * ws);
                    if (inside && q < 1.f) {
                        coll += 1.f - q;
                        if (q > 0.f) {
                            const float f = 1.f - rsqrtf(q);
                            rox = fmaf(wc, f, rox);
                            roy = fmaf(ws, f, roy);
                        } else {
                            rox -= 1.f;
                        }
                    }
                }
                if (!inside) break;
            }
        } else if (qmin < 1.f) {
            for (int o = 0; o < npair; ++o) {
                const float4 ob = op[o];
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const float wc = xs + (h ? ob.y : ob.x), ws = ys + (h ? ob.w : ob.z);
                    const float q = fmaf(wc, wc, ws * ws);
                    if (q < 1.f) {
                        coll += 1.f - q;
                        if (q > 0.f) {
                            const float f = 1.f - rsqrtf(q);
                            rox = fmaf(wc, f, rox);
                            roy = fmaf(ws, f, roy);
                        } else {
                            rox -= 1.f;            // atan2(0,0) = 0: h - X = (a, 0)
                        }
                    }
                }
            }
        }
        // lane slack residual (pkg/projection.py:308-310,323)
        const float up = fmaxf(Y - L.y_ub, 0.f), lo = fmaxf(L.y_lb - Y, 0.f);
        const float2 ro = make_float2(L.a * rox, fmaf(L.b, roy, up - lo));
        // back-projection g += Wd^T r_v + Wdd^T r_a + W^T r_o (+ lane); the basis row is re-read
        // from shared memory rather than held across the clip/obstacle section (register budget)
#pragma unroll
        for (int q = 0; q < WROW / 4; ++q) {
            const float4 f = wr[q];
            w[4 * q] = f.x; w[4 * q + 1] = f.y; w[4 * q + 2] = f.z; w[4 * q + 3] = f.w;
        }
#pragma unroll
        for (int k = 0; k < NC; ++k) {
            float2 g = make_float2(v[2 * k], v[2 * k + 1]);
            g = ffma2(w[NC + k], rv, g);
            g = ffma2(w[2 * NC + k], ra, g);
            g = ffma2(w[k], ro, g);
            v[2 * k] = g.x;
            v[2 * k + 1] = g.y;
        }
        if (!INIT) {
            // direct violations (pkg/constraints.py:124-138) and speed cost (pkg/bilevel.py:125-126)
            float r = coll + up + lo;
            r += fmaxf(dv - L.v_max, 0.f) + fmaxf(L.v_min - dv, 0.f);
            r += fmaxf(da - L.a_max, 0.f);
            const float sp = fmaxf(dv, 1e-6f);
            r += fmaxf(__fdividef(cross, sp * sp * sp) - L.k_max, 0.f);
            if (CURV) r += fmaxf(XD * XD * kcur - L.c_max, 0.f);
            v[NX] += r;
            if (want_cost) {                        // only the final iterate's cost is reported
                const float e = dv - L.v_max;
                v[NX + 1] = fmaf(e, e, v[NX + 1]);
            }
        }
    }
}

// Latency instance (P = 32, one CTA of 5-8 one-warp samples per SM, up to 255 registers; m and the
// obstacle pairs fixed at compile time, no curvature, unsorted tile): the same per-timestep arithmetic
// as sweep(), reorganised into three phases, each unrolled over the lane's JM timestep slots so the
// scheduler overlaps their independent dependency chains instead of running one slot after another:
//   A  forward X / Xd / Xdd, obstacle filter, polar split, coupled clips (branch-free);
//   B  the exact obstacle path for the rare slots inside some ellipse;
//   C  back-projection, direct residual and cost, accumulated in timestep order as sweep() does.
// A slot past m (only the last, on lanes p >= m - (JM-1)P) is evaluated on a clamped timestep and
// contributes exact zeros.
#ifndef BD_LAT_CH
#define BD_LAT_CH 1      // A/B on B200 (B = 1000, P = 32, round 2): 1 slot 0.213 ms, 2: 0.221 (round 1: 2 0.229, 3 0.246, 4 0.251)
#endif
#ifndef BD_LAT_CH_H
#define BD_LAT_CH_H 1    // with the remainder warp (3 full slots): 1 slot 0.201 ms, 2: 0.220, 3: 0.226
#endif
template <int P, bool INIT, int NV, int MT, int NPT, int TPB, bool HELPED = false>
__device__ __forceinline__ void sweep_lat(const float* __restrict__ wsm, const float4* __restrict__ osm,
                                          const float2 (&cxy)[NC], float (&v)[NV], float* dap, int p,
                                          const SceneLim& L, int& conf, bool want_cost) {
    // HELPED: only the full slots; the remainder warp (am_helper) evaluates the last MT mod P timesteps
    constexpr int JM = HELPED ? MT / P : (MT + P - 1) / P;
    constexpr int CHM = HELPED ? BD_LAT_CH_H : BD_LAT_CH;
    constexpr int CH = JM > CHM ? CHM : JM;                 // slots per phase group (register budget)
#pragma unroll
    for (int k = 0; k < NV; ++k) v[k] = 0.f;
#pragma unroll
    for (int j0 = 0; j0 < JM; j0 += CH) {
    float X[CH], Y[CH], qm[CH], dvs[CH], das[CH], crs[CH];
    float2 rv[CH], ra[CH];
    // ---- phase A
#pragma unroll
    for (int jj = 0; jj < CH; ++jj) {
        const int j = j0 + jj;
        const bool valid = j < JM && (HELPED || (MT % P == 0) || j + 1 < JM || p + j * P < MT);
        const int t = valid ? p + j * P : MT - 1;
        float w[WROW];
        const float4* wr = reinterpret_cast<const float4*>(wsm + t * WROW);
#pragma unroll
        for (int q = 0; q < WROW / 4; ++q) {
            const float4 f = wr[q];
            w[4 * q] = f.x; w[4 * q + 1] = f.y; w[4 * q + 2] = f.z; w[4 * q + 3] = f.w;
        }
        float2 P0 = make_float2(0.f, 0.f), P1 = P0, P2 = P0;
#pragma unroll
        for (int k = 0; k < NC; ++k) P0 = ffma2(w[k], cxy[k], P0);
        const float4* op = osm + t * NPT;
        float4 ob[NPT];
#pragma unroll
        for (int o = 0; o < NPT; ++o) ob[o] = op[o];
#pragma unroll
        for (int k = 0; k < NC; ++k) {
            P1 = ffma2(w[NC + k], cxy[k], P1);
            P2 = ffma2(w[2 * NC + k], cxy[k], P2);
        }
        const float xs0 = P0.x * L.inv_a, ys0 = P0.y * L.inv_b;
        float qmin = 3.0e38f;
#pragma unroll
        for (int o = 0; o < NPT; ++o) {
            const float2 wc = fadd2(make_float2(xs0, xs0), make_float2(ob[o].x, ob[o].y));
            const float2 ws = fadd2(make_float2(ys0, ys0), make_float2(ob[o].z, ob[o].w));
            const float2 q = ffma2(wc, wc, fmul2(ws, ws));
            qmin = fminf(qmin, fminf(q.x, q.y));
        }
        const float XD = P1.x, YD = P1.y, XDD = P2.x, YDD = P2.y;
        const float dv2 = fmaf(XD, XD, YD * YD);
        const float da2 = fmaf(XDD, XDD, YDD * YDD);
        const float iv = dv2 > 0.f ? rsqrtf(dv2) : 0.f;
        const float ia = da2 > 0.f ? rsqrtf(da2) : 0.f;
        const float dv = dv2 * iv, da = da2 * ia;
        const float cross = fabsf(fmaf(YDD, XD, -XDD * YD));
        const float gv = (da2 > 0.f ? cross : fabsf(YD)) * iv;
        const float gva = gv * ia;
        const float gap = dv2 > 0.f ? (da2 > 0.f ? gva : gv) : fabsf(YDD) * ia;
        const int di = min(j, JM - 1) * TPB;
        const float da_prev = INIT ? fminf(fmaxf(da, 0.f), L.a_max) : dap[di];
        const float vhi = L.v_max;
        const float vlo = fmaxf(L.v_min, sqrtf(da_prev * gap * L.inv_k_max));
        conf += (valid && vlo > vhi) ? 1 : 0;
        const float dvc = fminf(fmaxf(dv, fminf(vlo, vhi)), vhi);
        const float ahi = fminf(L.a_max, __fdividef(dvc * dvc * L.k_max, fmaxf(gap, 1e-8f)));
        const float dac = fminf(fmaxf(da, 0.f), ahi);
        if (j < JM) dap[di] = dac;          // (compile-time after unrolling)
        float2 rvj, raj;
        if (dv2 > 0.f) rvj = fmul2(make_float2((dv - dvc) * iv, (dv - dvc) * iv), P1);
        else rvj = make_float2(-dvc, 0.f);
        if (da2 > 0.f) raj = fmul2(make_float2((da - dac) * ia, (da - dac) * ia), P2);
        else raj = make_float2(-dac, 0.f);
        const float2 z2 = make_float2(0.f, 0.f);
        rv[jj] = valid ? rvj : z2;
        ra[jj] = valid ? raj : z2;
        X[jj] = P0.x; Y[jj] = P0.y;
        qm[jj] = valid ? qmin : 3.0e38f;
        dvs[jj] = dv; das[jj] = da; crs[jj] = cross;
    }
    // ---- phase B (rare): exact obstacle residuals of the slots inside some ellipse
    float rox[CH], roy[CH], coll[CH];
#pragma unroll
    for (int jj = 0; jj < CH; ++jj) {
        const int j = j0 + jj;
        rox[jj] = 0.f; roy[jj] = 0.f; coll[jj] = 0.f;
        if (qm[jj] < 1.f) {
            const int t = p + j * P;
            const float4* op = osm + t * NPT;
            const float xs = X[jj] * L.inv_a, ys = Y[jj] * L.inv_b;
            for (int o = 0; o < NPT; ++o) {
                const float4 ob = op[o];
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const float wc = xs + (h ? ob.y : ob.x), ws = ys + (h ? ob.w : ob.z);
                    const float q = fmaf(wc, wc, ws * ws);
                    if (q < 1.f) {
                        coll[jj] += 1.f - q;
                        if (q > 0.f) {
                            const float f = 1.f - rsqrtf(q);
                            rox[jj] = fmaf(wc, f, rox[jj]);
                            roy[jj] = fmaf(ws, f, roy[jj]);
                        } else {
                            rox[jj] -= 1.f;
                        }
                    }
                }
            }
        }
    }
    // ---- phase C: back-projection g += Wd^T r_v + Wdd^T r_a + W^T r_o, direct residual, cost
#pragma unroll
    for (int jj = 0; jj < CH; ++jj) {
        const int j = j0 + jj;
        const bool valid = j < JM && (HELPED || (MT % P == 0) || j + 1 < JM || p + j * P < MT);
        const int t = valid ? p + j * P : MT - 1;
        const float up = fmaxf(Y[jj] - L.y_ub, 0.f), lo = fmaxf(L.y_lb - Y[jj], 0.f);
        const float2 roj = make_float2(L.a * rox[jj], fmaf(L.b, roy[jj], up - lo));
        const float2 ro = valid ? roj : make_float2(0.f, 0.f);
        float w[WROW];
        const float4* wr = reinterpret_cast<const float4*>(wsm + t * WROW);
#pragma unroll
        for (int q = 0; q < WROW / 4; ++q) {
            const float4 f = wr[q];
            w[4 * q] = f.x; w[4 * q + 1] = f.y; w[4 * q + 2] = f.z; w[4 * q + 3] = f.w;
        }
#pragma unroll
        for (int k = 0; k < NC; ++k) {
            float2 g = make_float2(v[2 * k], v[2 * k + 1]);
            g = ffma2(w[NC + k], rv[jj], g);
            g = ffma2(w[2 * NC + k], ra[jj], g);
            g = ffma2(w[k], ro, g);
            v[2 * k] = g.x;
            v[2 * k + 1] = g.y;
        }
        if (!INIT) {
            const float dv = dvs[jj], da = das[jj];
            float r = coll[jj] + up + lo;
            r += fmaxf(dv - L.v_max, 0.f) + fmaxf(L.v_min - dv, 0.f);
            r += fmaxf(da - L.a_max, 0.f);
            const float sp = fmaxf(dv, 1e-6f);
            r += fmaxf(__fdividef(crs[jj], sp * sp * sp) - L.k_max, 0.f);
            v[NX] += valid ? r : 0.f;
            if (want_cost) {
                const float e = dv - L.v_max;
                v[NX + 1] = valid ? fmaf(e, e, v[NX + 1]) : v[NX + 1];
            }
        }
    }
    }
}

#ifndef BD_NO_ITMAX
#define BD_NO_ITMAX 0      // diagnostic builds only: drop the per-iteration batch-max atomics
#endif

__device__ __forceinline__ void named_arrive(int id, int n) {
    asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void named_sync(int id, int n) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

// One timestep t of one sample for the remainder warp: the arithmetic of one sweep_lat slot
// (phases A, B, C), its 22 back-projection partials, direct residual and cost written to out[0..23].
// dap_h carries the timestep's clipped acceleration between iterations, as dap does for a slot.
template <int NPT, bool INIT>
__device__ __forceinline__ void rem_eval(const float* __restrict__ wsm, const float4* __restrict__ osm,
                                         const float* __restrict__ c32, int t, const SceneLim& L, float& dap_h,
                                         int& conf, bool count, bool want_cost, float* out) {
    float2 cxy[NC];
#pragma unroll
    for (int q = 0; q < NC; ++q) cxy[q] = reinterpret_cast<const float2*>(c32)[q];
    float w[WROW];
    const float4* wr = reinterpret_cast<const float4*>(wsm + t * WROW);
#pragma unroll
    for (int q = 0; q < WROW / 4; ++q) {
        const float4 f = wr[q];
        w[4 * q] = f.x; w[4 * q + 1] = f.y; w[4 * q + 2] = f.z; w[4 * q + 3] = f.w;
    }
    float2 P0 = make_float2(0.f, 0.f), P1 = P0, P2 = P0;
#pragma unroll
    for (int k = 0; k < NC; ++k) P0 = ffma2(w[k], cxy[k], P0);
    const float4* op = osm + t * NPT;
    float4 ob[NPT];
#pragma unroll
    for (int o = 0; o < NPT; ++o) ob[o] = op[o];
#pragma unroll
    for (int k = 0; k < NC; ++k) {
        P1 = ffma2(w[NC + k], cxy[k], P1);
        P2 = ffma2(w[2 * NC + k], cxy[k], P2);
    }
    const float xs0 = P0.x * L.inv_a, ys0 = P0.y * L.inv_b;
    float qmin = 3.0e38f;
#pragma unroll
    for (int o = 0; o < NPT; ++o) {
        const float2 wc = fadd2(make_float2(xs0, xs0), make_float2(ob[o].x, ob[o].y));
        const float2 ws = fadd2(make_float2(ys0, ys0), make_float2(ob[o].z, ob[o].w));
        const float2 q = ffma2(wc, wc, fmul2(ws, ws));
        qmin = fminf(qmin, fminf(q.x, q.y));
    }
    const float XD = P1.x, YD = P1.y, XDD = P2.x, YDD = P2.y;
    const float dv2 = fmaf(XD, XD, YD * YD);
    const float da2 = fmaf(XDD, XDD, YDD * YDD);
    const float iv = dv2 > 0.f ? rsqrtf(dv2) : 0.f;
    const float ia = da2 > 0.f ? rsqrtf(da2) : 0.f;
    const float dv = dv2 * iv, da = da2 * ia;
    const float cross = fabsf(fmaf(YDD, XD, -XDD * YD));
    const float gv = (da2 > 0.f ? cross : fabsf(YD)) * iv;
    const float gva = gv * ia;
    const float gap = dv2 > 0.f ? (da2 > 0.f ? gva : gv) : fabsf(YDD) * ia;
    const float da_prev = INIT ? fminf(fmaxf(da, 0.f), L.a_max) : dap_h;
    const float vhi = L.v_max;
    const float vlo = fmaxf(L.v_min, sqrtf(da_prev * gap * L.inv_k_max));
    conf += (count && vlo > vhi) ? 1 : 0;
    const float dvc = fminf(fmaxf(dv, fminf(vlo, vhi)), vhi);
    const float ahi = fminf(L.a_max, __fdividef(dvc * dvc * L.k_max, fmaxf(gap, 1e-8f)));
    const float dac = fminf(fmaxf(da, 0.f), ahi);
    dap_h = dac;
    float2 rv, ra;
    if (dv2 > 0.f) rv = fmul2(make_float2((dv - dvc) * iv, (dv - dvc) * iv), P1);
    else rv = make_float2(-dvc, 0.f);
    if (da2 > 0.f) ra = fmul2(make_float2((da - dac) * ia, (da - dac) * ia), P2);
    else ra = make_float2(-dac, 0.f);
    float rox = 0.f, roy = 0.f, coll = 0.f;
    if (qmin < 1.f) {
        const float xs = P0.x * L.inv_a, ys = P0.y * L.inv_b;
        for (int o = 0; o < NPT; ++o) {
            const float4 obo = op[o];
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const float wc = xs + (h ? obo.y : obo.x), ws = ys + (h ? obo.w : obo.z);
                const float q = fmaf(wc, wc, ws * ws);
                if (q < 1.f) {
                    coll += 1.f - q;
                    if (q > 0.f) {
                        const float f = 1.f - rsqrtf(q);
                        rox = fmaf(wc, f, rox);
                        roy = fmaf(ws, f, roy);
                    } else {
                        rox -= 1.f;
                    }
                }
            }
        }
    }
    const float up = fmaxf(P0.y - L.y_ub, 0.f), lo = fmaxf(L.y_lb - P0.y, 0.f);
    const float2 ro = make_float2(L.a * rox, fmaf(L.b, roy, up - lo));
    float4* o4 = reinterpret_cast<float4*>(out);
    float g[NX + 2];
#pragma unroll
    for (int k = 0; k < NC; ++k) {
        float2 gk = fmul2(make_float2(w[NC + k], w[NC + k]), rv);
        gk = ffma2(w[2 * NC + k], ra, gk);
        gk = ffma2(w[k], ro, gk);
        g[2 * k] = gk.x;
        g[2 * k + 1] = gk.y;
    }
    g[NX] = 0.f;
    g[NX + 1] = 0.f;
    if (!INIT) {
        float r = coll + up + lo;
        r += fmaxf(dv - L.v_max, 0.f) + fmaxf(L.v_min - dv, 0.f);
        r += fmaxf(da - L.a_max, 0.f);
        const float sp = fmaxf(dv, 1e-6f);
        r += fmaxf(__fdividef(cross, sp * sp * sp) - L.k_max, 0.f);
        g[NX] = r;
        if (want_cost) {
            const float e = dv - L.v_max;
            g[NX + 1] = e * e;
        }
    }
#pragma unroll
    for (int q = 0; q < (NX + 2) / 4; ++q) o4[q] = make_float4(g[4 * q], g[4 * q + 1], g[4 * q + 2], g[4 * q + 3]);
}

// The remainder warp of a helped latency CTA (TPB = 32 (SPC + 1)): lane s * HELP + r evaluates
// timestep (MT / 32) * 32 + r of sample slot s every iteration, between the two CTA barriers the
// sample warps pass around their sweep (coefficients in shared memory -> barrier -> remainder
// timesteps -> barrier -> the sample warp adds the HELP partials after its reduce-scatter).  The
// sample warps then sweep 3 full slots instead of 3 + a 4-of-32-lane one (m = 100).  Mirrors
// am_samples' CTA barriers one for one, including the per-iteration-maxima table's.
template <int NPT, int MT, int TPB, int HELP>
__device__ __forceinline__ void am_helper(const AmArgs& a, int scene, int cta, int iters, unsigned char* smem) {
    constexpr int SPC = TPB / 32 - 1;
    static_assert(SPC * HELP <= 32, "remainder warp: one lane per (sample, remainder timestep)");
    const AmSmem lay(a.m, a.n_obs, a.neq, a.n_curv, a.s_cta, blockDim.x, 32, false, a.max_iters, HELP);
    const float* wsm = reinterpret_cast<const float*>(smem + lay.w);
    const float4* osm = reinterpret_cast<const float4*>(smem + lay.obs);
    const int lane = threadIdx.x & 31;
    const bool live = lane < SPC * HELP;
    const int s = live ? lane / HELP : SPC - 1;
    const int t = (MT / 32) * 32 + lane % HELP;
    const bool count = live && cta * a.s_cta + s < a.B;
    const float* c32 = reinterpret_cast<const float*>(smem + lay.scr + (size_t)s * AmSmem::SCR_BYTES + 192);
    float* out = reinterpret_cast<float*>(smem + lay.hlp) + lane * AmSmem::HSTR;
    const SceneLim L = a.lim[scene];
    float dap_h = 0.f;
    int conf = 0;
    float* dst = out;                                       // idle lanes write their own (unread) slot
    // named barriers: 1 = every sample's coefficients staged (samples arrive, this warp waits);
    // 2 + s = the partials of sample s published (this warp arrives, sample s waits) -- a sample
    // never waits for the other samples, only for the partials it needs
    auto publish = [&]() {
#pragma unroll
        for (int k = 0; k < SPC; ++k) named_arrive(2 + k, 64);
    };
    named_sync(1, TPB);
    rem_eval<NPT, true>(wsm, osm, c32, t, L, dap_h, conf, count, true, dst);
    publish();
    const bool record = a.replay == nullptr && !BD_NO_ITMAX;
    unsigned* itm_s = reinterpret_cast<unsigned*>(smem + lay.itm);
    if (record) {
        for (int k = threadIdx.x; k < iters; k += blockDim.x) itm_s[k] = 0u;
        __syncthreads();
    }
    for (int it = 0; it < iters; ++it) {
        named_sync(1, TPB);
        rem_eval<NPT, false>(wsm, osm, c32, t, L, dap_h, conf, count, it == iters - 1, dst);
        publish();
    }
    if (record) {
        __syncthreads();
        unsigned* itm = a.itmax + (size_t)scene * a.max_iters * ITMAX_SLOTS + (cta % ITMAX_SLOTS);
        for (int k = threadIdx.x; k < iters; k += blockDim.x)
            if (const unsigned v = itm_s[k]) atomicMax(itm + (size_t)k * ITMAX_SLOTS, v);
    }
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) conf += __shfl_xor_sync(0xffffffffu, conf, o);
    if (lane == 0 && conf) atomicAdd(a.conflicts + scene, (unsigned long long)conf);
}

// The all-gather fused into the epilogue: one value into every rank's symmetric buffer
// (kept out of line so the main loop's register allocation does not see it).
__device__ __noinline__ void p2p_store_all(void* const* bufs, int world, size_t off, long long row, double val) {
    for (int g = 0; g < world; ++g) reinterpret_cast<double*>(static_cast<char*>(bufs[g]) + off)[row] = val;
}

// Pair barrier of the two warps that share a sample when P == 64 (named barriers 1..4).
__device__ __forceinline__ void pair_sync() {
    asm volatile("bar.sync %0, 64;" ::"r"(1 + (int)(threadIdx.x >> 6)) : "memory");
}

#ifndef BD_AM_MINB
#define BD_AM_MINB 2       // x 256 threads: 128 registers per thread
#endif
// Stage the basis rows and the scene's obstacle tile (TMA bulk copies on one mbarrier) and the
// fp64 K blocks (threads) in shared memory; returns after a CTA barrier.
template <int P, bool CURV>
__device__ __forceinline__ void am_stage(const AmArgs& a, int scene, unsigned char* smem, uint64_t* stage_bar) {
    const int m = a.m, neq = a.neq, n_obs = a.n_obs;
    const int threads = blockDim.x;
    const AmSmem lay(m, n_obs, neq, a.n_curv, a.s_cta, threads, P, CURV, a.max_iters);
    float* wsm = reinterpret_cast<float*>(smem + lay.w);
    float4* osm = reinterpret_cast<float4*>(smem + lay.obs);
    double* ksm = reinterpret_cast<double*>(smem + lay.k);
    double* kbsm = reinterpret_cast<double*>(smem + lay.kb);
    double* asm_ = reinterpret_cast<double*>(smem + lay.a);
    float* csm = reinterpret_cast<float*>(smem + lay.curv);
    // ---- stage constants and the scene tile once per CTA: the basis rows and this scene's
    //      obstacle tile arrive by TMA bulk copy (one mbarrier), the small fp64 blocks by the threads
    const uint32_t w_bytes = (uint32_t)m * WROW * 4, o_bytes = (uint32_t)(n_obs / 2) * m * 16;
    if (threadIdx.x == 0) {
        mbar_init(stage_bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        mbar_expect_tx(stage_bar, w_bytes + o_bytes);
        bulk_load(wsm, a.wrow, w_bytes, stage_bar);
        if (o_bytes) bulk_load(osm, reinterpret_cast<const float4*>(a.obs) + (size_t)scene * (n_obs / 2) * m, o_bytes,
                               stage_bar);
    }
    for (int i = threadIdx.x; i < NX * KSTR; i += threads) ksm[i] = a.kblk[i];
    for (int i = threadIdx.x; i < NX * neq; i += threads) { kbsm[i] = a.kb[i]; asm_[i] = a.aeq[i]; }
    if (CURV)
        for (int i = threadIdx.x; i < 2 * a.n_curv; i += threads) csm[i] = a.curv[(size_t)scene * 2 * a.n_curv + i];
    mbar_wait(stage_bar, 0);
    __syncthreads();
}

// AM iterations for the samples of CTA `blk` of `scene` (constants already staged): prologue,
// `iters` iterations, outputs, conflict / error atomics.
template <int P, bool CURV, int MT, int NPT, int TPB, bool LAT, int HELP = 0>
__device__ __forceinline__ void am_samples(const AmArgs& a, int scene, int blk, int iters, unsigned char* smem) {
    constexpr bool LAT32 = LAT && P <= 32 && MT > 0 && NPT > 0 && NPT < SORT_MIN_PAIRS && !CURV;
    // HELP > 0: the last warp of the CTA is the remainder warp (am_helper); the others sweep full slots
    constexpr bool HELPED = LAT32 && P == 32 && HELP > 0;
    static_assert(HELP == 0 || (HELPED && HELP == MT % 32), "remainder warp: latency instance, MT mod 32 timesteps");
    if constexpr (HELPED) {
        if ((int)(threadIdx.x >> 5) == TPB / 32 - 1) {
            am_helper<NPT, MT, TPB, HELP>(a, scene, blk < 0 ? (int)blockIdx.x : blk, iters, smem);
            return;
        }
    }
    constexpr bool PAIR = (P == 64);
    constexpr int RP = PAIR ? 32 : P;                // reduction width / ownership stride
    constexpr int NV = ((NX + 2 + RP - 1) / RP) * RP;   // 22 back-projections + residual + cost, padded
    constexpr int ROWS = (NX + RP - 1) / RP;         // coefficient rows owned per lane
    const int m = a.m, neq = a.neq, n_obs = a.n_obs;
    const int threads = blockDim.x;
    const AmSmem lay(m, n_obs, neq, a.n_curv, a.s_cta, threads, P, CURV, a.max_iters, HELPED ? HELP : 0);
    float* wsm = reinterpret_cast<float*>(smem + lay.w);
    float4* osm = reinterpret_cast<float4*>(smem + lay.obs);
    double* ksm = reinterpret_cast<double*>(smem + lay.k);
    double* kbsm = reinterpret_cast<double*>(smem + lay.kb);
    double* asm_ = reinterpret_cast<double*>(smem + lay.a);
    float* csm = reinterpret_cast<float*>(smem + lay.curv);
    const int lane = threadIdx.x & 31;
    const int p = PAIR ? (int)(threadIdx.x % 64) : lane % P;        // timestep lane within the sample
    const int own = PAIR ? ((threadIdx.x & 32) ? 64 : lane) : p;     // ownership index (>= NX: none)
    auto gsync = [&]() { if (PAIR) pair_sync(); else __syncwarp(); };
    const int slot = threadIdx.x / P;
    const int local = (blk < 0 ? (int)blockIdx.x : blk) * a.s_cta + slot;
    const bool active = local < a.B;
    const size_t row = (size_t)scene * a.B + (active ? local : a.B - 1);
    double* su = reinterpret_cast<double*>(smem + lay.scr + (size_t)slot * AmSmem::SCR_BYTES);
    float* sc = reinterpret_cast<float*>(su + 24);
    float* dap = reinterpret_cast<float*>(smem + lay.dap) + threadIdx.x;
    float* kap = reinterpret_cast<float*>(smem + lay.kap) + threadIdx.x;
    unsigned short* kix = reinterpret_cast<unsigned short*>(smem + lay.kix) + threadIdx.x;
    const SceneLim L = a.lim[scene];
    const double rho = a.rho;

    // ---- prologue: xi_bar, equality residual correction delta = K_b (b - A xi_bar)
    for (int k = p; k < NX; k += P) su[k] = a.xi_bar[row * NX + k];
    gsync();
    double eb[MAX_NEQ];
    const double* brow = a.b ? a.b + row * neq : a.bscene + (size_t)scene * neq;
    for (int e = 0; e < neq; ++e) {
        double s = brow[e];
        for (int i = 0; i < NX; ++i) s = fma(-asm_[e * NX + i], su[i], s);
        eb[e] = s;
    }
    // value index i (0..21) <-> coefficient (axis i&1, kk = i>>1), state index ks = axis*NC + kk
    double c[ROWS];
    double* ell = su + 36;          // l = xi_bar + lambda, owned rows only (no cross-lane traffic)
    double* dl = su + 60;           // K_b (b - A xi_bar), used by the first update only
#pragma unroll
    for (int r = 0; r < ROWS; ++r) {
        const int i = own + RP * r;
        c[r] = 0.0;
        if (i < NX) {
            const int ks = (i & 1) * NC + (i >> 1);
            c[r] = su[ks];
            ell[ks] = c[r];
            double s = 0.0;
            for (int e = 0; e < neq; ++e) s = fma(kbsm[ks * neq + e], eb[e], s);
            dl[ks] = s;
            sc[i] = static_cast<float>(c[r]);
        }
    }
    // A sample whose iterate leaves the fp32 range of the sweep (Bernstein rows are a partition of
    // unity, so |X| <= max|c|, |Xd| <= 4 max|c|, |Xdd| <= 15 max|c|; below 1e17 every square stays
    // < 3e38) is marked out of range (`ovf`, sticky); its later non-finite values are not a batch
    // failure, and it reports an infinite residual and cost with its stage-1 coefficients: it ranks
    // after every finite sample, as the reference's huge / NaN residuals do for such set-points.
    bool ovf = false;
#pragma unroll
    for (int r = 0; r < ROWS; ++r)
        if (own + RP * r < NX) ovf |= !(fabs(c[r]) < 1e17);
    gsync();
    float2 cxy[NC];
#pragma unroll
    for (int q = 0; q < NC; ++q) cxy[q] = reinterpret_cast<const float2*>(sc)[q];

    int conf = 0;
    bool bad = false;
    float v[NV];
    float* xbuf = reinterpret_cast<float*>(smem + lay.scr + (size_t)slot * AmSmem::SCR_BYTES + 672);
    const float* hsm = reinterpret_cast<const float*>(smem + lay.hlp) + slot * HELP * AmSmem::HSTR + lane;
    float* rbuf = reinterpret_cast<float*>(smem + lay.red) + (size_t)slot * 32 * AmSmem::RSTR;
    auto reduce = [&]() {
        if constexpr (HELPED && NV == 32) {
            // column sums through shared memory: every lane stores its 24 partials as a row, lane j
            // adds column j over the 32 rows (independent loads, a 5-level add tree) -- a shorter
            // dependency chain than the 5-stage shuffle reduce-scatter, which held ~20 % of the
            // warps' stall samples (profiles/r02/am_kernel_lat32_help_v2)
            float4* rw = reinterpret_cast<float4*>(rbuf + lane * AmSmem::RSTR);
#pragma unroll
            for (int q = 0; q < (NX + 2) / 4; ++q) rw[q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
            __syncwarp();
            const int col = lane < NX + 2 ? lane : 0;
            float t[32];
#pragma unroll
            for (int l = 0; l < 32; ++l) t[l] = rbuf[l * AmSmem::RSTR + col];
#pragma unroll
            for (int h = 16; h >= 1; h >>= 1)
#pragma unroll
                for (int l = 0; l < h; ++l) t[l] += t[l + h];
            v[0] = t[0];
            __syncwarp();
        } else {
            group_reduce_scatter<RP>(v, lane);
        }
        if (PAIR) {                                   // second warp -> first warp partial sums
            if ((threadIdx.x & 32) && lane < NX + 2) xbuf[lane] = v[0];
            pair_sync();
            if (!(threadIdx.x & 32) && lane < NX + 2) v[0] += xbuf[lane];
        }
        if constexpr (HELPED) {                       // the remainder warp's timesteps of this sample
            named_sync(2 + slot, 64);
            if (lane < NX + 2) {
                float h = hsm[0];
#pragma unroll
                for (int r = 1; r < HELP; ++r) h += hsm[r * AmSmem::HSTR];
                v[0] += h;
            }
        }
    };
    if constexpr (HELPED) named_arrive(1, TPB);      // this sample's coefficients staged (am_helper)
    if constexpr (LAT32)
        sweep_lat<P, true, NV, MT, NPT, TPB, HELPED>(wsm, osm, cxy, v, dap, p, L, conf, true);
    else
        sweep<P, CURV, true, NV, MT, NPT, TPB>(wsm, osm, csm, cxy, v, dap, kap, kix, threads, p, m, n_obs / 2,
                                               a.n_curv, L, conf, a.sorted != 0);
    reduce();

    const int r_lane = NX % RP, r_slot = (NX / RP) * RP;
    const int c_lane = (NX + 1) % RP, c_slot = ((NX + 1) / RP) * RP;
    float resid = 0.f, cost = 0.f;
    const int cta = blk < 0 ? (int)blockIdx.x : blk;
    // per-iteration batch maxima: shared-memory atomics during the loop, one global atomic per
    // (CTA, iteration) afterwards (per-iteration global atomics cost 8 % of the latency launch)
    unsigned* itm_s = reinterpret_cast<unsigned*>(smem + lay.itm);
    const bool record = a.replay == nullptr && !BD_NO_ITMAX;
    if (record) {
        for (int t = threadIdx.x; t < iters; t += threads) itm_s[t] = 0u;
        __syncthreads();
    }

    for (int it = 0; it < iters; ++it) {
        // ---- coefficient update: lambda step, then c <- c + K (l - c - rho g) (+ delta on the first step)
        const bool first = (it == 0);
#pragma unroll
        for (int r = 0; r < ROWS; ++r) {
            const int i = own + RP * r;
            if (i < NX) {
                const int ax = i & 1, kk = i >> 1, ks = ax * NC + kk;
                const double g = static_cast<double>(v[P * r]);
                double l = ell[ks];
                if (!first) {
                    l = fma(-0.5 * rho, g, l);
                    ell[ks] = l;
                }
                su[ax * KROW + kk] = l - c[r] - rho * g;   // per-axis stride 12 (16-B aligned)
            }
        }
        gsync();
#pragma unroll
        for (int r = 0; r < ROWS; ++r) {
            const int i = own + RP * r;
            if (i < NX) {
                const int ax = i & 1, kk = i >> 1;
                const double2* kr = reinterpret_cast<const double2*>(ksm + i * KSTR);
                const double2* ur = reinterpret_cast<const double2*>(su + ax * KROW);
                double s0 = first ? dl[ax * NC + kk] : 0.0, s1 = 0.0;
#pragma unroll
                for (int q = 0; q < NC / 2; ++q) {
                    const double2 kq = kr[q];
                    const double2 uq = ur[q];
                    s0 = fma(kq.x, uq.x, s0);
                    s1 = fma(kq.y, uq.y, s1);
                }
                s0 = fma(kr[NC / 2].x, su[ax * KROW + NC - 1], s0);
                c[r] += s0 + s1;
                const double ac = fabs(c[r]);
                bad |= !(ac <= DBL_MAX);                      // NaN / inf (pkg/projection.py:290-291)
                ovf |= (ac >= 1e17) && (ac <= DBL_MAX);
                sc[i] = static_cast<float>(c[r]);
            }
        }
        gsync();
#pragma unroll
        for (int q = 0; q < NC; ++q) cxy[q] = reinterpret_cast<const float2*>(sc)[q];
        // ---- projections, back-projection, residual at the new iterate
        if constexpr (HELPED) named_arrive(1, TPB);
        if constexpr (LAT32)
            sweep_lat<P, false, NV, MT, NPT, TPB, HELPED>(wsm, osm, cxy, v, dap, p, L, conf, it == iters - 1);
        else
            sweep<P, CURV, false, NV, MT, NPT, TPB>(wsm, osm, csm, cxy, v, dap, kap, kix, threads, p, m, n_obs / 2,
                                                    a.n_curv, L, conf, a.sorted != 0, it == iters - 1);   // cost: last sweep only
        reduce();
        resid = v[r_slot];
        cost = v[c_slot];
        // ---- residual history + batch max for the batch-global early exit (pkg/projection.py:327-330)
        const bool owner = (own == r_lane);
        if (a.hist_out && owner && active)
            a.hist_out[((size_t)scene * a.max_iters + it) * a.B + local] = resid;
        if (record) {
            const float rk = resid != resid ? INFINITY : resid;   // a NaN never passes the exit test
            float mx = owner ? rk : 0.f;
            if (P < 32) {
#pragma unroll
                for (int o = 16; o >= 1; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
                if (lane == 0) atomicMax(itm_s + it, float_key(mx));
            } else if (owner) {
                atomicMax(itm_s + it, float_key(rk));
            }
        }
    }

    if (record) {
        __syncthreads();
        unsigned* itm = a.itmax + (size_t)scene * a.max_iters * ITMAX_SLOTS + (cta % ITMAX_SLOTS);
        for (int t = threadIdx.x; t < iters; t += threads)
            if (const unsigned v = itm_s[t]) atomicMax(itm + (size_t)t * ITMAX_SLOTS, v);
    }
    // ---- outputs (out-of-range samples: stage-1 coefficients, +inf residual and cost)
    {
        constexpr unsigned gmask = RP >= 32 ? 0xffffffffu : ((1u << (RP & 31)) - 1u);
        const bool gov = (__ballot_sync(0xffffffffu, ovf) & (gmask << (lane & ~(RP - 1)))) != 0u;
        if (gov) {
            bad = false;
            resid = INFINITY;
            cost = INFINITY;
#pragma unroll
            for (int r = 0; r < ROWS; ++r) {
                const int i = own + RP * r;
                if (i < NX) c[r] = a.xi_bar[row * NX + (i & 1) * NC + (i >> 1)];
            }
        }
    }
    if (active) {
#pragma unroll
        for (int r = 0; r < ROWS; ++r) {
            const int i = own + RP * r;
            if (i < NX) a.xi_out[row * NX + (i & 1) * NC + (i >> 1)] = c[r];
        }
        if (own == r_lane) a.resid_out[row] = static_cast<double>(resid);
        if (a.cost_out && own == c_lane) a.cost_out[row] = static_cast<double>(cost);
        if (a.p2p_bufs && (own == r_lane || own == c_lane))
            p2p_store_all(a.p2p_bufs, a.p2p_world, own == r_lane ? a.p2p_res_off : a.p2p_cost_off,
                          a.p2p_row0 + local, static_cast<double>(own == r_lane ? resid : cost));
    } else {
        conf = 0;
        bad = false;
    }
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) conf += __shfl_xor_sync(0xffffffffu, conf, o);
    const unsigned anybad = __ballot_sync(0xffffffffu, bad);
    if (lane == 0) {
        if (conf) atomicAdd(a.conflicts + scene, (unsigned long long)conf);
        if (anybad) atomicOr(a.err + scene, ERR_NONFINITE);
    }
}

// LAT: latency instances, one CTA of 5-8 samples per SM (P = 64: two-warp samples, <= 128 registers;
// P = 32 / 16: one-warp / half-warp samples, whose <= 2 warps per SM sub-partition may use up to
// 255 registers and run the phase-split sweep_lat)
template <int P, bool CURV, int MT = 0, int NPT = 0, int TPB = 0, bool LAT = false, int HELP = 0>
__global__ void __launch_bounds__(LAT ? TPB : 256, LAT ? 1 : BD_AM_MINB) am_kernel(const AmArgs a) {
    // P <= 32: a sample is a group of P lanes of one warp.  P == 64: a sample spans two warps
    // (latency mapping for small batches); each warp reduce-scatters its partial sums, the second
    // warp hands them to the first through shared memory and the first warp owns the update.
    extern __shared__ __align__(16) unsigned char smem[];

    const int scene = blockIdx.y;
    int iters = a.max_iters;
    if (a.replay != nullptr) {
        iters = a.replay[scene];
        if (iters <= 0) return;
    }
    __shared__ __align__(8) uint64_t stage_bar;
    am_stage<P, CURV>(a, scene, smem, &stage_bar);
    am_samples<P, CURV, MT, NPT, TPB, LAT, HELP>(a, scene, -1, iters, smem);
    // ---- batch-global early exit folded into the last CTA of the scene (no extra launch)
    if (a.replay == nullptr && a.done_ctr != nullptr) {
        __shared__ bool last;
        __syncthreads();
        if (threadIdx.x == 0) {
            __threadfence();
            last = atomicAdd(a.done_ctr + scene, 1u) == gridDim.x - 1;
        }
        __syncthreads();
        if (last) {
            __threadfence();
            exit_scan_block(a.itmax + (size_t)scene * a.max_iters * ITMAX_SLOTS, a.max_iters, a.tol, scene,
                            a.iters_used, a.replay_out, a.conflicts);
            if (threadIdx.x == 0) a.done_ctr[scene] = 0u;
        }
    }
}

// Dense scenes: rewrite each (scene, timestep) row of the pair tile [(-x0,-x1,-y0,-y1) per pair]
// in place as obstacles (ox', oy') sorted ascending by ox' = -x/a (stable), the layout of the
// sorted-window obstacle pass.  One thread per row; rows are tiny (<= a few hundred values).
__global__ void sort_tile_kernel(float4* tile, int rows, int npair) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= rows) return;
    float4* row4 = tile + (size_t)r * npair;
    float2* row2 = reinterpret_cast<float2*>(row4);
    constexpr int CAP = 256;
    float xs[CAP], ys[CAP];
    const int n = min(2 * npair, CAP);
    for (int p = 0; p < n / 2; ++p) {
        const float4 v = row4[p];
        xs[2 * p] = v.x; xs[2 * p + 1] = v.y; ys[2 * p] = v.z; ys[2 * p + 1] = v.w;
    }
    for (int i = 1; i < n; ++i) {                 // insertion sort: stable, ties keep obstacle order
        const float kx = xs[i], ky = ys[i];
        int j = i - 1;
        while (j >= 0 && xs[j] > kx) { xs[j + 1] = xs[j]; ys[j + 1] = ys[j]; --j; }
        xs[j + 1] = kx; ys[j + 1] = ky;
    }
    for (int i = 0; i < n; ++i) row2[i] = make_float2(xs[i], ys[i]);
}

}  // namespace bd
