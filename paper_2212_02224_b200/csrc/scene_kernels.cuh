// device scene construction and control emission (sm_100a).
//
// build_scene + ego_flat_state (pkg/planners.py:99-160) and observe (pkg/highway.py:208-246)
// for a batch of worlds, writing the AM kernel's scene tiles directly; controls_on_grid ->
// flat_to_controls (pkg/planners.py:209-216, pkg/basis.py:206-234) for a batch of trajectories.
// fp64 throughout; the neighbour ordering reproduces Python's stable sort on the exactly
// rounded squared distance (no FMA contraction: __dmul_rn / __dadd_rn).
#pragma once

#include "bd_common.cuh"

namespace bd {

constexpr int OBS_DIM = 55;
constexpr int OBS_NEIGHBORS = 10;        // NUM_OBSERVED_NEIGHBORS (pkg/highway.py:19)
constexpr double SENTINEL = 1e4;         // SENTINEL_DISTANCE / SENTINEL_RANGE

struct SceneBuildArgs {
    int S, n_veh_max, n_obs, n_pad, m, neq;
    double range, wheelbase, v_max, a_max, k_max, c_max, v_min, other_len, other_wid;
    const double* ego;      // S x 8: x y psi v accel steer length width
    const double* veh;      // S x n_veh_max x 5: x y psi v lateral_rate
    const int* n_veh;       // S
    const double* road;     // S x 2: lane_count lane_width
    const double* times;    // m
    // outputs (AM scene buffers + optional host-facing copies)
    float* tile;            // S x m x n_pad/2 x 4 (-x0/a, -x1/a, -y0/b, -y1/b)
    SceneLim* lim;          // S
    double* bscene;         // S x neq
    double* ox64;           // S x n_obs x m
    double* oy64;
    double* lim64;          // S x 9
    double* b0_out;         // S x 6 (nullable)
    double* observation;    // S x 55 (nullable)
};

// Stable rank of vehicle j among the flagged ones by (squared distance, index).
__device__ __forceinline__ int stable_rank(const double* d2, const unsigned char* ok, int n, int j) {
    int r = 0;
    for (int k = 0; k < n; ++k) r += ok[k] && ((d2[k] < d2[j]) || (d2[k] == d2[j] && k < j));
    return r;
}

// One CTA per world.  Shared: squared distances, in-range flags, the chosen neighbour per slot.
__global__ void __launch_bounds__(256) build_scene_kernel(const SceneBuildArgs a) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int s = blockIdx.x;
    const int nv = a.n_veh[s];
    double* d2 = reinterpret_cast<double*>(smem);
    int* slot_obs = reinterpret_cast<int*>(d2 + a.n_veh_max);      // n_obs entries: vehicle id or -1
    int* slot_view = slot_obs + a.n_obs;                              // 10 entries
    unsigned char* inr = reinterpret_cast<unsigned char*>(slot_view + OBS_NEIGHBORS);
    unsigned char* all = inr + a.n_veh_max;
    const double* E = a.ego + (size_t)s * 8;
    const double ex = E[0], ey = E[1], epsi = E[2], ev = E[3], eacc = E[4], esteer = E[5], elen = E[6], ewid = E[7];
    const double* V = a.veh + (size_t)s * a.n_veh_max * 5;
    for (int i = threadIdx.x; i < a.n_obs; i += blockDim.x) slot_obs[i] = -1;
    for (int i = threadIdx.x; i < OBS_NEIGHBORS; i += blockDim.x) slot_view[i] = -1;
    for (int j = threadIdx.x; j < nv; j += blockDim.x) {
        const double dx = __dadd_rn(V[j * 5], -ex), dy = __dadd_rn(V[j * 5 + 1], -ey);
        d2[j] = __dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy));
        inr[j] = fabs(dx) <= a.range;                 // abs(veh.x - ego.x) <= obstacle_range
        all[j] = 1;
    }
    __syncthreads();
    for (int j = threadIdx.x; j < nv; j += blockDim.x) {
        if (inr[j]) {
            const int r = stable_rank(d2, inr, nv, j);
            if (r < a.n_obs) slot_obs[r] = j;
        }
        const int rv = stable_rank(d2, all, nv, j);
        if (rv < OBS_NEIGHBORS) slot_view[rv] = j;
    }
    __syncthreads();
    // combined_ellipse(ego.length, ego.width, 5, 2) (pkg/planners.py:90-96)
    const double ea = 1.4142135623730951 * ((elen + a.other_len) / 2.0);
    const double eb = 1.4142135623730951 * ((ewid + a.other_wid) / 2.0);
    const int lanes = (int)a.road[s * 2];
    const double lw = a.road[s * 2 + 1];
    const double ylb = -lw / 2.0, yub = (lanes - 1) * lw + lw / 2.0;
    // obstacle rows: constant-velocity predictions, far sentinels for empty slots
    for (int e = threadIdx.x; e < a.n_obs * a.m; e += blockDim.x) {
        const int i = e / a.m, t = e % a.m;
        const int j = slot_obs[i];
        BD_CHECK(j < nv);
        double ox, oy;
        if (j >= 0) {
            ox = __dadd_rn(V[j * 5], __dmul_rn(V[j * 5 + 3], a.times[t]));
            oy = __dadd_rn(V[j * 5 + 1], __dmul_rn(V[j * 5 + 4], a.times[t]));
        } else {
            ox = __dadd_rn(__dadd_rn(ex, SENTINEL), 100.0 * i);
            oy = 0.0;
        }
        a.ox64[((size_t)s * a.n_obs + i) * a.m + t] = ox;
        a.oy64[((size_t)s * a.n_obs + i) * a.m + t] = oy;
        float* tp = a.tile + ((((size_t)s * a.m + t) * (a.n_pad / 2) + i / 2) * 4) + (i & 1);
        tp[0] = (float)(-ox / ea);
        tp[2] = (float)(-oy / eb);
    }
    for (int e = threadIdx.x; e < (a.n_pad - a.n_obs) * a.m; e += blockDim.x) {   // even padding row
        const int i = a.n_obs + e / a.m, t = e % a.m;
        float* tp = a.tile + ((((size_t)s * a.m + t) * (a.n_pad / 2) + i / 2) * 4) + (i & 1);
        tp[0] = -1e18f;
        tp[2] = -1e18f;
    }
    if (threadIdx.x == 0) {
        SceneLim q;
        q.a = (float)ea; q.b = (float)eb; q.inv_a = (float)(1.0 / ea); q.inv_b = (float)(1.0 / eb);
        q.v_min = (float)a.v_min; q.v_max = (float)a.v_max; q.a_max = (float)a.a_max; q.k_max = (float)a.k_max;
        q.inv_k_max = (float)(1.0 / a.k_max); q.c_max = (float)a.c_max; q.y_lb = (float)ylb; q.y_ub = (float)yub;
        a.lim[s] = q;
        const double l9[9] = {ea, eb, a.v_min, a.v_max, a.a_max, a.k_max, a.c_max, ylb, yub};
        for (int k = 0; k < 9; ++k) a.lim64[s * 9 + k] = l9[k];
        // ego_flat_state (pkg/planners.py:99-113)
        double c, sn;
        sincos(epsi, &sn, &c);
        const double psid = __dmul_rn(ev, tan(esteer)) / a.wheelbase;
        const double b0[6] = {ex, ey, __dmul_rn(ev, c), __dmul_rn(ev, sn),
                              __dadd_rn(__dmul_rn(eacc, c), -__dmul_rn(__dmul_rn(ev, psid), sn)),
                              __dadd_rn(__dmul_rn(eacc, sn), __dmul_rn(__dmul_rn(ev, psid), c))};
        for (int k = 0; k < a.neq; ++k) a.bscene[s * a.neq + k] = k < 6 ? b0[k] : 0.0;
        if (a.b0_out)
            for (int k = 0; k < 6; ++k) a.b0_out[s * 6 + k] = b0[k];
    }
    if (a.observation && threadIdx.x < OBS_NEIGHBORS + 1) {
        // observe (pkg/highway.py:208-246)
        double* o = a.observation + (size_t)s * OBS_DIM;
        double c, sn;
        sincos(epsi, &sn, &c);
        if (threadIdx.x == OBS_NEIGHBORS) {
            o[0] = epsi;
            o[1] = __dmul_rn(ev, c);
            o[2] = __dmul_rn(ev, sn);
            o[53] = __dadd_rn(ey, -ylb);
            o[54] = __dadd_rn(yub, -ey);
        } else {
            const int slot = threadIdx.x, j = slot_view[slot];
            double* f = o + 3 + 5 * slot;
            if (j >= 0) {
                const double* v = V + j * 5;
                double cj, sj;
                sincos(v[2], &sj, &cj);
                const double vx = __dmul_rn(v[3], cj), vy = __dadd_rn(__dmul_rn(v[3], sj), v[4]);
                f[0] = __dadd_rn(v[0], -ex);
                f[1] = __dadd_rn(v[1], -ey);
                f[2] = __dadd_rn(vx, -__dmul_rn(ev, c));
                f[3] = __dadd_rn(vy, -__dmul_rn(ev, sn));
                f[4] = __dadd_rn(v[2], -epsi);
            } else {
                f[0] = SENTINEL; f[1] = 0.0; f[2] = 0.0; f[3] = 0.0; f[4] = 0.0;
            }
        }
    }
}

// flat_to_controls on the control grid + actuator clipping (pkg/planners.py:209-216):
// thread per (trajectory, control instant), fp64.
struct ControlArgs {
    int count, n_ctrl;
    const double* wd;    // n_ctrl x NC
    const double* wdd;   // n_ctrl x NC
    const double* xi;    // count x NX
    double wheelbase, a_max, steer_limit, eps_v;
    double* accel;       // count x n_ctrl
    double* steer;
    int* singular;       // count (SpeedSingularity)
};

__global__ void controls_kernel(const ControlArgs a) {
    const size_t id = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (id >= (size_t)a.count * a.n_ctrl) return;
    const int s = (int)(id / a.n_ctrl), t = (int)(id % a.n_ctrl);
    const double* c = a.xi + (size_t)s * NX;
    double xd = 0, yd = 0, xdd = 0, ydd = 0;
    for (int k = 0; k < NC; ++k) {
        const double w1 = a.wd[t * NC + k], w2 = a.wdd[t * NC + k];
        xd = fma(w1, c[k], xd); yd = fma(w1, c[NC + k], yd);
        xdd = fma(w2, c[k], xdd); ydd = fma(w2, c[NC + k], ydd);
    }
    const double v = hypot(xd, yd);
    if (!(v > a.eps_v)) atomicOr(a.singular + s, 1);
    const double kappa = (ydd * xd - xdd * yd) / (v * v * v);
    const double delta = atan(kappa * a.wheelbase);
    const double acc = (xd * xdd + yd * ydd) / v;
    a.accel[id] = fmin(fmax(acc, -a.a_max), a.a_max);
    a.steer[id] = fmin(fmax(delta, -a.steer_limit), a.steer_limit);
}

}  // namespace bd
