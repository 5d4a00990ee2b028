// batched closed-loop highway simulation on the device (sm_100a).
//
// step (pkg/highway.py:358-410) for S worlds at once — neighbour IDM car following and MOBIL
// lane changes decided on the frozen snapshot (:249-317), ego RK4 bicycle (:320-336), neighbour
// updates, separating-axis collision test (:339-355) and lane departure — plus the inner loop of
// run_episode (:487-532): executing the planned controls open loop, stopping a world on collision
// or at the end of the road.  One CTA per world, one thread per neighbour; fp64 with the
// reference's operation order (no FMA contraction: __dmul_rn / __dadd_rn), so discrete outcomes
// (lane choices, collisions) follow the reference tick for tick.
#pragma once

#include <math_constants.h>

#include "bd_common.cuh"

namespace bd {

struct SimArgs {
    int S, n_max, n_steps, n_ctrl, ctrl_offset, period;
    double dt, wheelbase;
    double idm_v0, idm_T, idm_s0, idm_a, idm_b, idm_delta, idm_bhard, idm_sqrt_ab2;
    double pol, b_safe, a_thr, cooldown;
    double* ego;            // S x 8: x y psi v accel steer length width      (WorldBatch.ego)
    double* ego_ts;         // S: ego target speed (a follower's IDM v0 in MOBIL)
    double* veh;            // S x n_max x 5: x y psi v lateral_rate          (WorldBatch.veh)
    double* vext;           // S x n_max x 7: length width target_speed target_lane cooldown accel lane_index
    const int* n_veh;       // S
    const double* road;     // S x 2: lane_count lane_width                   (WorldBatch.road)
    double* world;          // S x 5: time step_count collided collision_step(-1: none) lane_departed
    const double* ctrl;     // S x n_ctrl x 2: accel steer
    const double* x_end;    // S: stop at ego.x >= x_end or on collision (run_episode); null: plain ticks
    int* active;            // S: worlds with 0 are skipped; cleared when a world stops (nullable)
    int* steps_done;        // S: ticks executed by this call (nullable)
    double* snap;           // S x n_steps x (8 + 4 n_max): t, ego x y psi v accel steer, collided,
                            //   neighbours x y psi v (nullable)
};

constexpr int VEXT = 7;

__device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double sub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double dvd(double a, double b) { return __ddiv_rn(a, b); }

// int(np.clip(round(y / w), 0, lanes - 1)) (pkg/highway.py:65-66); round = half to even
__device__ __forceinline__ int sim_lane_of(double y, int lanes, double w) {
    const double r = rint(dvd(y, w));
    return (int)fmin(fmax(r, 0.0), (double)(lanes - 1));
}

// x ** 4.0 as CPython's pow (correctly rounded): x^2 as a double-double, squared once more
__device__ __forceinline__ double pow4(double x) {
    const double h = mul(x, x), l = fma(x, x, -h);
    const double p = mul(h, h), pe = fma(h, h, -p);
    return add(p, fma(2.0 * h, l, fma(l, l, pe)));
}

struct SimWorld {   // frozen snapshot of one world (all_vehicles order: ego first)
    const double *x, *y, *v, *len, *ts;
    const int* lane;
    int n1;         // vehicles incl. ego
};

// idm_accel (pkg/highway.py:249-255)
__device__ double sim_idm(const SimArgs& a, double gap, double v, double dv, double v0) {
    if (gap <= 0.0) return -a.idm_bhard;
    const double s_star = add(add(a.idm_s0, mul(v, a.idm_T)), dvd(mul(v, dv), a.idm_sqrt_ab2));
    const double vr = dvd(v, v0);
    const double pv = (a.idm_delta == 4.0) ? pow4(vr) : pow(vr, a.idm_delta);
    const double q = dvd(s_star, gap);
    const double acc = mul(a.idm_a, sub(sub(1.0, pv), mul(q, q)));
    return fmin(fmax(acc, -a.idm_bhard), a.idm_a);
}

// _leader_follower (pkg/highway.py:258-269); -1 = none
__device__ void sim_lf(const SimWorld& w, int lane, double x, int skip, int& leader, int& follower) {
    leader = follower = -1;
    for (int j = 0; j < w.n1; ++j) {
        if (j == skip || w.lane[j] != lane) continue;
        const double xj = w.x[j];
        if (xj > x && (leader < 0 || xj < w.x[leader])) leader = j;
        else if (xj <= x && (follower < 0 || xj > w.x[follower])) follower = j;
    }
    BD_CHECK(leader < w.n1 && follower < w.n1 && leader != skip && follower != skip);
}

// _gap / _accel_toward (pkg/highway.py:272-280)
__device__ __forceinline__ double sim_gap(const SimWorld& w, int rear, int front) {
    return sub(sub(w.x[front], w.x[rear]), dvd(add(w.len[front], w.len[rear]), 2.0));
}
__device__ double sim_toward(const SimArgs& a, const SimWorld& w, int me, int leader) {
    const double v0 = w.ts[me] > 0 ? w.ts[me] : a.idm_v0;
    if (leader < 0) return sim_idm(a, CUDART_INF, w.v[me], 0.0, v0);
    return sim_idm(a, sim_gap(w, me, leader), w.v[me], sub(w.v[me], w.v[leader]), v0);
}

// mobil_lane_change (pkg/highway.py:283-317)
__device__ bool sim_mobil(const SimArgs& a, const SimWorld& w, int j, int target, int lanes) {
    if (!(0 <= target && target < lanes) || target == w.lane[j]) return false;
    int nl, nf, ol, of;
    sim_lf(w, target, w.x[j], j, nl, nf);
    if (nf >= 0) {
        const double v0 = w.ts[nf] > 0 ? w.ts[nf] : a.idm_v0;
        const double decel = sim_idm(a, sim_gap(w, nf, j), w.v[nf], sub(w.v[nf], w.v[j]), v0);
        if (decel < -a.b_safe) return false;
    }
    sim_lf(w, w.lane[j], w.x[j], j, ol, of);
    const double own = sub(sim_toward(a, w, j, nl), sim_toward(a, w, j, ol));
    double others = 0.0;
    if (nf >= 0) others = add(others, sub(sim_toward(a, w, nf, j), sim_toward(a, w, nf, nl)));
    if (of >= 0) others = add(others, sub(sim_toward(a, w, of, ol), sim_toward(a, w, of, j)));
    return add(own, mul(a.pol, others)) > a.a_thr;
}

// integrate_bicycle (pkg/highway.py:320-336)
__device__ void sim_deriv(const double s[4], double acc, double tan_steer, double wb, double k[4]) {
    k[0] = mul(s[3], cos(s[2]));
    k[1] = mul(s[3], sin(s[2]));
    k[2] = dvd(mul(s[3], tan_steer), wb);
    k[3] = acc;
}
__device__ void sim_rk4(double s[4], double acc, double steer, double dt, double wb) {
    const double ts = tan(steer), h = mul(0.5, dt);
    double k1[4], k2[4], k3[4], k4[4], t[4];
    sim_deriv(s, acc, ts, wb, k1);
    for (int i = 0; i < 4; ++i) t[i] = add(s[i], mul(h, k1[i]));
    sim_deriv(t, acc, ts, wb, k2);
    for (int i = 0; i < 4; ++i) t[i] = add(s[i], mul(h, k2[i]));
    sim_deriv(t, acc, ts, wb, k3);
    for (int i = 0; i < 4; ++i) t[i] = add(s[i], mul(dt, k3[i]));
    sim_deriv(t, acc, ts, wb, k4);
    const double c = dvd(dt, 6.0);
    for (int i = 0; i < 4; ++i)
        s[i] = add(s[i], mul(c, add(add(add(k1[i], mul(2.0, k2[i])), mul(2.0, k3[i])), k4[i])));
    s[3] = (0.0 > s[3]) ? 0.0 : s[3];
}

// footprints_overlap (pkg/highway.py:339-355): separating-axis test of two oriented rectangles
__device__ void sim_corners(double x, double y, double psi, double len, double wid, double cx[4], double cy[4]) {
    const double c = cos(psi), s = sin(psi), hx = dvd(len, 2.0), hy = dvd(wid, 2.0);
    const double lx[4] = {hx, hx, -hx, -hx}, ly[4] = {hy, -hy, -hy, hy};
    for (int i = 0; i < 4; ++i) {
        cx[i] = add(add(mul(lx[i], c), mul(ly[i], -s)), x);
        cy[i] = add(add(mul(lx[i], s), mul(ly[i], c)), y);
    }
}
__device__ bool sim_overlap(const double A[5], const double B[5]) {
    double ax[4], ay[4], bx[4], by[4];
    sim_corners(A[0], A[1], A[2], A[3], A[4], ax, ay);
    sim_corners(B[0], B[1], B[2], B[3], B[4], bx, by);
    for (int r = 0; r < 2; ++r) {
        const double psi = r ? B[2] : A[2];
        const double c = cos(psi), s = sin(psi);
        for (int q = 0; q < 2; ++q) {
            const double ux = q ? -s : c, uy = q ? c : s;
            double amin = CUDART_INF, amax = -CUDART_INF, bmin = CUDART_INF, bmax = -CUDART_INF;
            for (int i = 0; i < 4; ++i) {
                const double pa = add(mul(ax[i], ux), mul(ay[i], uy));
                const double pb = add(mul(bx[i], ux), mul(by[i], uy));
                amin = fmin(amin, pa); amax = fmax(amax, pa);
                bmin = fmin(bmin, pb); bmax = fmax(bmax, pb);
            }
            if (amax < bmin || bmax < amin) return false;
        }
    }
    return true;
}

// One CTA per world; the world runs n_steps ticks inside the launch.
__global__ void __launch_bounds__(128) sim_kernel(const SimArgs a) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int s = blockIdx.x;
    __shared__ int stop;
    if (a.active && !a.active[s]) {
        if (threadIdx.x == 0 && a.steps_done) a.steps_done[s] = 0;
        return;
    }
    const int n = a.n_veh[s], n1 = n + 1, nm = a.n_max;
    double* sx = reinterpret_cast<double*>(smem);
    double* sy = sx + (nm + 1);
    double* sv = sy + (nm + 1);
    double* sl = sv + (nm + 1);
    double* st = sl + (nm + 1);
    double* dacc = st + (nm + 1);                        // per-neighbour decision: acceleration
    int* sln = reinterpret_cast<int*>(dacc + nm);
    int* dtgt = sln + (nm + 1);                          // and target lane
    const SimWorld w{sx, sy, sv, sl, st, sln, n1};
    if (threadIdx.x == 0) stop = 0;
    const int lanes = (int)a.road[2 * s];
    const double lw = a.road[2 * s + 1];
    double* E = a.ego + (size_t)s * 8;
    double* V = a.veh + (size_t)s * nm * 5;
    double* X = a.vext + (size_t)s * nm * VEXT;
    double* W = a.world + (size_t)s * 5;
    const int SNAP = 8 + 4 * nm;
    int done = 0;
    for (int j = 0; j < a.n_steps; ++j) {
        // ---- frozen snapshot (all_vehicles order: ego, then neighbours)
        for (int i = threadIdx.x; i < n1; i += blockDim.x) {
            if (i == 0) { sx[0] = E[0]; sy[0] = E[1]; sv[0] = E[3]; sl[0] = E[6]; st[0] = a.ego_ts[s]; }
            else {
                const double* v = V + (size_t)(i - 1) * 5;
                sx[i] = v[0]; sy[i] = v[1]; sv[i] = v[3];
                sl[i] = X[(size_t)(i - 1) * VEXT]; st[i] = X[(size_t)(i - 1) * VEXT + 2];
            }
            sln[i] = sim_lane_of(sy[i], lanes, lw);
        }
        const double step_count = W[1];
        __syncthreads();
        // ---- neighbour decisions on the snapshot (pkg/highway.py:365-378)
        for (int i = threadIdx.x; i < n; i += blockDim.x) {
            const int jv = i + 1, lane = sln[jv];
            int leader, follower;
            sim_lf(w, lane, sx[jv], jv, leader, follower);
            dacc[i] = sim_toward(a, w, jv, leader);
            int target = (int)X[(size_t)i * VEXT + 3];
            const bool settled = fabs(sub(sy[jv], mul((double)target, lw))) < 0.2;
            if (X[(size_t)i * VEXT + 4] <= 0.0 && settled && ((long long)step_count + i) % a.period == 0) {
                for (int cand = lane - 1; cand <= lane + 1; cand += 2)
                    if (0 <= cand && cand < lanes && sim_mobil(a, w, jv, cand, lanes)) { target = cand; break; }
            }
            dtgt[i] = target;
        }
        // ---- ego RK4 (every thread, identical inputs -> identical registers; thread 0 stores)
        const double* C = a.ctrl + ((size_t)s * a.n_ctrl + min(a.ctrl_offset + j, a.n_ctrl - 1)) * 2;
        const double acc_e = C[0], steer_e = C[1];
        double es[4] = {E[0], E[1], E[2], E[3]};
        sim_rk4(es, acc_e, steer_e, a.dt, a.wheelbase);
        const double EA[5] = {es[0], es[1], es[2], E[6], E[7]};
        __syncthreads();              // all snapshot / ego reads done before any write
        if (threadIdx.x == 0) { E[0] = es[0]; E[1] = es[1]; E[2] = es[2]; E[3] = es[3]; E[4] = acc_e; E[5] = steer_e; }
        // ---- neighbour updates (pkg/highway.py:386-397) + collision test against the new ego
        bool hit = false;
        double* snap = a.snap ? a.snap + ((size_t)s * a.n_steps + j) * SNAP : nullptr;
        for (int i = threadIdx.x; i < n; i += blockDim.x) {
            double* v = V + (size_t)i * 5;
            double* x = X + (size_t)i * VEXT;
            double tl = x[3], cd = x[4];
            if (dtgt[i] != (int)tl) { tl = dtgt[i]; cd = a.cooldown; }
            cd = fmax(0.0, sub(cd, a.dt));
            const double vel = fmax(0.0, add(v[3], mul(dacc[i], a.dt)));
            const double px = add(v[0], mul(vel, a.dt));
            const double err = sub(mul(tl, lw), v[1]);
            const double lat = fmin(fmax(mul(1.5, err), -1.5), 1.5);
            const double py = add(v[1], mul(lat, a.dt));
            const double psi = atan2(lat, fmax(vel, 0.5));
            v[0] = px; v[1] = py; v[2] = psi; v[3] = vel; v[4] = lat;
            x[3] = tl; x[4] = cd; x[5] = dacc[i]; x[6] = sim_lane_of(py, lanes, lw);
            const double VB[5] = {px, py, psi, x[0], x[1]};
            hit |= sim_overlap(EA, VB);
            BD_CHECK(i < nm && 11 + 4 * i < SNAP);
            if (snap) { snap[8 + 4 * i] = px; snap[9 + 4 * i] = py; snap[10 + 4 * i] = psi; snap[11 + 4 * i] = vel; }
        }
        hit = __syncthreads_or(hit);
        if (threadIdx.x == 0) {
            W[0] = add(W[0], a.dt);
            W[1] = step_count + 1.0;
            if (hit) {
                W[2] = 1.0;
                if (W[3] < 0) W[3] = W[1];
            }
            const double half = dvd(E[7], 2.0);
            if (sub(es[1], half) < -dvd(lw, 2.0) || add(es[1], half) > add(mul((double)(lanes - 1), lw), dvd(lw, 2.0)))
                W[4] = 1.0;
            if (snap) {
                snap[0] = W[0]; snap[1] = es[0]; snap[2] = es[1]; snap[3] = es[2]; snap[4] = es[3];
                snap[5] = acc_e; snap[6] = steer_e; snap[7] = W[2];
                for (int i = n; i < nm; ++i) snap[8 + 4 * i] = snap[9 + 4 * i] = snap[10 + 4 * i] = snap[11 + 4 * i] = 0.0;
            }
            // run_episode termination (pkg/highway.py:524-529)
            stop = a.x_end && (W[2] != 0.0 || es[0] >= a.x_end[s]);
        }
        __syncthreads();
        done = j + 1;
        if (stop) break;
    }
    if (threadIdx.x == 0) {
        if (a.steps_done) a.steps_done[s] = done;
        if (a.active && stop) a.active[s] = 0;
    }
}

}  // namespace bd
