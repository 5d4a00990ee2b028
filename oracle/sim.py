"""Oracle restatement of the highway simulator tick — TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Restates ``step`` (pkg/highway.py:358-410) and what it calls — ``lane_of`` (:65-66),
``idm_accel`` (:249-255), ``_leader_follower`` (:258-269), ``_gap`` / ``_accel_toward``
(:272-280), ``mobil_lane_change`` (:283-317), ``integrate_bicycle`` (:320-336) and
``footprints_overlap`` (:339-355) — over flat float64 arrays, one world at a time, in plain
Python.  Pinned against ``tests/golden/sim.npz`` (reference ``step`` run here by
tools/gen_golden.py).

World arrays (the same layout the device simulator keeps in HBM):
  ego  [9]      x, y, psi, v, accel, steer, length, width, target_speed
  veh  [n, 12]  x, y, psi, v, lateral_rate, length, width, target_speed, target_lane, cooldown,
                accel, lane_index
  ws   [5]      time, step_count, collided, collision_step (-1 = none), lane_departed
  road [4]      lane_count, lane_width, length, dt
"""

from __future__ import annotations

import math

import numpy as np

IDM = dict(v0=12.0, time_headway=1.5, s0=2.0, a_max=1.5, b_comfort=2.0, delta=4.0, b_hard=6.0)   # :73-81
MOBIL = dict(politeness=0.3, b_safe=4.0, a_threshold=0.1, cooldown=4.0)                           # :84-89
VX, VY, VPSI, VV, VLAT, VLEN, VWID, VTS, VTL, VCD, VACC, VLANE = range(12)


def lane_of(y, lanes, width):
    return int(np.clip(round(y / width), 0, lanes - 1))


def idm_accel(gap, v, dv, v0):
    p = IDM
    if gap <= 0.0:
        return -p["b_hard"]
    s_star = p["s0"] + v * p["time_headway"] + v * dv / (2.0 * np.sqrt(p["a_max"] * p["b_comfort"]))
    accel = p["a_max"] * (1.0 - (v / v0) ** p["delta"] - (s_star / gap) ** 2)
    return float(np.clip(accel, -p["b_hard"], p["a_max"]))


def _vehicles(ego, veh):
    """all_vehicles(): ego first, then neighbours, as (x, y, v, length, target_speed) rows."""
    rows = [(ego[0], ego[1], ego[3], ego[6], ego[8])]
    rows += [(r[VX], r[VY], r[VV], r[VLEN], r[VTS]) for r in veh]
    return rows


def leader_follower(vs, lane, x, lanes, width, skip):
    leader = follower = None
    for j, r in enumerate(vs):
        if j == skip or lane_of(r[1], lanes, width) != lane:
            continue
        if r[0] > x and (leader is None or r[0] < vs[leader][0]):
            leader = j
        elif r[0] <= x and (follower is None or r[0] > vs[follower][0]):
            follower = j
    return leader, follower


def _gap(rear, front):
    return front[0] - rear[0] - (front[3] + rear[3]) / 2.0


def accel_toward(me, leader):
    v0 = me[4] if me[4] > 0 else IDM["v0"]
    if leader is None:
        return idm_accel(np.inf, me[2], 0.0, v0)
    return idm_accel(_gap(me, leader), me[2], me[2] - leader[2], v0)


def mobil_lane_change(vs, j, target, lanes, width):
    me = vs[j]
    if not (0 <= target < lanes) or target == lane_of(me[1], lanes, width):
        return False
    nl, nf = leader_follower(vs, target, me[0], lanes, width, j)
    if nf is not None:
        f = vs[nf]
        decel = idm_accel(_gap(f, me), f[2], f[2] - me[2], f[4] if f[4] > 0 else IDM["v0"])
        if decel < -MOBIL["b_safe"]:
            return False
    ol, of = leader_follower(vs, lane_of(me[1], lanes, width), me[0], lanes, width, j)
    get = lambda i: None if i is None else vs[i]  # noqa: E731
    own = accel_toward(me, get(nl)) - accel_toward(me, get(ol))
    others = 0.0
    if nf is not None:
        others += accel_toward(vs[nf], me) - accel_toward(vs[nf], get(nl))
    if of is not None:
        others += accel_toward(vs[of], get(ol)) - accel_toward(vs[of], me)
    return own + MOBIL["politeness"] * others > MOBIL["a_threshold"]


def _deriv(s, accel, steer, wheelbase):
    return np.array([s[3] * np.cos(s[2]), s[3] * np.sin(s[2]), s[3] * np.tan(steer) / wheelbase, accel])


def integrate_bicycle(s, accel, steer, dt, wheelbase=2.5):
    k1 = _deriv(s, accel, steer, wheelbase)
    k2 = _deriv(s + 0.5 * dt * k1, accel, steer, wheelbase)
    k3 = _deriv(s + 0.5 * dt * k2, accel, steer, wheelbase)
    k4 = _deriv(s + dt * k3, accel, steer, wheelbase)
    out = s + (dt / 6.0) * (k1 + 2 * k2 + 2 * k3 + k4)
    out[3] = max(out[3], 0.0)
    return out


def _corners(x, y, psi, length, width):
    c, s = np.cos(psi), np.sin(psi)
    hx, hy = length / 2.0, width / 2.0
    local = np.array([[hx, hy], [hx, -hy], [-hx, -hy], [-hx, hy]])
    return local @ np.array([[c, -s], [s, c]]).T + np.array([x, y])


def overlap(a, b):
    """a, b = (x, y, psi, length, width)."""
    ca, cb = _corners(*a), _corners(*b)
    for psi in (a[2], b[2]):
        for axis in (np.array([np.cos(psi), np.sin(psi)]), np.array([-np.sin(psi), np.cos(psi)])):
            pa, pb = ca @ axis, cb @ axis
            if pa.max() < pb.min() or pb.max() < pa.min():
                return False
    return True


def step(ego, veh, ws, road, accel, steer, wheelbase=2.5):
    """One tick; returns new (ego, veh, ws) arrays (inputs untouched)."""
    ego, veh, ws = ego.copy(), veh.copy(), ws.copy()
    lanes, width, dt = int(road[0]), float(road[1]), float(road[3])
    vs = _vehicles(ego, veh)
    period = max(1, int(round(1.0 / dt)))
    decisions = []
    for i, r in enumerate(veh):
        lane = lane_of(r[VY], lanes, width)
        leader, _ = leader_follower(vs, lane, r[VX], lanes, width, i + 1)
        acc = accel_toward(vs[i + 1], None if leader is None else vs[leader])
        target = int(r[VTL])
        settled = abs(r[VY] - target * width) < 0.2
        if r[VCD] <= 0.0 and settled and (int(ws[1]) + i) % period == 0:
            for cand in (lane - 1, lane + 1):
                if 0 <= cand < lanes and mobil_lane_change(vs, i + 1, cand, lanes, width):
                    target = cand
                    break
        decisions.append((acc, target))
    s = integrate_bicycle(np.array(ego[:4]), accel, steer, dt, wheelbase)
    ego[:4] = s
    ego[4], ego[5] = accel, steer
    for r, (acc, target) in zip(veh, decisions):
        if target != int(r[VTL]):
            r[VTL] = target
            r[VCD] = MOBIL["cooldown"]
        r[VCD] = max(0.0, r[VCD] - dt)
        r[VV] = max(0.0, r[VV] + acc * dt)
        r[VX] += r[VV] * dt
        err = r[VTL] * width - r[VY]
        r[VLAT] = float(np.clip(1.5 * err, -1.5, 1.5))
        r[VY] += r[VLAT] * dt
        r[VPSI] = float(np.arctan2(r[VLAT], max(r[VV], 0.5)))
        r[VLANE] = lane_of(r[VY], lanes, width)
        r[VACC] = acc
    ws[0] += dt
    ws[1] += 1
    for r in veh:
        if overlap((ego[0], ego[1], ego[2], ego[6], ego[7]), (r[VX], r[VY], r[VPSI], r[VLEN], r[VWID])):
            ws[2] = 1.0
            if ws[3] < 0:
                ws[3] = ws[1]
            break
    half = ego[7] / 2.0
    if ego[1] - half < -width / 2.0 or ego[1] + half > (lanes - 1) * width + width / 2.0:
        ws[4] = 1.0
    return ego, veh, ws
