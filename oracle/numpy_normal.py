"""Test infrastructure: a numpy-free-of-numpy restatement of the device's parallel reproduction of
numpy's Generator(PCG64).standard_normal stream (csrc/numpy_normals.cuh), for CPU tests.

Serial reference: numpy itself.  This module restates the kernel's parallel form -- raw outputs per
position, "a draw starting at every position", start resolution by walking back to a sync point
and replaying, the cover painting and the scan -- so the CPU suite can pin the algorithm against
numpy before the GPU runs it.  Not imported by the package.
"""
import math

import numpy as np

ZIG_R = 3.6541528853610087963519472518
ZIG_INV_R = 0.27366123732975827203338247596
CMAX = 64


def _u01(r):
    return (r >> 11) * (1.0 / 9007199254740992.0)


def draw_at(raw, j, tables):
    """(value, consumption) of a draw starting at raw position j (numpy random_standard_normal);
    consumption 0 if it would need raw values beyond the evaluated range or CMAX."""
    ki, wi, fi = tables
    R = len(raw)
    k = j
    while True:
        if k >= R or k - j >= CMAX:
            return 0.0, 0
        r = int(raw[k])
        k += 1
        idx = r & 0xFF
        r >>= 8
        sign = r & 1
        rabs = (r >> 1) & 0x000FFFFFFFFFFFFF
        x = float(rabs) * float(wi[idx])
        if sign:
            x = -x
        if rabs < int(ki[idx]):
            return x, k - j
        if idx == 0:
            while True:
                if k + 1 >= R or k + 1 - j >= CMAX:
                    return 0.0, 0
                xx = -ZIG_INV_R * math.log1p(-_u01(int(raw[k])))
                yy = -math.log1p(-_u01(int(raw[k + 1])))
                k += 2
                if yy + yy > xx * xx:
                    return (-(ZIG_R + xx) if (rabs >> 8) & 1 else ZIG_R + xx), k - j
        else:
            if k >= R:
                return 0.0, 0
            u = _u01(int(raw[k]))
            k += 1
            if (float(fi[idx - 1]) - float(fi[idx])) * u + float(fi[idx]) < math.exp(-0.5 * x * x):
                return x, k - j


def parallel_stream(bitgen, count, block_len, tables, rc=16384):
    """(z, positions) as the kernel computes them: chunks of `rc` raw positions, each starting at a
    known draw start; z = the first `count` normals of the bit generator's stream,
    positions[b] = raw outputs consumed by the first b blocks."""
    s0 = bitgen.state
    base, done = 0, 0
    z = np.empty(count)
    nb = count // block_len
    positions = np.zeros(nb + 1, dtype=np.int64)
    while done < count:
        g = np.random.PCG64()
        g.state = s0
        g.advance(base)
        raw = g.random_raw(rc + CMAX)
        xv = np.empty(rc)
        cv = np.empty(rc, dtype=np.int64)
        for j in range(rc):
            xv[j], cv[j] = draw_at(raw, j, tables)
        start = np.zeros(rc, dtype=np.int64)
        for j in range(rc):                  # slow positions: sync-point walk + replay
            if cv[j] == 1:
                continue
            q, run = j, 0
            while q > 0 and run < CMAX:
                run = run + 1 if cv[q - 1] == 1 else 0
                q -= 1
            if run >= CMAX:
                q += CMAX
            cur = q
            while cur < j and cv[cur] != 0:
                cur += cv[cur]
            start[j] = 1 if cur == j else 0
        covered = np.zeros(rc, dtype=bool)   # cover painting by slow starts
        for j in np.nonzero((start == 1) & (cv > 1))[0]:
            covered[j + 1:j + cv[j]] = True
        is_start = np.where(cv == 1, ~covered, start == 1)
        starts = np.nonzero(is_start)[0]
        for j in starts:
            if done < count:
                if cv[j] == 0:
                    raise RuntimeError("a draw needed more than CMAX raw values")
                z[done] = xv[j]
                if (done + 1) % block_len == 0:
                    positions[(done + 1) // block_len] = base + j + cv[j]
            done += 1
        last = starts[-1]
        base += int(last + cv[last])
    return z, positions
