"""Independent numpy zero-detail reconstruction f^^ from the
complete leaves of every level -- the "second implementation" check of SPEC.md:215.

Level by level over dense arrays instead of the oracle's memoised recursion:
  1. R(Lambda) = leaves + their ancestors; internal values = (sum of the 2^d
     children in children order) / 2^d (prediction.hpp:51-60);
  2. top-down, a cell outside R takes predict() of the level above with the
     clamp / wrap stencil rule (Decision D.8) in the reference operation order
     (prediction.hpp:143-159; numpy does not contract to FMA, so the same order
     gives the same bits).
"""
import numpy as np

from paper_2103_02903_b200.abi import BC_PERIODIC, level_extent

C1 = -0.125


def _periodic(rc, d):
    return [rc.bc_kind[2 * i] == BC_PERIODIC for i in range(d)]


def _coord(c, n, per):
    return np.mod(c, n) if per else np.clip(c, 0, n - 1)


def reconstruct(rc, d, q, leaves):
    """leaves: {level: (idx (n, d) int32, f (q, n))}.  Returns (q, n_finest), lexicographic."""
    J0, J1 = rc.j_min, rc.j_max
    per = _periodic(rc, d)
    shp = {m: level_extent(rc, d, m)[:d] for m in range(J0, J1 + 1)}
    val = {m: np.zeros((q,) + shp[m]) for m in shp}
    inR = {m: np.zeros(shp[m], dtype=bool) for m in shp}
    for m, (idx, f) in leaves.items():
        if idx.shape[0] == 0:
            continue
        key = tuple(idx[:, a] for a in range(d))
        inR[m][key] = True
        for h in range(q):
            val[m][h][key] = f[h]
    # 1. ancestors (complete tree) and their projected values, bottom-up
    for m in range(J1 - 1, J0 - 1, -1):
        if d == 1:
            ch = [inR[m + 1][0::2], inR[m + 1][1::2]]
            kids = [val[m + 1][:, 0::2], val[m + 1][:, 1::2]]
        else:
            ch = [inR[m + 1][dx::2, dy::2] for dx in (0, 1) for dy in (0, 1)]
            kids = [val[m + 1][:, dx::2, dy::2] for dx in (0, 1) for dy in (0, 1)]
        internal = ch[0] & ~inR[m]
        acc = np.zeros_like(kids[0])
        for k in kids:
            acc = acc + k
        proj = acc / float(1 << d)
        val[m][:, internal] = proj[:, internal]
        inR[m] |= internal
    # 2. zero-detail prediction, top-down
    for m in range(J0 + 1, J1 + 1):
        P = val[m - 1]
        if d == 1:
            n = shp[m][0]
            x = np.arange(n)
            px = x >> 1
            st = [P[:, _coord(px + o, shp[m - 1][0], per[0])] for o in (-1, 0, 1)]
            s0 = np.where((x & 1) == 0, 1.0, -1.0)
            q1 = 0.0 + C1 * (st[2] - st[0])
            pred = st[1] + s0 * q1
        else:
            nx, ny = shp[m]
            x, y = np.meshgrid(np.arange(nx), np.arange(ny), indexing="ij")
            px, py = x >> 1, y >> 1
            st = {}
            for ox in (-1, 0, 1):
                for oy in (-1, 0, 1):
                    cx = _coord(px + ox, shp[m - 1][0], per[0])
                    cy = _coord(py + oy, shp[m - 1][1], per[1])
                    st[(ox + 1) * 3 + (oy + 1)] = P[:, cx, cy]
            s0 = np.where((x & 1) == 0, 1.0, -1.0)
            s1 = np.where((y & 1) == 0, 1.0, -1.0)
            qx = 0.0 + C1 * (st[7] - st[1])
            qy = 0.0 + C1 * (st[5] - st[3])
            inner = ((st[8] - st[2]) - st[6]) + st[0]
            qxy = 0.0 + (C1 * C1) * inner
            a = (st[4] + s0 * qx) + s1 * qy
            pred = a - (s0 * s1) * qxy
        out = np.where(inR[m], val[m], pred)
        val[m] = out
    return val[J1].reshape(q, -1)


def additional_error(f_adapt, f_ref, row):
    """E[m] = sum |m^^ - m_ref| / sum |m_ref|; absolute if the reference is zero."""
    row = np.asarray(row, dtype=np.float64)
    ma = np.zeros(f_adapt.shape[1])
    mb = np.zeros(f_ref.shape[1])
    for h in range(row.size):
        ma = ma + row[h] * f_adapt[h]
        mb = mb + row[h] * f_ref[h]
    num, den = float(np.abs(ma - mb).sum()), float(np.abs(mb).sum())
    return (num if den < 1e-300 else num / den), num, den
