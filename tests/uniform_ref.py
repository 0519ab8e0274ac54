"""Uniform finest-grid reference LBM (SPEC.md:326-334 `reference_step`) in numpy.

Independent of both the oracle and the product: used for the epsilon = 0
equivalence check (acceptance 3).  State = post-collision f*.
One step: stream f^h(k) = f^{h*}(k - eta^h) with the boundary closure
(PAPER.md:937-944 / Decisions D.14), then collide, then the
config-5 obstacle blend.
"""
import numpy as np

from paper_2103_02903_b200.abi import (BC_COPY, BC_BOUNCE_BACK, BC_ANTI_BOUNCE_BACK, BC_PERIODIC,
                                       BC_VELOCITY_BOUNCE_BACK, EQ_BURGERS_D1Q2, EQ_EULER_D1Q3X3,
                                       EQ_ADVECTION_D2Q4, EQ_EULER_D2Q4X4, EQ_NS_D2Q9, level_extent)


def equilibrium(sc, m):
    q = sc.q
    P = list(sc.eq_params)
    meq = np.zeros_like(m)
    if sc.equilibrium == EQ_BURGERS_D1Q2:
        u = m[0]
        meq[0] = u
        meq[1] = 0.5 * u * u
    elif sc.equilibrium == EQ_EULER_D1Q3X3:
        gam, lam2 = P[0], sc.lam * sc.lam
        rho, qq, E = m[0], m[3], m[6]
        u = qq / rho
        p = (gam - 1.0) * (E - 0.5 * rho * u * u)
        F = [qq, qq * u + p, u * (E + p)]
        U = [rho, qq, E]
        for i in range(3):
            meq[3 * i], meq[3 * i + 1], meq[3 * i + 2] = U[i], F[i], lam2 * U[i]
    elif sc.equilibrium == EQ_ADVECTION_D2Q4:
        u = m[0]
        meq[0], meq[1], meq[2], meq[3] = u, P[0] * u, P[1] * u, 0.0
    elif sc.equilibrium == EQ_EULER_D2Q4X4:
        gam = P[0]
        rho, qx, qy, E = m[0], m[4], m[8], m[12]
        u, v = qx / rho, qy / rho
        p = (gam - 1.0) * (E - 0.5 * rho * (u * u + v * v))
        Fx = [qx, qx * u + p, qx * v, u * (E + p)]
        Fy = [qy, qy * u, qy * v + p, v * (E + p)]
        U = [rho, qx, qy, E]
        for i in range(4):
            meq[4 * i], meq[4 * i + 1], meq[4 * i + 2], meq[4 * i + 3] = U[i], Fx[i], Fy[i], 0.0
    elif sc.equilibrium == EQ_NS_D2Q9:
        cs2 = P[0]
        rho, qx, qy = m[0], m[1], m[2]
        q2 = qx * qx + qy * qy
        meq[0], meq[1], meq[2] = rho, qx, qy
        meq[3] = 3.0 * (-2.0 * cs2 * rho + q2 / rho)
        meq[4] = -3.0 * cs2 * qx
        meq[5] = -3.0 * cs2 * qy
        meq[6] = 9.0 * (cs2 * cs2 * rho - cs2 * q2 / rho)
        meq[7] = (qx * qx - qy * qy) / rho
        meq[8] = qx * qy / rho
    else:
        raise ValueError("unknown equilibrium")
    return meq


def opposite(sc):
    q, bs = sc.q, sc.q // sc.nblocks
    opp = [-1] * q
    for h in range(q):
        for k in range(q):
            if k // bs == h // bs and all(sc.eta[k][i] == -sc.eta[h][i] for i in range(sc.d)):
                opp[h] = k
                break
    return opp


def obstacle_alpha(sc, rc):
    nx, ny = level_extent(rc, sc.d, rc.j_max)
    dx = 2.0 ** (-rc.j_max)
    ns = rc.obstacle_subsamples
    cx, cy, r = rc.obstacle_center[0], rc.obstacle_center[1], rc.obstacle_radius
    xs = np.arange(nx, dtype=np.float64)
    ys = np.arange(ny, dtype=np.float64)
    cnt = np.zeros((nx, ny))
    sub = (np.arange(ns) + 0.5) / ns
    for a in sub:
        sx = rc.origin[0] + (xs + a) * dx
        rx = (sx - cx) * (sx - cx)
        for b in sub:
            sy = rc.origin[1] + (ys + b) * dx
            ry = (sy - cy) * (sy - cy)
            cnt += (rx[:, None] + ry[None, :]) < r * r
    return cnt / (ns * ns)


class UniformLBM:
    def __init__(self, sc, rc, fstar_soa):
        self.sc, self.rc = sc, rc
        self.q, self.d = sc.q, sc.d
        nx, ny = level_extent(rc, sc.d, rc.j_max)
        self.shape = (nx, ny)
        self.f = fstar_soa.reshape(self.q, nx, ny).copy()
        self.M = np.array(sc.M[: self.q * self.q]).reshape(self.q, self.q)
        self.Minv = np.array(sc.Minv[: self.q * self.q]).reshape(self.q, self.q)
        self.s = np.array(sc.s[: self.q])
        self.opp = opposite(sc)
        self.alpha = obstacle_alpha(sc, rc) if rc.obstacle == 1 else None

    def step(self):
        sc, rc, q = self.sc, self.rc, self.q
        nx, ny = self.shape
        fs = self.f
        X, Y = np.meshgrid(np.arange(nx), np.arange(ny), indexing="ij")
        new = np.empty_like(fs)
        per = [rc.bc_kind[0] == BC_PERIODIC, self.d == 2 and rc.bc_kind[2] == BC_PERIODIC]
        for h in range(q):
            ex = sc.eta[h][0]
            ey = sc.eta[h][1] if self.d == 2 else 0
            sx, sy = X - ex, Y - ey
            if per[0]:
                sx = sx % nx
            if per[1]:
                sy = sy % ny
            outx = (sx < 0) | (sx >= nx)
            outy = (sy < 0) | (sy >= ny)
            out = outx | outy
            cx, cy = np.clip(sx, 0, nx - 1), np.clip(sy, 0, ny - 1)
            val = fs[h][cx, cy].copy()
            if out.any():
                face = np.where(outx, np.where(sx < 0, 0, 1), np.where(sy < 0, 2, 3))
                for fc in range(4):
                    sel = out & (face == fc)
                    if not sel.any():
                        continue
                    kind = rc.bc_kind[fc]
                    if kind == BC_COPY:
                        val[sel] = fs[h][cx, cy][sel]
                    elif kind in (BC_BOUNCE_BACK, BC_ANTI_BOUNCE_BACK, BC_VELOCITY_BOUNCE_BACK):
                        hb = self.opp[h]
                        v = fs[hb][sel]
                        if kind == BC_ANTI_BOUNCE_BACK:
                            v = -v
                        if kind == BC_VELOCITY_BOUNCE_BACK:
                            v = v + rc.bc_add[fc][h]
                        val[sel] = v
            new[h] = val
        m = np.einsum("ij,jxy->ixy", self.M, new)
        meq = equilibrium(sc, m)
        mp = (1.0 - self.s)[:, None, None] * m + self.s[:, None, None] * meq
        f = np.einsum("ij,jxy->ixy", self.Minv, mp)
        if self.alpha is not None:
            a = self.alpha[None]
            feq = np.array(rc.obstacle_feq[:q])[:, None, None]
            f = np.where(a > 0, a * feq + (1.0 - a) * f, f)
        self.f = f

    def soa(self):
        return self.f.reshape(self.q, -1)
