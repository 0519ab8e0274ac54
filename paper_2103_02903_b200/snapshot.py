"""Snapshot and metrics I/O either side of the step.

The reference specifies these formats in SPEC.md but does not implement them.

`cells_<step>.csv`, one row per complete leaf:
- levels ascending; within a level, CellIndex (lexicographic) order;
- columns: `level, k0[, k1], x0[, x1], edge, m<h>...`;
- `x` is the lower corner `origin + k * edge`, with `edge = 2^-level` (cell.hpp:67-76, Decision A.2);
- `m<h>` are the conserved moments, i.e. rows h of M with s_h = 0, computed as `m = M f` in the
  `DenseMatrix::multiply` order (dense_matrix.hpp:42-54);
- floats are written with 17 significant digits, so a reload returns the same doubles.

`metrics.csv` gets one line per step. It is append-only and flushed on every line.
Columns: `step, leaves, internal, mesh_or, mem_or, fallback_leaves, ms, E`. The occupation rates are:
- MeshOR = #S(Lambda) / #finest cells, with denominator 2^{dJ} in the unit box;
- MemOR = #(leaves + internal) / #(cells of the full tree over all levels).
"""
import math
import os

import numpy as np

from .abi import level_cells, level_extent


def conserved_rows(scheme):
    """Rows h of M with relaxation s_h == 0 (the conserved moments)."""
    return [h for h in range(scheme.q) if scheme.s[h] == 0.0]


def moments(scheme, f, rows):
    """m_i = sum_j M[i, j] f_j, accumulated from 0.0 in j order (dense_matrix.hpp:42-54)."""
    q = scheme.q
    out = np.zeros((len(rows), f.shape[1]))
    for r, i in enumerate(rows):
        acc = np.zeros(f.shape[1])
        for j in range(q):
            acc = acc + scheme.M[i * q + j] * f[j]
        out[r] = acc
    return out


def _fmt(v):
    return format(float(v), ".17g")


def write_snapshot(solver, step, directory, rows=None):
    """Write cells_<step>.csv for the solver's current state. Returns the path."""
    sc, rc, d = solver.scheme, solver.cfg, solver.d
    rows = conserved_rows(sc) if rows is None else list(rows)
    os.makedirs(directory, exist_ok=True)
    path = os.path.join(directory, f"cells_{int(step)}.csv")
    hdr = ["level"] + [f"k{i}" for i in range(d)] + [f"x{i}" for i in range(d)] + ["edge"] + [f"m{h}" for h in rows]
    with open(path, "w") as fh:
        fh.write(",".join(hdr) + "\n")
        for lv in range(rc.j_min, rc.j_max + 1):
            idx, f = solver.read_leaves(lv)
            if idx.shape[0] == 0:
                continue
            edge = math.ldexp(1.0, -lv)
            m = moments(sc, f, rows)
            for i in range(idx.shape[0]):
                k = [int(idx[i, a]) for a in range(d)]
                x = [rc.origin[a] + k[a] * edge for a in range(d)]
                cols = [str(lv)] + [str(v) for v in k] + [_fmt(v) for v in x] + [_fmt(edge)]
                cols += [_fmt(m[r, i]) for r in range(len(rows))]
                fh.write(",".join(cols) + "\n")
    return path


def read_snapshot(path):
    """Reload a cells_<step>.csv: {level: (idx (n, d) int32, moments (r, n))}, plus the column names."""
    with open(path) as fh:
        hdr = fh.readline().strip().split(",")
        d = sum(1 for c in hdr if c.startswith("k"))
        nm = sum(1 for c in hdr if c.startswith("m"))
        per = {}
        for line in fh:
            c = line.strip().split(",")
            lv = int(c[0])
            per.setdefault(lv, ([], []))
            per[lv][0].append([int(v) for v in c[1:1 + d]])
            per[lv][1].append([float(v) for v in c[2 + 2 * d:2 + 2 * d + nm]])
    out = {lv: (np.array(a, dtype=np.int32).reshape(-1, d), np.array(b).reshape(-1, nm).T) for lv, (a, b) in per.items()}
    return out, hdr


def occupation_rates(rc, d, stats):
    """(MeshOR, MemOR) of the mesh after the last step."""
    full_leaves = level_cells(rc, d, rc.j_max)
    full_tree = sum(level_cells(rc, d, lv) for lv in range(rc.j_min, rc.j_max + 1))
    nl = stats.levels
    leaves = sum(int(stats.leaves[i]) for i in range(nl))
    internal = sum(int(stats.internal[i]) for i in range(nl))
    return leaves / full_leaves, (leaves + internal) / full_tree


class MetricsWriter:
    """Append-only metrics.csv, flushed per line."""

    COLUMNS = ("step", "leaves", "internal", "mesh_or", "mem_or", "fallback_leaves", "ms", "E")

    def __init__(self, directory, rc, d):
        os.makedirs(directory, exist_ok=True)
        self.path = os.path.join(directory, "metrics.csv")
        self.rc, self.d = rc, d
        new = not os.path.exists(self.path)
        self.fh = open(self.path, "a")
        if new:
            self.fh.write(",".join(self.COLUMNS) + "\n")
            self.fh.flush()

    def append(self, step, stats, E=None):
        mesh_or, mem_or = occupation_rates(self.rc, self.d, stats)
        nl = stats.levels
        vals = [str(int(step)), str(sum(int(stats.leaves[i]) for i in range(nl))),
                str(sum(int(stats.internal[i]) for i in range(nl))), _fmt(mesh_or), _fmt(mem_or),
                str(int(stats.fallback_leaves)), _fmt(stats.ms_total), "" if E is None else _fmt(E)]
        self.fh.write(",".join(vals) + "\n")
        self.fh.flush()

    def close(self):
        self.fh.close()
