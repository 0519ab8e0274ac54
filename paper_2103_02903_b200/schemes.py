"""Scheme / run-configuration builders for the five BASELINE configurations.

Thin wrappers over the C++ builders (csrc/host_configs.cpp, exported through
the C-ABI) plus numpy helpers for the initial full-finest-mesh datum.
"""
import ctypes as C

import numpy as np

from . import _lib
from .abi import SchemeSpec, RunConfig, level_cells, level_extent, level_extent3

CONFIG_NAMES = {
    1: "D1Q2 Burgers",
    2: "D1Q3x3 Euler (Lax)",
    3: "D2Q4 advection (periodic disc)",
    4: "D2Q4x4 Euler (4-quadrant Riemann)",
    5: "D2Q9 Navier-Stokes (cylinder, Re=1200)",
    6: "D3Q6 advection (sphere, PAPER 7.3)",
}


def build_config(config_id: int, j_max: int = 0, epsilon: float = -1.0):
    """SchemeSpec / RunConfig for BASELINE config `config_id` (1..5).

    j_max > 0 overrides J_bar (parity tests use reduced sizes); epsilon >= 0
    overrides the threshold (epsilon = 0 is the uniform-mesh mode)."""
    sc, rc = SchemeSpec(), RunConfig()
    st = _lib.lib().mrlbm_build_config(int(config_id), int(j_max), float(epsilon), C.byref(sc), C.byref(rc))
    if st != 0:
        raise ValueError(f"mrlbm_build_config({config_id}) failed with status {st}")
    return sc, rc


def config_steps(config_id: int, rc: RunConfig) -> int:
    return int(_lib.lib().mrlbm_config_steps(int(config_id), C.byref(rc)))


def finest_cells(sc: SchemeSpec, rc: RunConfig) -> np.ndarray:
    """int32 coordinates (N, d) of the full finest mesh in CellIndex order."""
    nx, ny = level_extent(rc, sc.d, rc.j_max)
    if sc.d == 1:
        return np.arange(nx, dtype=np.int32).reshape(-1, 1)
    if sc.d == 3:
        ext = level_extent3(rc, 3, rc.j_max)
        g = np.meshgrid(*[np.arange(n, dtype=np.int32) for n in ext], indexing="ij")
        return np.stack([a.ravel() for a in g], axis=1).astype(np.int32)
    xs, ys = np.meshgrid(np.arange(nx, dtype=np.int32), np.arange(ny, dtype=np.int32), indexing="ij")
    return np.stack([xs.ravel(), ys.ravel()], axis=1).astype(np.int32)


def initial_finest(config_id: int, sc: SchemeSpec, rc: RunConfig, seed: int = 2103_02903) -> np.ndarray:
    """Equilibrium populations on the full finest mesh, SoA (q, N) float64."""
    f = np.empty((sc.q, level_cells(rc, sc.d, rc.j_max)), dtype=np.float64)
    st = _lib.lib().mrlbm_initial_finest(int(config_id), C.byref(sc), C.byref(rc), C.c_uint64(seed),
                                         f.ctypes.data_as(C.c_void_p))
    if st != 0:
        raise ValueError(f"mrlbm_initial_finest({config_id}) failed with status {st}")
    return f


def stream_table(d: int, gap: int, eta, side: int):
    """Flattened reconstruction table of the product (offsets (n, d), weights (n,))."""
    cap = 64 if d < 3 else 256
    off = np.zeros((cap, d), dtype=np.int32)
    w = np.zeros(cap, dtype=np.float64)
    n = C.c_int(0)
    e = (C.c_int32 * 3)(*([int(v) for v in eta] + [0] * (3 - len(eta))))
    st = _lib.lib().mrlbm_stream_table(d, gap, e, side, cap, off.ctypes.data_as(C.c_void_p),
                                       w.ctypes.data_as(C.c_void_p), C.byref(n))
    if st != 0:
        raise ValueError(f"mrlbm_stream_table failed with status {st}")
    return off[: n.value].copy(), w[: n.value].copy()
