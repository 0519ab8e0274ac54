"""ctypes mirror of include/mrlbm_gpu.h (struct layouts must match the C header).

Pure layout definitions; no library is loaded here so the oracle wrapper
(oracle/pyoracle.py) can share the descriptor types.
"""
import ctypes as C

MAX_Q = 16
MAX_LEVELS = 16

OK, ERR_CONFIG, ERR_NUMERIC, ERR_CUDA, ERR_CAPACITY, ERR_STATE = 0, 2, 3, 4, 5, 6
BC_COPY, BC_BOUNCE_BACK, BC_ANTI_BOUNCE_BACK, BC_PERIODIC, BC_VELOCITY_BOUNCE_BACK = 0, 1, 2, 3, 4
EQ_BURGERS_D1Q2, EQ_EULER_D1Q3X3, EQ_ADVECTION_D2Q4, EQ_EULER_D2Q4X4, EQ_NS_D2Q9 = 1, 2, 3, 4, 5
PHASES = ("project", "details", "flags", "compact", "transfer", "stream")


class SchemeSpec(C.Structure):
    """SchemeSpec."""
    _fields_ = [
        ("d", C.c_int32), ("q", C.c_int32), ("nblocks", C.c_int32), ("equilibrium", C.c_int32),
        ("lam", C.c_double),
        ("eta", (C.c_int32 * 3) * MAX_Q),
        ("M", C.c_double * (MAX_Q * MAX_Q)),
        ("Minv", C.c_double * (MAX_Q * MAX_Q)),
        ("s", C.c_double * MAX_Q),
        ("eq_params", C.c_double * 8),
    ]


class RunConfig(C.Structure):
    """RunConfig + DomainBox + boundaries + obstacle."""
    _fields_ = [
        ("j_min", C.c_int32), ("j_max", C.c_int32),
        ("base_cells", C.c_int64 * 3),
        ("origin", C.c_double * 3),
        ("epsilon", C.c_double),
        ("mu", C.c_int32), ("gamma", C.c_int32), ("graduation", C.c_int32),
        ("bc_kind", C.c_int32 * 6),
        ("bc_add", (C.c_double * MAX_Q) * 6),
        ("obstacle", C.c_int32), ("obstacle_subsamples", C.c_int32),
        ("obstacle_center", C.c_double * 3),
        ("obstacle_radius", C.c_double),
        ("obstacle_feq", C.c_double * MAX_Q),
    ]


class StepStats(C.Structure):
    _fields_ = [
        ("levels", C.c_int32),
        ("leaves", C.c_int64 * MAX_LEVELS),
        ("internal", C.c_int64 * MAX_LEVELS),
        ("virtual_cells", C.c_int64 * MAX_LEVELS),
        ("fallback_leaves", C.c_int64),
        ("leaf_updates", C.c_int64),
        ("ms_total", C.c_double),
        ("ms_phase", C.c_double * 8),
        ("bytes_model", C.c_int64),
        ("bytes_stream", C.c_int64),
        ("kernel_launches", C.c_int64),
        ("bytes_phase", C.c_int64 * 8),
    ]


class TieRecord(C.Structure):
    """mrlbm_tie_record: a group metric within 1e-12 relative of a threshold."""
    _fields_ = [
        ("step", C.c_int32), ("level", C.c_int32), ("cell", C.c_int32 * 3), ("which", C.c_int32),
        ("metric", C.c_double), ("threshold", C.c_double),
    ]


def tie_tuples(recs, n):
    """(step, level, cell..., which, metric, threshold) tuples of the first n records."""
    return [(r.step, r.level, r.cell[0], r.cell[1], r.cell[2], r.which, r.metric, r.threshold) for r in recs[:n]]


def level_extent(cfg: RunConfig, d: int, level: int):
    """(nx, ny) of a level box (ny = 1 in 1D); the 3D box is level_extent3."""
    sh = level - cfg.j_min
    nx = cfg.base_cells[0] << sh
    ny = (cfg.base_cells[1] << sh) if d >= 2 else 1
    return nx, ny


def level_extent3(cfg: RunConfig, d: int, level: int):
    sh = level - cfg.j_min
    return tuple((cfg.base_cells[a] << sh) if a < d else 1 for a in range(3))


def level_cells(cfg: RunConfig, d: int, level: int) -> int:
    nx, ny, nz = level_extent3(cfg, d, level)
    return nx * ny * nz
