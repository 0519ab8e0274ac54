"""Host-side mirror of the reference's solver interface for the hot path.

`Solver` wraps one C-ABI context (one GPU stream, all levels resident in HBM):
load a complete-leaf FieldSet in CellIndex order, run Algorithm-1 steps
(adapt -> stream -> collide), read leaves back.  Errors raise like the
reference's exceptions (ValueError ~ std::invalid_argument, FloatingPointError
~ std::domain_error, RuntimeError otherwise).
"""
import ctypes as C

import numpy as np

from . import _lib
from .abi import StepStats, TieRecord, tie_tuples, PHASES, ERR_CONFIG, ERR_NUMERIC


class MRLBMError(RuntimeError):
    pass


def _raise(status, msg):
    if status == ERR_CONFIG:
        raise ValueError(msg)
    if status == ERR_NUMERIC:
        raise FloatingPointError(msg)
    raise MRLBMError(f"status {status}: {msg}")


def drag_lift(fx, fy, rho0, u0, L):
    """C_D, C_L = 2 F / (rho0 u0^2 L), through the C-ABI."""
    lib = _lib.lib()
    cd, cl = C.c_double(0.0), C.c_double(0.0)
    st = lib.mrlbm_drag_lift(float(fx), float(fy), float(rho0), float(u0), float(L), C.byref(cd), C.byref(cl))
    if st != 0:
        _raise(st, "drag_lift: rho0 u0^2 L must be positive")
    return cd.value, cl.value


def strouhal(cl, dt, u0, L, skip=0):
    """St = L f / u0 of the dominant shedding frequency of a lift series (
    SPEC.md:477-485).  Returns (St, frequency resolution).  Raises FloatingPointError
    ("no dominant peak") for a flat spectrum."""
    lib = _lib.lib()
    y = np.ascontiguousarray(cl, dtype=np.float64)
    st, df = C.c_double(0.0), C.c_double(0.0)
    code = lib.mrlbm_strouhal(y.ctypes.data_as(C.c_void_p), y.size, int(skip), float(dt), float(u0), float(L),
                              C.byref(st), C.byref(df))
    if code != 0:
        _raise(code, "strouhal: no dominant peak" if code == ERR_NUMERIC else "strouhal: need >= 8 samples, dt > 0")
    return st.value, df.value


class Solver:
    def __init__(self, scheme, cfg):
        self.L = _lib.lib()
        self.scheme, self.cfg = scheme, cfg
        self.d, self.q = scheme.d, scheme.q
        h = C.c_void_p()
        st = self.L.mrlbm_create(C.byref(scheme), C.byref(cfg), C.byref(h))
        if st != 0:
            _raise(st, "mrlbm_create failed (invalid configuration or no CUDA device)")
        self.h = h

    def _check(self, st):
        if st != 0:
            _raise(st, self.L.mrlbm_last_error(self.h).decode())

    def load_leaves(self, level, idx, f):
        idx = np.ascontiguousarray(idx, dtype=np.int32)
        f = np.ascontiguousarray(f, dtype=np.float64)
        n = idx.shape[0]
        assert f.shape == (self.q, n)
        self._check(self.L.mrlbm_load_leaves(self.h, int(level), n, idx.ctypes.data_as(C.c_void_p),
                                             f.ctypes.data_as(C.c_void_p)))

    def commit(self):
        self._check(self.L.mrlbm_commit(self.h))

    def tie_log(self, reset=False):
        """Near-threshold tie records since commit, sorted: list of (step, level, cx, cy,
        cz, which, metric, threshold) tuples (include/mrlbm_gpu.h, mrlbm_tie_log)."""
        n = C.c_int64(0)
        self._check(self.L.mrlbm_tie_log(self.h, None, 0, C.byref(n), 0))
        recs = (TieRecord * max(1, n.value))()
        self._check(self.L.mrlbm_tie_log(self.h, recs, n.value, C.byref(n), int(bool(reset))))
        return tie_tuples(recs, n.value)

    def step(self, n=1):
        stats = StepStats()
        self._check(self.L.mrlbm_step(self.h, int(n), C.byref(stats)))
        return stats

    def level_count(self, level):
        n = C.c_int64(0)
        self._check(self.L.mrlbm_level_count(self.h, int(level), C.byref(n)))
        return n.value

    def read_leaves(self, level):
        n = self.level_count(level)
        idx = np.zeros((n, self.d), dtype=np.int32)
        f = np.zeros((self.q, n), dtype=np.float64)
        if n:
            self._check(self.L.mrlbm_read_leaves(self.h, int(level), idx.ctypes.data_as(C.c_void_p),
                                                 f.ctypes.data_as(C.c_void_p)))
        return idx, f

    def read_leaves_into(self, level, idx, f):
        """Read one level into caller-provided (e.g. pinned) buffers: idx (n, d) int32,
        f (q, n) float64, both C-contiguous with n = level_count(level)."""
        n = self.level_count(level)
        assert idx.shape == (n, self.d) and f.shape == (self.q, n)
        assert idx.flags.c_contiguous and f.flags.c_contiguous
        if n:
            self._check(self.L.mrlbm_read_leaves(self.h, int(level), idx.ctypes.data_as(C.c_void_p),
                                                 f.ctypes.data_as(C.c_void_p)))
        return n

    def finest_count(self):
        n = C.c_int64(0)
        self._check(self.L.mrlbm_finest_count(self.h, C.byref(n)))
        return n.value

    def reconstruct_finest(self):
        """Zero-detail reconstruction f^^ of the current state on the full finest grid,
        (q, n) float64, lexicographic."""
        f = np.zeros((self.q, self.finest_count()), dtype=np.float64)
        self._check(self.L.mrlbm_reconstruct_finest(self.h, f.ctypes.data_as(C.c_void_p)))
        return f

    def additional_error(self, reference, row):
        """E[m] against `reference` (a Solver on the same finest grid, typically epsilon=0),
        m = sum_h row[h] f^h.  Returns (E, sum|diff|, sum|m_ref|)."""
        row = np.ascontiguousarray(row, dtype=np.float64)
        assert row.shape == (self.q,)
        e = C.c_double(0.0)
        sums = np.zeros(2, dtype=np.float64)
        self._check(self.L.mrlbm_additional_error(self.h, reference.h, row.ctypes.data_as(C.c_void_p), C.byref(e),
                                                  sums.ctypes.data_as(C.c_void_p)))
        return e.value, float(sums[0]), float(sums[1])

    def set_force_tracking(self, capacity_steps):
        """Record the obstacle force (Fx, Fy) of each following step on the device
        (config 5).  0 turns it off."""
        self._check(self.L.mrlbm_set_force_tracking(self.h, int(capacity_steps)))

    def force_history(self):
        """(fx, fy) arrays of the per-step obstacle forces recorded since tracking began."""
        n = C.c_int(0)
        self._check(self.L.mrlbm_force_history(self.h, None, None, 0, C.byref(n)))
        fx = np.zeros(n.value, dtype=np.float64)
        fy = np.zeros(n.value, dtype=np.float64)
        if n.value:
            self._check(self.L.mrlbm_force_history(self.h, fx.ctypes.data_as(C.c_void_p),
                                                   fy.ctypes.data_as(C.c_void_p), n.value, C.byref(n)))
        return fx, fy

    def set_profiling(self, on=True):
        """True / 1: an event after every kernel (one stream); 2: phase events only with the
        step's forks active; False / 0: off."""
        self._check(self.L.mrlbm_set_profiling(self.h, int(on)))

    def profile_text(self, reset=True):
        """Per-kernel device times of the profiled steps: {(kernel, level): (ms, launches)}."""
        buf = C.create_string_buffer(1 << 16)
        self._check(self.L.mrlbm_profile_text(self.h, buf, len(buf), int(bool(reset))))
        out = {}
        for line in buf.value.decode().splitlines():
            k, lv, ms, n = line.split()
            out[(k, int(lv))] = (float(ms), int(n))
        return out

    def set_graph(self, on=True):
        self._check(self.L.mrlbm_set_graph(self.h, int(bool(on))))

    def stream_handle(self):
        return self.L.mrlbm_stream_handle(self.h)

    def synchronize(self):
        self._check(self.L.mrlbm_synchronize(self.h))

    def close(self):
        if getattr(self, "h", None):
            self.L.mrlbm_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @staticmethod
    def phase_dict(stats):
        return {p: stats.ms_phase[i] for i, p in enumerate(PHASES)}
