"""ctypes wrapper of the CPU oracle (oracle/_lib/libmrlbm_oracle.so) and of the
reference-primitive shim (oracle/_ref/libmrlbm_refprims.so).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and the
bench's cpu_baseline / --impl reference legs, never by the product package.
"""
import ctypes as C
import os
import subprocess

import numpy as np

from paper_2103_02903_b200.abi import SchemeSpec, RunConfig, TieRecord, tie_tuples

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_lib", "libmrlbm_oracle.so")
REFPRIMS_SO = os.path.join(HERE, "_ref", "libmrlbm_refprims.so")
REF_INCLUDE = "/root/reference/proj/core/include"


def build():
    """Compile the oracle and the reference shim (needs /root/reference)."""
    if os.path.isdir(REF_INCLUDE):
        subprocess.run(["make", "-s", "-C", HERE], check=True)
    if not os.path.exists(ORACLE_SO):
        raise RuntimeError("oracle library missing and /root/reference not available to build it")


_orc = None
_ref = None


def oracle_lib():
    global _orc
    if _orc is None:
        if not os.path.exists(ORACLE_SO):
            build()
        L = C.CDLL(ORACLE_SO)
        vp = C.c_void_p
        P = C.POINTER
        L.oracle_create.argtypes = [P(SchemeSpec), P(RunConfig), P(vp)]
        L.oracle_load_leaves.argtypes = [vp, C.c_int, C.c_int64, vp, vp]
        L.oracle_commit.argtypes = [vp]
        L.oracle_step.argtypes = [vp, C.c_int]
        L.oracle_level_count.argtypes = [vp, C.c_int, P(C.c_int64)]
        L.oracle_internal_count.argtypes = [vp, C.c_int, P(C.c_int64)]
        L.oracle_read_leaves.argtypes = [vp, C.c_int, vp, vp]
        L.oracle_fallback_leaves.argtypes = [vp]
        L.oracle_reconstruct_finest.argtypes = [vp, vp]
        L.oracle_fallback_leaves.restype = C.c_int64
        L.oracle_last_error.argtypes = [vp]
        L.oracle_last_error.restype = C.c_char_p
        L.oracle_destroy.argtypes = [vp]
        L.oracle_destroy.restype = None
        L.oracle_set_threads.argtypes = [C.c_int]
        L.oracle_tie_log.argtypes = [vp, P(TieRecord), C.c_int, P(C.c_int64), C.c_int]
        L.oracle_build_config.argtypes = [C.c_int, C.c_int, C.c_double, P(SchemeSpec), P(RunConfig)]
        L.oracle_initial_finest.argtypes = [C.c_int, P(SchemeSpec), P(RunConfig), C.c_uint64, vp]
        L.oracle_set_force_tracking.argtypes = [vp, C.c_int]
        L.oracle_force_history.argtypes = [vp, vp, vp, C.c_int, P(C.c_int)]
        L.oracle_stream_table.argtypes = [C.c_int, C.c_int, P(C.c_int32), C.c_int, C.c_int, vp, vp, P(C.c_int)]
        _orc = L
    return _orc


def ref_lib():
    global _ref
    if _ref is None:
        if not os.path.exists(REFPRIMS_SO):
            build()
        L = C.CDLL(REFPRIMS_SO)
        vp = C.c_void_p
        L.ref_predict.restype = C.c_double
        L.ref_predict.argtypes = [C.c_int, C.c_int, vp, vp]
        L.ref_project.restype = C.c_double
        L.ref_project.argtypes = [C.c_int, vp]
        L.ref_derive_weights.argtypes = [C.c_int, vp, vp]
        L.ref_prediction_coeffs.argtypes = [C.c_int, vp]
        L.ref_inverse.argtypes = [C.c_int, vp, vp]
        L.ref_multiply.argtypes = [C.c_int, vp, vp, vp]
        L.ref_multiply.restype = None
        L.ref_children2.argtypes = [C.c_int, C.c_int64, C.c_int64, C.c_int, vp]
        L.ref_parent2.argtypes = [C.c_int, C.c_int64, C.c_int64, C.c_int, vp]
        L.ref_cellindex_slots2.argtypes = [C.c_int, vp, vp]
        _ref = L
    return _ref


def build_config(config_id, j_max=0, epsilon=-1.0):
    """The oracle's own descriptors for BASELINE config `config_id` (independent of the
    product's builder; pinned field by field in tests/test_descriptors.py)."""
    sc, rc = SchemeSpec(), RunConfig()
    st = oracle_lib().oracle_build_config(int(config_id), int(j_max), float(epsilon), C.byref(sc), C.byref(rc))
    if st != 0:
        raise ValueError(f"oracle_build_config({config_id}) failed with status {st}")
    return sc, rc


def finest_cells(sc, rc):
    """int32 coordinates (N, d) of the full finest mesh in CellIndex order."""
    sh = rc.j_max - rc.j_min
    nx = int(rc.base_cells[0]) << sh
    if sc.d == 1:
        return np.arange(nx, dtype=np.int32).reshape(-1, 1)
    ny = int(rc.base_cells[1]) << sh
    if sc.d == 3:
        nz = int(rc.base_cells[2]) << sh
        g = np.meshgrid(np.arange(nx, dtype=np.int32), np.arange(ny, dtype=np.int32),
                        np.arange(nz, dtype=np.int32), indexing="ij")
        return np.stack([a.ravel() for a in g], axis=1).astype(np.int32)
    xs, ys = np.meshgrid(np.arange(nx, dtype=np.int32), np.arange(ny, dtype=np.int32), indexing="ij")
    return np.stack([xs.ravel(), ys.ravel()], axis=1).astype(np.int32)


def initial_finest(config_id, sc, rc, seed=2103_02903):
    """The oracle's initial datum (D.22) on the full finest mesh, SoA (q, N)."""
    n = finest_cells(sc, rc).shape[0]
    f = np.empty((sc.q, n), dtype=np.float64)
    st = oracle_lib().oracle_initial_finest(int(config_id), C.byref(sc), C.byref(rc), C.c_uint64(seed),
                                            f.ctypes.data_as(C.c_void_p))
    if st != 0:
        raise ValueError(f"oracle_initial_finest({config_id}) failed with status {st}")
    return f


def set_threads(n):
    return oracle_lib().oracle_set_threads(int(n))


class Oracle:
    """Same call sequence as paper_2103_02903_b200.Solver, on the CPU."""

    def __init__(self, scheme, cfg):
        self.L = oracle_lib()
        self.d, self.q = scheme.d, scheme.q
        self.n_finest = 1
        for i in range(scheme.d):
            self.n_finest *= int(cfg.base_cells[i]) << (cfg.j_max - cfg.j_min)
        h = C.c_void_p()
        st = self.L.oracle_create(C.byref(scheme), C.byref(cfg), C.byref(h))
        if st != 0:
            raise ValueError(f"oracle_create failed with status {st}")
        self.h = h

    def _check(self, st):
        if st != 0:
            msg = self.L.oracle_last_error(self.h).decode()
            if st == 2:
                raise ValueError(msg)
            if st == 3:
                raise FloatingPointError(msg)
            raise RuntimeError(f"oracle status {st}: {msg}")

    def load_leaves(self, level, idx, f):
        idx = np.ascontiguousarray(idx, dtype=np.int32)
        f = np.ascontiguousarray(f, dtype=np.float64)
        self._check(self.L.oracle_load_leaves(self.h, int(level), idx.shape[0], idx.ctypes.data_as(C.c_void_p),
                                              f.ctypes.data_as(C.c_void_p)))

    def commit(self):
        self._check(self.L.oracle_commit(self.h))

    def step(self, n=1):
        self._check(self.L.oracle_step(self.h, int(n)))

    def tie_log(self, reset=False):
        """Near-threshold tie records since commit, sorted (same tuples as Solver.tie_log)."""
        n = C.c_int64(0)
        self._check(self.L.oracle_tie_log(self.h, None, 0, C.byref(n), 0))
        recs = (TieRecord * max(1, n.value))()
        self._check(self.L.oracle_tie_log(self.h, recs, n.value, C.byref(n), int(bool(reset))))
        return tie_tuples(recs, n.value)

    def level_count(self, level):
        n = C.c_int64(0)
        self._check(self.L.oracle_level_count(self.h, int(level), C.byref(n)))
        return n.value

    def internal_count(self, level):
        n = C.c_int64(0)
        self._check(self.L.oracle_internal_count(self.h, int(level), C.byref(n)))
        return n.value

    def fallback_leaves(self):
        return int(self.L.oracle_fallback_leaves(self.h))

    def read_leaves(self, level):
        n = self.level_count(level)
        idx = np.zeros((n, self.d), dtype=np.int32)
        f = np.zeros((self.q, n), dtype=np.float64)
        if n:
            self._check(self.L.oracle_read_leaves(self.h, int(level), idx.ctypes.data_as(C.c_void_p),
                                                  f.ctypes.data_as(C.c_void_p)))
        return idx, f

    def reconstruct_finest(self):
        """f^^ on the full finest grid, (q, n) lexicographic (oracle rec())."""
        f = np.zeros((self.q, self.n_finest), dtype=np.float64)
        self._check(self.L.oracle_reconstruct_finest(self.h, f.ctypes.data_as(C.c_void_p)))
        return f

    def set_force_tracking(self, on=True):
        self._check(self.L.oracle_set_force_tracking(self.h, int(bool(on))))

    def force_history(self):
        n = C.c_int(0)
        self._check(self.L.oracle_force_history(self.h, None, None, 0, C.byref(n)))
        fx = np.zeros(n.value)
        fy = np.zeros(n.value)
        self._check(self.L.oracle_force_history(self.h, fx.ctypes.data_as(C.c_void_p), fy.ctypes.data_as(C.c_void_p),
                                                n.value, C.byref(n)))
        return fx, fy

    def close(self):
        if getattr(self, "h", None):
            self.L.oracle_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def stream_table(d, gap, eta, side):
    cap = 64 if d < 3 else 256
    off = np.zeros((cap, d), dtype=np.int32)
    w = np.zeros(cap, dtype=np.float64)
    n = C.c_int(0)
    e = (C.c_int32 * 3)(*([int(v) for v in eta] + [0] * (3 - len(eta))))
    st = oracle_lib().oracle_stream_table(d, gap, e, side, cap, off.ctypes.data_as(C.c_void_p),
                                          w.ctypes.data_as(C.c_void_p), C.byref(n))
    if st != 0:
        raise ValueError(f"oracle_stream_table failed with status {st}")
    return off[: n.value].copy(), w[: n.value].copy()
