"""The C-ABI library loads on a CPU-only host and exports every symbol that
include/*.h declares (no compute calls without a GPU)."""
import ctypes as C
import os
import re

from paper_2103_02903_b200 import _lib, build_config, config_steps, initial_finest, finest_cells

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    syms = set()
    inc = os.path.join(ROOT, "include")
    for fn in os.listdir(inc):
        if fn.endswith(".h"):
            txt = open(os.path.join(inc, fn)).read()
            syms |= set(re.findall(r"\b(mrlbm_[a-z_]+)\s*\(", txt))
    return syms


def test_library_exports_all_declared_symbols():
    L = _lib.lib()
    syms = declared_symbols()
    assert len(syms) >= 15
    for s in sorted(syms):
        assert hasattr(L, s), f"missing export {s}"


def test_config_steps():
    """N = ceil(T / dt) (Decision D.11)."""
    expect = {1: 2048, 2: 6882, 3: 512, 4: 2048, 5: 50000}
    for cid, n in expect.items():
        sc, rc = build_config(cid)
        assert config_steps(cid, rc) == n


def test_initial_datum_equilibrium():
    """f(0) = M^-1 m^eq(u0): conserved moments equal u0 at cell centres."""
    import numpy as np
    sc, rc = build_config(4, 5)
    f = initial_finest(4, sc, rc)
    M = np.array(sc.M[:256]).reshape(16, 16)
    m = M @ f
    idx = finest_cells(sc, rc)
    x = (idx[:, 0] + 0.5) / 32
    y = (idx[:, 1] + 0.5) / 32
    rho = np.where((x > 0.5) & (y > 0.5), 1.5, np.where((x < 0.5) & (y > 0.5), 0.5323,
                   np.where((x < 0.5) & (y < 0.5), 0.138, 0.5323)))
    assert np.allclose(m[0], rho, rtol=1e-14)


def test_create_without_gpu_fails_loudly():
    """No CPU fallback: on a host without a CUDA device mrlbm_create must fail."""
    import torch
    if torch.cuda.is_available():
        return
    from paper_2103_02903_b200 import Solver
    sc, rc = build_config(3, 5)
    try:
        Solver(sc, rc)
    except Exception:
        return
    raise AssertionError("mrlbm_create succeeded without a CUDA device")
