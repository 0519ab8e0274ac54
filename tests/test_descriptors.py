"""Every field of the product's scheme / run descriptors and its initial data, pinned
against the oracle's independent builder (oracle/mrlbm_oracle.cpp, build_descriptors:
written from BASELINE.json and the decisions ledger D.2, D.9, D.14-D.22, with M^-1 from
the reference DenseMatrix::inverse).  Before this pin the oracle reached the
descriptors only through the product (paper_2103_02903_b200.build_config), so a wrong
s2, Ladd term or obstacle_feq would have passed parity.
"""
import ctypes as C

import numpy as np
import pytest

from paper_2103_02903_b200 import build_config, initial_finest
from paper_2103_02903_b200.abi import SchemeSpec, RunConfig

CASES = [(1, 0, -1.0), (2, 0, -1.0), (3, 0, -1.0), (3, 0, 0.0), (4, 0, -1.0), (5, 0, -1.0),
         (1, 7, -1.0), (2, 9, -1.0), (4, 6, -1.0), (5, 6, -1.0), (5, 9, -1.0), (5, 10, -1.0),
         (6, 0, -1.0), (6, 5, -1.0), (6, 5, 0.0)]


def oracle_config(cid, J=0, eps=-1.0):
    from oracle import pyoracle
    return pyoracle.build_config(cid, J, eps)


def fields(struct):
    out = {}
    for name, _ in struct._fields_:
        v = getattr(struct, name)
        out[name] = np.ctypeslib.as_array(v).copy() if hasattr(v, "_length_") else v
    return out


@pytest.mark.parametrize("cid,J,eps", CASES)
def test_descriptors_bitwise(cid, J, eps):
    psc, prc = build_config(cid, J, eps)
    osc, orc = oracle_config(cid, J, eps)
    for a, b, kind in ((psc, osc, "scheme"), (prc, orc, "run config")):
        assert bytes(a) == bytes(b), {k: (v, fields(b)[k]) for k, v in fields(a).items()
                                      if not np.array_equal(np.asarray(v), np.asarray(fields(b)[k]))}


def test_config5_values_from_the_paper():
    """Spot values of the config-5 descriptor (D.14-D.17)."""
    osc, orc = oracle_config(5)
    cs2 = 1.0 / 3.0
    mu = 1.0 * 0.05 * 0.125 / 1200.0
    s2 = 1.0 / (0.5 + mu / (cs2 * 2.0 ** -12 * 1.0))
    assert osc.s[7] == s2 and abs(s2 - 1.773050) < 1e-6
    assert list(osc.s[:9]) == [0, 0, 0, 1.5, 1.5, 1.5, 1.5, s2, s2]
    # Ladd term 2 w_h rho0 (xi_h . u_w) / c_s^2 on the inlet for h = 1 (w = 1/9, xi_x = 1)
    assert orc.bc_add[0][1] == 2.0 * (1.0 / 9) * 1.0 * 0.05 / cs2 and orc.bc_add[1][1] == 0.0
    # obstacle target: rest equilibrium at rho0 = 1 has mass 1 and zero momentum
    feq = np.array(orc.obstacle_feq[:9])
    eta = np.array([[osc.eta[h][0], osc.eta[h][1]] for h in range(9)])
    assert abs(feq.sum() - 1.0) < 1e-15 and np.all(np.abs(feq @ eta) < 1e-16)


@pytest.mark.parametrize("cid,J", [(1, 8), (2, 8), (3, 6), (4, 6), (5, 6), (5, 8), (6, 5), (6, 6)])
def test_initial_data_bitwise(cid, J):
    from oracle import pyoracle
    psc, prc = build_config(cid, J)
    a = initial_finest(cid, psc, prc)
    b = pyoracle.initial_finest(cid, psc, prc)
    assert np.array_equal(a.view(np.uint64), b.view(np.uint64))
