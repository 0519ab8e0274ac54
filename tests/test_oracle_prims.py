"""Pin the checker and the product's host tables against the REFERENCE's own
primitives (oracle/_ref/libmrlbm_refprims.so, compiled from
/root/reference/proj/core/include) and against SPEC/PAPER known answers."""
import ctypes as C
import itertools
from fractions import Fraction

import numpy as np
import pytest

from paper_2103_02903_b200 import build_config, stream_table
from oracle import pyoracle


def ref():
    return pyoracle.ref_lib()


def vp(a):
    return a.ctypes.data_as(C.c_void_p)


def test_table1_coefficients():
    """derive_prediction_weights reproduces Table 1."""
    expect = {1: [Fraction(-1, 8)], 2: [Fraction(-22, 128), Fraction(3, 128)],
              3: [Fraction(-201, 1024), Fraction(11, 256), Fraction(-5, 1024)]}
    for g, ex in expect.items():
        num = np.zeros(3, dtype=np.int64)
        den = np.zeros(3, dtype=np.int64)
        n = ref().ref_derive_weights(g, vp(num), vp(den))
        assert n == g
        assert [Fraction(int(a), int(b)) for a, b in zip(num[:n], den[:n])] == ex


def test_prediction_weight_fan_2d():
    """2D gamma=1 one-hot fan for delta=(0,0) (PAPER Fig. 4 with the
    reference's minus cross term, prediction.hpp:158)."""
    delta = np.array([0, 0], dtype=np.int32)
    W = np.zeros((3, 3))
    for ox, oy in itertools.product(range(3), range(3)):
        st = np.zeros(9)
        st[ox * 3 + oy] = 1.0
        W[ox, oy] = ref().ref_predict(2, 1, vp(st), vp(delta))
    # index [x+1][y+1]
    assert W[1, 1] == 1.0
    assert W[0, 1] == 1 / 8 and W[1, 0] == 1 / 8      # W and S
    assert W[2, 1] == -1 / 8 and W[1, 2] == -1 / 8    # E and N
    assert W[2, 0] == 1 / 64 and W[0, 2] == 1 / 64    # SE and NW
    assert W[2, 2] == -1 / 64 and W[0, 0] == -1 / 64  # NE and SW


def test_predict_linear_1d():
    """d=1 linear data: left child mean = k - 1/4."""
    k = 7.0
    st = np.array([k - 1, k, k + 1])
    assert ref().ref_predict(1, 1, vp(st), vp(np.array([0], dtype=np.int32))) == k - 0.25
    assert ref().ref_predict(1, 1, vp(st), vp(np.array([1], dtype=np.int32))) == k + 0.25


def test_project_examples():
    """SPEC.md:151-153."""
    assert ref().ref_project(1, vp(np.array([1.0, 3.0]))) == 2.0
    assert ref().ref_project(2, vp(np.array([1.0, 2.0, 3.0, 4.0]))) == 2.5
    assert ref().ref_project(2, vp(np.array([0.3] * 4))) == 0.3


def test_children_parent_examples():
    """cell.hpp:80-116; SPEC.md:50-61 including the negative ghost index."""
    out = np.zeros(8, dtype=np.int64)
    assert ref().ref_children2(0, 0, 0, 5, vp(out)) == 0
    assert out.reshape(4, 2).tolist() == [[0, 0], [0, 1], [1, 0], [1, 1]]
    p = np.zeros(2, dtype=np.int64)
    assert ref().ref_parent2(5, -1, 4, 0, vp(p)) == 4
    assert p.tolist() == [-1, 2]


def test_cellindex_order_is_lexicographic():
    """CellIndex slots (cell_set.hpp:333-354) = lexicographic order, last axis
    fastest: the payload contract of mrlbm_read_leaves."""
    rng = np.random.default_rng(0)
    pts = np.unique(rng.integers(-3, 20, size=(200, 2)), axis=0)
    rng.shuffle(pts)
    slots = np.zeros(len(pts), dtype=np.int64)
    n = ref().ref_cellindex_slots2(len(pts), vp(np.ascontiguousarray(pts, dtype=np.int64)), vp(slots))
    assert n == len(pts)
    order = np.lexsort((pts[:, 1], pts[:, 0]))
    assert (slots[order] == np.arange(len(pts))).all()


@pytest.mark.parametrize("cid", [1, 2, 3, 4, 5])
def test_minv_bitwise_reference_inverse(cid):
    """The descriptor's M^-1 equals DenseMatrix::inverse(M) bit for bit
    (dense_matrix.hpp:58-113), so GPU and oracle collide with identical doubles."""
    sc, _ = build_config(cid)
    q = sc.q
    M = np.array(sc.M[: q * q])
    out = np.zeros(q * q)
    assert ref().ref_inverse(q, vp(M), vp(out)) == 0
    assert np.array_equal(out.view(np.uint64), np.array(sc.Minv[: q * q]).view(np.uint64))


def test_d2q4_moment_example():
    """D2Q4 M with lambda=5 on f=(1,1,1,1) -> m=(4,0,0,0)."""
    lam = 5.0
    M = np.array([[1, 1, 1, 1], [lam, 0, -lam, 0], [0, lam, 0, -lam], [lam * lam, -lam * lam, lam * lam, -lam * lam]],
                 dtype=np.float64).ravel()
    y = np.zeros(4)
    ref().ref_multiply(4, vp(M), vp(np.ones(4)), vp(y))
    assert y.tolist() == [4.0, 0.0, 0.0, 0.0]


def _exact_table(d, g, eta, side):
    c = Fraction(-1, 8)

    def pw(delta):
        if d == 1:
            s = 1 if delta[0] == 0 else -1
            return {(-1,): -s * c, (0,): Fraction(1), (1,): s * c}
        s0 = 1 if delta[0] == 0 else -1
        s1 = 1 if delta[1] == 0 else -1
        w = {(0, 0): Fraction(1)}

        def add(k, v):
            w[k] = w.get(k, 0) + v
        add((1, 0), s0 * c); add((-1, 0), -s0 * c); add((0, 1), s1 * c); add((0, -1), -s1 * c)
        t = -s0 * s1 * c * c
        add((1, 1), t); add((-1, 1), -t); add((1, -1), -t); add((-1, -1), t)
        return w

    n = 2 ** g
    inb = lambda x: all(0 <= xi < n for xi in x)  # noqa: E731
    cur = {}
    for x in itertools.product(range(-1, n + 1), repeat=d):
        xe = tuple(xi + e for xi, e in zip(x, eta))
        if (inb(xe) and not inb(x)) if side == 0 else (inb(x) and not inb(xe)):
            cur[x] = Fraction(1)
    for _ in range(g):
        nxt = {}
        for cc, w in cur.items():
            p = tuple(ci >> 1 for ci in cc)
            dl = tuple(ci - 2 * pi for ci, pi in zip(cc, p))
            for o, wo in pw(dl).items():
                k = tuple(pi + oi for pi, oi in zip(p, o))
                nxt[k] = nxt.get(k, 0) + w * wo
        cur = nxt
    return {k: v for k, v in sorted(cur.items()) if v != 0}, cur


def test_gap1_table_row():
    """gap 1, eta=+1 (d=1), incoming -> offsets {-2,-1,0}, w {-1/8, 1, 1/8}."""
    off, w = stream_table(1, 1, (1,), 0)
    assert off[:, 0].tolist() == [-2, -1, 0]
    assert w.tolist() == [-0.125, 1.0, 0.125]


@pytest.mark.parametrize("d,eta", [(1, (1,)), (1, (-1,)), (2, (1, 0)), (2, (0, -1)), (2, (1, 1)), (2, (-1, 1))])
def test_tables_three_ways(d, eta):
    """Product (push), oracle (pull over reference predict) and exact rationals
    (correctly rounded) agree bit for bit; exact on constants."""
    for g in range(0, 7 if d == 2 else 10):
        for side in (0, 1):
            a_off, a_w = stream_table(d, g, eta, side)
            b_off, b_w = pyoracle.stream_table(d, g, eta, side)
            exact, _ = _exact_table(d, g, eta, side)
            assert np.array_equal(a_off, b_off) and np.array_equal(a_w.view(np.uint64), b_w.view(np.uint64))
            assert [tuple(o) for o in a_off.tolist()] == list(exact.keys())
            assert all(float(v) == x for v, x in zip(exact.values(), a_w))
            # |E| = |A| = 2^g (|ex| + |ey|) - |ex||ey| and sum of weights = |E|
            ex, ey = abs(eta[0]), abs(eta[1]) if d == 2 else 0
            card = (2 ** g) * (ex + ey) - ex * ey if d == 2 else ex
            assert sum(exact.values()) == card


def test_deep_gap_rounding():
    """Gap >= 10 diagonal weights need 54+ bits: both builders round to nearest."""
    for g in (10, 11):
        a_off, a_w = stream_table(2, g, (1, 1), 0)
        b_off, b_w = pyoracle.stream_table(2, g, (1, 1), 0)
        assert np.array_equal(a_w.view(np.uint64), b_w.view(np.uint64))


@pytest.mark.parametrize("d,eta", [(1, (1,)), (1, (-1,)), (2, (1, 0)), (2, (0, 1)), (2, (1, 1)), (2, (-1, 1)), (2, (0, 0))])
def test_table_exactness_sets(d, eta):
    """Product (support propagation in push form) and oracle (memo keys of the pull
    recursion) agree on the exactness sets of every table (Decision D.13)."""
    from paper_2103_02903_b200 import _lib
    L = _lib.lib()
    O = pyoracle.oracle_lib()
    O.oracle_stream_table_sets.argtypes = [C.c_int, C.c_int, C.POINTER(C.c_int32), C.c_int, C.c_int, C.c_void_p,
                                           C.POINTER(C.c_int), C.c_void_p, C.POINTER(C.c_int)]
    L.mrlbm_stream_table_sets.argtypes = [C.c_int, C.c_int, C.POINTER(C.c_int32), C.c_int, C.c_int, C.c_void_p,
                                          C.c_void_p, C.POINTER(C.c_int)]
    e = (C.c_int32 * 3)(*([int(v) for v in eta] + [0] * (3 - len(eta))))
    for g in range(0, 6):
        for side in (0, 1):
            cap = 4096
            dep = np.zeros((cap, d), dtype=np.int32)
            par = np.zeros((cap, d), dtype=np.int32)
            nd, npar = C.c_int(), C.c_int()
            assert O.oracle_stream_table_sets(d, g, e, side, cap, vp(dep), C.byref(nd), vp(par), C.byref(npar)) == 0
            box = np.zeros(4, dtype=np.int32)
            par2 = np.zeros((cap, d), dtype=np.int32)
            n2 = C.c_int()
            assert L.mrlbm_stream_table_sets(d, g, e, side, cap, vp(box), vp(par2), C.byref(n2)) == 0
            assert npar.value == n2.value
            assert np.array_equal(par[: npar.value], par2[: n2.value])
            if nd.value:
                dd = dep[: nd.value]
                assert box[0] == dd[:, 0].min() and box[1] == dd[:, 0].max()
                if d == 2:
                    assert box[2] == dd[:, 1].min() and box[3] == dd[:, 1].max()
            # parents sit in the 3^d box around the leaf for |eta| <= 1
            assert (np.abs(par[: npar.value]) <= 1).all()
