"""Pins for oracle.schemes / oracle.brent (CPU).  Each test names the paper /
SPEC passage or mathematical fact it pins."""
import os

import numpy as np
import pytest

import oracle as O

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _golden_strassen():
    vals = {}
    with open(os.path.join(GOLDEN, "strassen_scalar.txt")) as f:
        for line in f:
            line = line.split("#", 1)[0].strip()
            if line:
                key, *rest = line.split()
                vals[key] = [int(v) for v in rest]
    return vals


def test_strassen_worked_example_intermediates():
    # S:226 / S:233 / S:240 / S:247: scalar-block Strassen example, exact.
    g = _golden_strassen()
    s = O.strassen()
    A = np.array(g["A"]).reshape(2, 2)
    B = np.array(g["B"]).reshape(2, 2)
    res = O.lcma_i64(A, B, s, intermediates=True)
    assert res.At.reshape(-1).tolist() == g["At"]
    assert res.Bt.reshape(-1).tolist() == g["Bt"]
    assert res.H.reshape(-1).tolist() == g["H"]
    assert res.C.reshape(-1).tolist() == g["C"]


def test_strassen_nnz_and_c11_dependencies():
    s = O.strassen()
    assert s.R == 7
    assert s.nnz() == (12, 12, 12)                      # P:234 ||U||_0 = 12
    # "C_{1,1} in Strassen's Algorithm depends on H1, H4, H5, and H7"
    assert set(np.nonzero(s.W[:, 0, 0])[0].tolist()) == {0, 3, 4, 6}


@pytest.mark.parametrize("make", [O.strassen, O.laderman, O.strassen2,
                                  lambda: O.standard(2, 2, 2), lambda: O.standard(3, 4, 5),
                                  lambda: O.standard(1, 1, 1)])
def test_brent_valid(make):
    s = make()
    fails, _, checked = O.brent(s)
    assert fails == 0
    assert checked == (s.m * s.k) * (s.k * s.n) * (s.m * s.n)


def test_laderman_rank_and_nnz():
    s = O.laderman()
    assert (s.m, s.k, s.n, s.R) == (3, 3, 3, 23)
    assert s.nnz() == (51, 51, 51)


def test_strassen2_rank_and_nnz():
    s = O.strassen2()
    assert (s.m, s.k, s.n, s.R) == (4, 4, 4, 49)
    assert s.nnz() == (144, 144, 144)                   # S:83 nnz multiplies


@pytest.mark.parametrize("tensor", ["U", "V", "W"])
def test_every_single_sign_flip_detected(tensor):
    # a single sign flip must be detected; we flip every nonzero in turn.
    for make in (O.strassen, O.laderman):
        s = make()
        T = getattr(s, tensor)
        for idx in zip(*np.nonzero(T)):
            T2 = T.copy()
            T2[idx] = -T2[idx]
            s2 = O.Scheme("x", s.m, s.k, s.n, *(T2 if t == tensor else getattr(s, t)
                                                 for t in "UVW"))
            fails, first, _ = O.brent(s2)
            assert fails >= 1
            assert first[6] != first[7]


def test_zero_entry_set_detected():
    s = O.strassen()
    U = s.U.copy()
    U[0, 0, 1] = 1          # A12 wrongly added into At_1
    fails, _, _ = O.brent(O.Scheme("x", 2, 2, 2, U, s.V, s.W))
    assert fails > 0


def test_w_sign_flip_failure_count():
    # flipping W[0,0,0] (H1 -> C11) breaks exactly the tuples whose observed
    # sum involves r=1 and C11: the 2 nonzero U*V products of H1 landing in C11
    # plus the cancelling cross terms -- brute force gives a fixed count.
    s = O.strassen()
    W = s.W.copy()
    W[0, 0, 0] = -1
    fails, _, _ = O.brent(O.Scheme("x", 2, 2, 2, s.U, s.V, W))
    # H1 = (A11+A22)(B11+B22) has 4 terms; each term's coefficient into C11
    # changes by -2, so exactly those 4 (i,l,l2,j,i2=0,j2=0) tuples fail.
    assert fails == 4


def test_compose_identity_and_standard():
    s = O.strassen()
    c = O.compose(s, O.standard(1, 1, 1))
    assert np.array_equal(c.U, s.U) and np.array_equal(c.V, s.V) and np.array_equal(c.W, s.W)
    st = O.compose(O.standard(2, 2, 2), O.standard(2, 2, 2))
    ref = O.standard(4, 4, 4)
    # equal up to a permutation of r: compare the multisets of (U_r,V_r,W_r)
    key = lambda sc: sorted((sc.U[r].tobytes(), sc.V[r].tobytes(), sc.W[r].tobytes())
                            for r in range(sc.R))
    assert key(st) == key(ref)
    assert O.brent(st)[0] == 0


def test_standard_scheme_shapes():
    s = O.standard(3, 4, 5)
    assert s.R == 60 and s.nnz() == (60, 60, 60)
    s = O.standard(2, 2, 2)
    assert s.R == 8 and s.nnz() == (8, 8, 8)


def test_loader_roundtrip_and_errors():
    for make in (O.strassen, O.laderman):
        s = make()
        s2 = O.load_scheme_text(O.scheme_to_text(s))
        assert np.array_equal(s.U, s2.U) and np.array_equal(s.V, s2.V) and np.array_equal(s.W, s2.W)
    txt = O.scheme_to_text(O.strassen()).splitlines()
    txt[2] = "2 0"          # first U row -> coefficient 2
    with pytest.raises(O.SchemeFileError, match="outside"):
        O.load_scheme_text("\n".join(txt))
    with pytest.raises(O.SchemeFileError, match="line 1"):
        O.load_scheme_text("2 2 x 7\n")
    txt = O.scheme_to_text(O.strassen()).splitlines()
    txt[1] = "V 1"
    with pytest.raises(O.SchemeFileError, match="line 2"):
        O.load_scheme_text("\n".join(txt))
    # comments are ignored
    s = O.load_scheme_text("# header\n" + O.scheme_to_text(O.strassen()))
    assert s.R == 7
