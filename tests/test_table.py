"""Reconstruction table (product, binary128) against the SPEC known answers,
the reproduction invariants and the independent mpmath restatement
(tests/golden/recon_golden.npz from oracle/recon_ref.py)."""
import json
import os

import numpy as np
import pytest

import paper_2401_16543_b200 as K
from paper_2401_16543_b200.table import evaluate

HERE = os.path.dirname(os.path.abspath(__file__))
SPEC = json.load(open(os.path.join(HERE, "golden", "spec_examples.json")))
GOLD = os.path.join(HERE, "golden", "recon_golden.npz")
CASES = [(2, 2), (2, 3), (3, 2), (3, 3)]


def mavg_1d(c, k):
    return ((c + 0.5) ** (k + 1) - (c - 0.5) ** (k + 1)) / (k + 1)


def graded(dim, lo, hi):
    out = []
    for n in range(lo, hi + 1):
        if dim == 2:
            out += [(n - k, k, 0) for k in range(n + 1)]
        else:
            out += [(a, b, n - a - b) for a in range(n, -1, -1) for b in range(n - a, -1, -1)]
    return out


@pytest.fixture(scope="module", params=CASES, ids=[f"d{d}r{r}" for d, r in CASES])
def rset(request):
    d, r = request.param
    return K.precompute(r, dim=d)


def test_geometry_known_answers():
    for R in (2, 3):
        rs = K.precompute(R, dim=2)
        key = f"2,{R}"
        assert [st.count for st in rs.st] == SPEC["geometry"]["substencil_sizes"][key]
        assert rs.st[0].degree == SPEC["geometry"]["degrees_full"][key]
        assert rs.n_face_points() == SPEC["geometry"]["points_total"][key]
        nf, nd = SPEC["kernel_recon"]["vector_counts"][key]
        assert rs.n_stencils * rs.n_face_points() == nf
        assert rs.n_stencils * rs.n_derivs() == nd
    rs = K.precompute(2, dim=2)
    assert all(st.degree == 1 for st in rs.st[1:])
    s2 = [tuple(c[:2]) for c in rs.cells(2)]
    assert sorted(s2) == sorted(tuple(c) for c in SPEC["geometry"]["s2_r2"]["cells"])
    cells = {tuple(c[:2]) for c in rs.offsets}
    assert all(tuple(c) in cells for c in SPEC["geometry"]["contains_r2"]["in"])
    assert all(tuple(c) not in cells for c in SPEC["geometry"]["contains_r2"]["out"])
    # lexicographic by (k, j, i) (geometry.hpp:19-21)
    keys = [(c[2], c[1], c[0]) for c in rs.offsets]
    assert keys == sorted(keys)
    # GL2 nodes/weights and exactness
    assert rs.gl_nodes[1] == pytest.approx(SPEC["geometry"]["gl2_nodes"]["value"], abs=1e-16)
    assert list(rs.gl_weights) == pytest.approx(SPEC["geometry"]["gl2_weights"]["value"], abs=1e-16)
    assert np.dot(rs.gl_weights, rs.gl_nodes ** 2) == pytest.approx(1 / 12, abs=1e-16)
    east = rs.points[2:4, :2]
    assert np.allclose(east, np.array(SPEC["geometry"]["east_face_r2"]["points"]), rtol=0, atol=1e-16)
    # 3-D counts (PAPER: 9 or 19 derivatives)
    r32, r33 = K.precompute(2, dim=3), K.precompute(3, dim=3)
    assert [st.count for st in r32.st] == [33, 7] + [11] * 6
    assert [st.count for st in r33.st] == [123, 33] + [32] * 6
    assert [st.degree for st in r32.st] == [3, 1] + [1] * 6
    assert [st.degree for st in r33.st] == [5, 3] + [2] * 6
    assert r32.n_derivs() == 9 and r33.n_derivs() == 19
    assert r32.n_face_points() == 24 and r33.n_face_points() == 54


def test_union_of_substencils_is_full(rset):
    u = set()
    for st in rset.st[1:]:
        u |= set(st.gather.tolist())
    assert u == set(range(rset.st[0].count))


def test_point_vectors_sum_to_one_and_reproduce_polynomials(rset):
    """S:221 / S:790: every (sub)stencil x face point reproduces cell-averaged
    monomials up to its degree to < 1e-9 (unit-cell scale)."""
    dim = rset.dim
    worst = 0.0
    for st in rset.st:
        cells = rset.offsets[st.gather]
        assert np.abs(st.face.sum(axis=1) - 1.0).max() < 1e-12
        for m in graded(dim, 0, st.degree):
            g = np.array([np.prod([mavg_1d(float(c[a]), m[a]) for a in range(dim)]) for c in cells])
            exact = np.array([np.prod([x[a] ** m[a] for a in range(dim)]) for x in rset.points])
            worst = max(worst, np.abs(st.face @ g - exact).max())
    assert worst < SPEC["kernel_recon"]["reproduction_tol_point"]["value"]


def test_derivative_vectors_reproduce(rset):
    """derivative vectors reproduce monomial derivatives at 0 to 1e-8."""
    dim = rset.dim
    from math import factorial
    worst = 0.0
    for st in rset.st:
        cells = rset.offsets[st.gather]
        for m in graded(dim, 0, st.degree):
            g = np.array([np.prod([mavg_1d(float(c[a]), m[a]) for a in range(dim)]) for c in cells])
            for ia, al in enumerate(rset.alphas):
                exact = float(np.prod([factorial(al[a]) for a in range(3)])) if tuple(al) == tuple(m) else 0.0
                worst = max(worst, abs(float(st.deriv[ia] @ g) - exact))
    assert worst < SPEC["kernel_recon"]["reproduction_tol_deriv"]["value"]


def test_x2_on_full_r2_stencil_at_east_point():
    """g = averages of x^2 on the R=2 full stencil, x* = (1/2, 0) -> 1/4.
    The face points sit at (1/2, +-1/(2 sqrt 3)); x^2 does not depend on y."""
    rs = K.precompute(2, dim=2)
    cells = rs.offsets[rs.st[0].gather]
    g = np.array([mavg_1d(float(c[0]), 2) for c in cells])
    for s in (2, 3):  # east face
        assert evaluate(rs.st[0].face_row(s), g) == pytest.approx(0.25, abs=1e-13)
    with pytest.raises(ValueError):
        evaluate(rs.st[0].face_row(2), g[:-1])


def test_linear_weights(rset):
    g = rset.gamma
    assert g.sum() == pytest.approx(1.0, abs=1e-15)
    ref = SPEC["weno"]["gamma_2d" if rset.dim == 2 else "gamma_3d"]["value"]
    assert g.tolist() == pytest.approx(ref, rel=1e-14)


def _group(dim):
    """Signed axis permutations g(x)_b = s_b x_pi(b) of the square / cube."""
    import itertools
    for perm in itertools.permutations(range(dim)):
        for signs in itertools.product((1, -1), repeat=dim):
            yield tuple(perm) + tuple(range(dim, 3)), tuple(signs) + (1,) * (3 - dim)


def test_exact_symmetry_every_group_element(rset):
    """kernel_recon.hpp:105-106 / S:223: the vector of a mirrored or rotated
    quadrature point (derivative) on the image (sub)stencil is EXACTLY the
    permuted original (derivatives: times the sign of the odd flipped orders),
    for every element of the square's / cube's symmetry group (x, y, z mirrors
    and axis swaps) — tolerance 0."""
    dim = rset.dim
    pos = {tuple(o): h for h, o in enumerate(rset.offsets)}
    members = [sorted(st.gather.tolist()) for st in rset.st]
    pts = rset.points
    n_el = 0
    for perm, sg in _group(dim):
        n_el += 1
        gcell = {h: pos[tuple(sg[b] * rset.offsets[h][perm[b]] for b in range(3))]
                 for h in range(len(rset.offsets))}
        for q, st in enumerate(rset.st):
            img = sorted(gcell[h] for h in st.gather)
            q2 = members.index(img)
            st2 = rset.st[q2]
            loc2 = {h: i for i, h in enumerate(st2.gather)}
            perm_l = [loc2[gcell[h]] for h in st.gather]
            for s in range(len(pts)):
                x2 = [sg[b] * pts[s][perm[b]] for b in range(3)]
                s2 = int(np.argmin(np.abs(pts - x2).sum(1)))
                assert np.abs(pts[s2] - x2).max() < 1e-15
                out = np.empty(st2.count)
                out[perm_l] = st.face[s]
                assert np.array_equal(out, st2.face[s2]), (perm, sg, q, s)
            al = [tuple(a) for a in rset.alphas]
            for a, alpha in enumerate(al):
                a2 = tuple(alpha[perm[b]] for b in range(3))
                sign = np.prod([sg[b] for b in range(3) if a2[b] % 2])
                out = np.empty(st2.count)
                out[perm_l] = sign * st.deriv[a]
                assert np.array_equal(out, st2.deriv[al.index(a2)]), (perm, sg, q, alpha)
    assert n_el == (8 if dim == 2 else 48)


def test_golden_mpmath_vectors():
    """The binary128 table equals the independent 40-digit mpmath restatement
    (oracle/recon_ref.py) rounded to FP64."""
    if not os.path.exists(GOLD):
        pytest.skip("tests/golden/recon_golden.npz not generated (tools/make_golden.py)")
    gold = np.load(GOLD)
    keys = sorted({k.rsplit("_", 1)[0] for k in gold.files})
    assert keys
    for key in keys:
        dim, R, q = int(key[1]), int(key[3]), int(key[5:])
        st = K.precompute(R, dim=dim).st[q]
        assert int(gold[key + "_degree"]) == st.degree
        cells = K.precompute(R, dim=dim).offsets[st.gather]
        assert np.array_equal(gold[key + "_cells"][:, :dim], cells[:, :dim])
        F = gold[key + "_face"]
        ulp = np.abs(F.view(np.int64) - st.face.view(np.int64))
        assert ulp.max() <= 1, (key, ulp.max())
        assert np.abs(gold[key + "_deriv"] - st.deriv).max() < 1e-14, key


def test_deterministic_and_hashed():
    a = K.ReconstructionSet(2, dim=3)
    b = K.ReconstructionSet(2, dim=3)
    assert a.hash == b.hash
    assert all(np.array_equal(x.face, y.face) and np.array_equal(x.deriv, y.deriv)
               for x, y in zip(a.st, b.st))


def test_invalid_radius_raises():
    with pytest.raises(ValueError):
        K.ReconstructionSet(4, dim=2)
    with pytest.raises(ValueError):
        K.ReconstructionSet(2, dim=1)
