"""Pins of the oracle's volume assembly (M_L, A) against closed forms and invariants.

Paper: M_X = int phi phi (lumped; rho*Cp factor = reading R1), A_X = -nu int
grad phi . grad phi.  None of these expected values come from the oracle itself.
"""
import numpy as np
import pytest
import scipy.sparse as sp

import oracle as O
from paper_1707_03581_b200 import inputs as I

NU, RHO_CP = 50.0, 3.6e6


def _csr(rp, col, val, n):
    return sp.csr_matrix((val, col, rp), shape=(n, n))


def _box(cells, size, jitter=0.0, seed=3, origin=(0.0, 0.0, 0.0)):
    nx, ny, nz = cells
    h = (size[0] / nx, size[1] / ny, size[2] / nz)
    return I.kuhn_box_union(origin, h, cells, [(0, nx, 0, ny, 0, nz)],
                            lambda a, s, c: np.full(c.shape[0], 1, np.int32), jitter, seed)


def _single_tet():
    # reference tetrahedron (0,0,0),(1,0,0),(0,1,0),(0,0,1); one face tagged 4 so that the
    # oracle sees an (empty) interface plane
    m = I.Mesh(xyz=np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1.0]]),
               tets=np.array([[0, 1, 2, 3]], np.int32),
               bfaces=np.array([[0, 2, 1], [0, 1, 3], [0, 3, 2], [1, 2, 3]], np.int32),
               bface_tag=np.array([4, 0, 0, 0], np.int32))
    return m


def _oracle(fixed, moving=None, **kw):
    if moving is None:
        moving = _box((1, 1, 1), (0.1, 0.1, 0.1), origin=(5.0, 5.0, 5.0))
    return O.Oracle(fixed, moving, kw.get("nu", NU), kw.get("rho_cp", RHO_CP), 1000.0)


def test_single_tet_closed_form():
    """Reference tet: V = 1/6, M_L = rho Cp V/4 per node; A = -nu V grad.grad with
    grad lambda = (-1,-1,-1), e1, e2, e3  ->  -nu/6 [[3,-1,-1,-1],[-1,1,0,0],...]."""
    o = _oracle(_single_tet())
    rp, col, A, B, ML, benv = o.volume()
    Am = _csr(rp, col, A, o.n).toarray()[:4, :4]
    expect = -NU / 6.0 * np.array([[3, -1, -1, -1], [-1, 1, 0, 0], [-1, 0, 1, 0], [-1, 0, 0, 1.0]])
    np.testing.assert_allclose(Am, expect, rtol=0, atol=1e-13)
    np.testing.assert_allclose(ML[:4], RHO_CP / 24.0, rtol=1e-15)


@pytest.mark.parametrize("jitter", [0.0, 0.1])
def test_lumped_mass_sums_to_volume(jitter):
    """sum_i M_L,ii / (rho Cp) = domain volume (north star invariant; jitter keeps the
    boundary, so the volume is exact)."""
    f = _box((6, 5, 4), (0.3, 0.2, 0.1), jitter=jitter)
    m = _box((3, 3, 2), (0.1, 0.1, 0.05), jitter=jitter, origin=(0.0, 0.0, 0.1))
    o = _oracle(f, m)
    ML = o.volume()[4]
    assert abs(ML[:o.nf].sum() / RHO_CP - 0.3 * 0.2 * 0.1) < 1e-15
    assert abs(ML[o.nf:].sum() / RHO_CP - 0.1 * 0.1 * 0.05) < 1e-16


def test_lshape_volume():
    fixed, moving = I.lshape_pair(0.05, 0.05, jitter=0.1)
    o = _oracle(fixed, moving)
    ML = o.volume()[4]
    vol = 0.6 * 0.6 * 2.0 + 1.5 * 0.6 * 0.25 + 1.5 * 0.2 * 0.1
    assert abs(ML[:o.nf].sum() / RHO_CP - vol) < 1e-12


@pytest.mark.parametrize("jitter", [0.0, 0.1])
def test_stiffness_rows_sum_to_zero_symmetric_nsd(jitter):
    f = _box((6, 5, 4), (0.3, 0.2, 0.1), jitter=jitter)
    o = _oracle(f)
    rp, col, A, B, ML, benv = o.volume()
    Am = _csr(rp, col, A, o.n)
    scale = abs(A).max()
    assert abs(Am @ np.ones(o.n)).max() < 1e-13 * scale
    assert abs(Am - Am.T).max() < 1e-14 * scale
    rng = np.random.default_rng(0)
    for _ in range(5):
        x = rng.standard_normal(o.n)
        assert x @ (Am @ x) <= 1e-12 * scale * (x @ x)


def test_kuhn_seven_point_stencil():
    """Unjittered Kuhn P1 on a lattice (hx, hy, hz): interior rows are the 7-point stencil
    diag = -2 nu (hy hz/hx + hx hz/hy + hx hy/hz), axis neighbour x: nu hy hz/hx (etc.),
    face/body-diagonal neighbours 0; interior M_L = rho Cp hx hy hz."""
    cells = (5, 4, 3)
    size = (0.5, 0.2, 0.09)
    hx, hy, hz = size[0] / cells[0], size[1] / cells[1], size[2] / cells[2]
    o = _oracle(_box(cells, size))
    rp, col, A, B, ML, benv = o.volume()
    Am = _csr(rp, col, A, o.n).toarray()
    nxn, nyn = cells[0] + 1, cells[1] + 1
    for (i, j, k) in [(2, 2, 1), (1, 1, 1), (3, 2, 2)]:
        r = i + nxn * (j + nyn * k)
        row = Am[r, :o.nf]
        assert abs(row[r] + 2 * NU * (hy * hz / hx + hx * hz / hy + hx * hy / hz)) < 1e-12
        assert abs(row[r + 1] - NU * hy * hz / hx) < 1e-12
        assert abs(row[r - 1] - NU * hy * hz / hx) < 1e-12
        assert abs(row[r + nxn] - NU * hx * hz / hy) < 1e-12
        assert abs(row[r + nxn * nyn] - NU * hx * hy / hz) < 1e-12
        others = np.delete(row, [r, r - 1, r + 1, r - nxn, r + nxn, r - nxn * nyn, r + nxn * nyn])
        assert abs(others).max() < 1e-12
        assert abs(ML[r] - RHO_CP * hx * hy * hz) < 1e-9


def test_patch_test_linear_field():
    """A u = 0 on interior rows for a linear field u (patch test), jittered mesh."""
    f = _box((6, 5, 4), (0.3, 0.2, 0.1), jitter=0.1)
    o = _oracle(f)
    rp, col, A, B, ML, benv = o.volume()
    Am = _csr(rp, col, A, o.n)
    x = np.concatenate([f.xyz, np.zeros((o.n - o.nf, 3))])
    u = 1.0 + 2.0 * x[:, 0] - 3.0 * x[:, 1] + 0.5 * x[:, 2]
    u[o.nf:] = 0.0
    interior = np.ones(o.n, bool)
    interior[np.unique(f.bfaces)] = False
    interior[o.nf:] = False
    assert abs((Am @ u)[interior]).max() < 1e-11 * abs(A).max()


def test_cfg_counts_match_survey():
    """Node and nnz counts of cfg 0 (N = 327, Z = 3,413)."""
    c = I.make_config("cfg0")
    o = O.Oracle.from_config(c)
    assert o.n == 327 and o.nf == 255
    assert len(o.volume()[1]) == 3413
