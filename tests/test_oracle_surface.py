"""Pins of the oracle's surface terms: Robin B_env, b_env and the interface
operator M_B, C_B, b(t) on Gamma_R(t), against exact polynomial integrals and
invariants.  Expected values are computed here from closed forms, never by the oracle.
"""
import math

import numpy as np
import pytest
import scipy.sparse as sp

import oracle as O
from paper_1707_03581_b200 import inputs as I

ALPHA = 1000.0


def rect_int_lin_lin(a, b, x0, x1, y0, y1):
    """Exact int_{[x0,x1]x[y0,y1]} (a0 + a1 x + a2 y)(b0 + b1 x + b2 y) dx dy."""
    def m(i, j):
        return ((x1 ** (i + 1) - x0 ** (i + 1)) / (i + 1)) * ((y1 ** (j + 1) - y0 ** (j + 1)) / (j + 1))
    # monomials: 1, x, y
    e = [(0, 0), (1, 0), (0, 1)]
    tot = 0.0
    for p in range(3):
        for q in range(3):
            tot += a[p] * b[q] * m(e[p][0] + e[q][0], e[p][1] + e[q][1])
    return tot


def _csr(rp, col, val, n):
    return sp.csr_matrix((val, col, rp), shape=(n, n))


# ---------------------------------------------------------------------------- Robin

def test_robin_sums_closed_form_cfg0():
    """sum_ij B = -sum alpha_i |Gamma_i|; sum b_env = sum alpha_i int T_i dS with
    T_1 = 24 + 0.25 z exact over each box face (BJ cfg 0)."""
    c = I.make_config("cfg0")
    o = O.Oracle.from_config(c)
    rp, col, A, B, ML, benv = o.volume()
    nf = o.nf
    Bm = _csr(rp, col, B, o.n)
    # fixed rail [0,1]x[0,.2]x[0,.1]: env faces x=0,1 (0.2x0.1) and y=0,.2 (1x0.1), floor z=0
    env_f = 2 * 0.2 * 0.1 + 2 * 1.0 * 0.1
    floor = 1.0 * 0.2
    sumB_f = Bm[:nf, :nf].sum()
    assert abs(sumB_f - (-(10.0 * env_f + 50.0 * floor))) < 1e-12
    Tmid = 24.0 + 0.25 * 0.05          # linear T_1 averaged over a face spanning z in [0,.1]
    benv_f = 10.0 * env_f * Tmid + 50.0 * floor * 24.0
    assert abs(benv[:nf].sum() - benv_f) < 1e-10
    # moving stock 0.25x0.2x0.1 at z in [.1,.2]: env faces x (0.2x0.1) x2, y=0 (0.25x0.1),
    # top z=.2 (0.25x0.2); cooling y=.2 face (0.25x0.1), T_2 = 18
    env_m = 2 * 0.2 * 0.1 + 0.25 * 0.1 + 0.25 * 0.2
    cool = 0.25 * 0.1
    assert abs(Bm[nf:, nf:].sum() - (-(10.0 * env_m + 200.0 * cool))) < 1e-12
    benv_m = 10.0 * (2 * 0.2 * 0.1 + 0.25 * 0.1) * (24 + 0.25 * 0.15) + 10.0 * 0.25 * 0.2 * (24 + 0.25 * 0.2) \
        + 200.0 * cool * 18.0
    assert abs(benv[nf:].sum() - benv_m) < 1e-10


def test_robin_consistent_surface_mass_floor_stencil():
    """Unjittered floor (z = 0) lattice hx x hy split along (0,0)-(1,1): an interior floor
    node has B_ii = -alpha hx hy / 2 (6 triangles x S/6), x-edge and diagonal-edge entries
    -alpha hx hy / 12 (2 triangles x S/12), anti-diagonal 0 (consistent mass S/12 (1+d))."""
    f, m = I.rail_pair((8, 4, 2), (2, 2, 2))
    o = O.Oracle(f, m, 50.0, 3.6e6, ALPHA, robin=[I.Robin(0, I.TAG_FLOOR, 50.0, 24.0)])
    rp, col, A, B, ML, benv = o.volume()
    Bm = _csr(rp, col, B, o.n).toarray()
    hx, hy = 1.0 / 8, 0.2 / 4
    nxn = 9
    r = 3 + nxn * 2        # interior floor node (i=3, j=2, k=0)
    assert abs(Bm[r, r] + 50.0 * hx * hy / 2) < 1e-14
    assert abs(Bm[r, r + 1] + 50.0 * hx * hy / 12) < 1e-14
    assert abs(Bm[r, r + nxn] + 50.0 * hx * hy / 12) < 1e-14
    assert abs(Bm[r, r + nxn + 1] + 50.0 * hx * hy / 12) < 1e-14
    assert abs(Bm[r, r + nxn - 1]) < 1e-15
    assert abs(benv[r] - 50.0 * 24.0 * hx * hy) < 1e-12  # 6 faces x alpha T S/3


def test_robin_linear_exactness():
    """u^T B v = -alpha int_{floor} u v for linear u, v (consistent surface mass is exact)."""
    f, m = I.rail_pair((8, 4, 2), (2, 2, 2), jitter=0.1, seed=5)
    o = O.Oracle(f, m, 50.0, 3.6e6, ALPHA, robin=[I.Robin(0, I.TAG_FLOOR, 50.0, 24.0)])
    rp, col, A, B, ML, benv = o.volume()
    Bm = _csr(rp, col, B, o.n)
    a, b = (1.0, 2.0, -3.0), (0.5, -1.0, 4.0)
    x = np.zeros((o.n, 3))
    x[:o.nf] = f.xyz
    u = a[0] + a[1] * x[:, 0] + a[2] * x[:, 1]
    v = b[0] + b[1] * x[:, 0] + b[2] * x[:, 1]
    u[o.nf:] = 0
    v[o.nf:] = 0
    exact = rect_int_lin_lin(a, b, 0.0, 1.0, 0.0, 0.2)
    assert abs(u @ (Bm @ v) + 50.0 * exact) < 1e-11 * abs(50.0 * exact)


# ---------------------------------------------------------------------------- interface

def _pair(jitter, rail=(16, 4, 2), stock=(5, 3, 2), seed=1707):
    f, m = I.rail_pair(rail, stock, jitter=jitter, seed=seed)
    return f, m, O.Oracle(f, m, 50.0, 3.6e6, ALPHA)


@pytest.mark.parametrize("jitter", [0.0, 0.1])
@pytest.mark.parametrize("x0", [0.0, 0.375, 0.6346, 0.75, 0.123456])
def test_interface_area_rowsum_friction(jitter, x0):
    """|Gamma_R| = 0.25 x 0.2 at every offset (stock always on the rail); rows of
    M_B + C_B sum to 0 (partition of unity of the other side); 1^T b_X = eta |Gamma_R| / 2
    on each side."""
    f, m, o = _pair(jitter)
    eta = 500.0
    rp, col, val, bG, area = o.interface((x0, 0.0, 0.0), eta)
    assert abs(area - 0.05) < 1e-15
    K = _csr(rp, col, val, o.n)
    assert abs(K @ np.ones(o.n)).max() < 1e-15 * ALPHA
    assert abs(bG[:o.nf].sum() - eta * 0.05 / 2) < 1e-13
    assert abs(bG[o.nf:].sum() - eta * 0.05 / 2) < 1e-13


@pytest.mark.parametrize("jitter", [0.0, 0.1])
@pytest.mark.parametrize("x0", [0.0, 0.31, 0.75])
def test_interface_linear_exactness(jitter, x0):
    """u^T C_B v = alpha int_{Gamma_R} u v, u^T M_B,fix u' = -alpha int u u' and
    v^T M_B,mov v' = -alpha int v v' for linear fields (exact polynomial integrals over the
    rectangle Gamma_R = [x0, x0+.25] x [0, .2])."""
    f, m, o = _pair(jitter)
    rp, col, val, bG, area = o.interface((x0, 0.0, 0.0), 0.0)
    K = _csr(rp, col, val, o.n)
    nf = o.nf
    a, a2, b, b2 = (1.0, 2.0, -3.0), (0.3, -1.0, 2.0), (0.5, -1.0, 4.0), (2.0, 0.7, -0.2)
    xf = f.xyz
    xm = m.xyz + np.array([x0, 0.0, 0.0])   # current position of the stock nodes

    def lin(c, x):
        return c[0] + c[1] * x[:, 0] + c[2] * x[:, 1]
    U = np.zeros(o.n)
    U[:nf] = lin(a, xf)
    U2 = np.zeros(o.n)
    U2[:nf] = lin(a2, xf)
    V = np.zeros(o.n)
    V[nf:] = lin(b, xm)
    V2 = np.zeros(o.n)
    V2[nf:] = lin(b2, xm)
    box = (x0, x0 + 0.25, 0.0, 0.2)
    tol = 1e-12
    ex = rect_int_lin_lin(a, b, *box)
    assert abs(U @ (K @ V) - ALPHA * ex) < tol * ALPHA * abs(ex)
    assert abs(V @ (K @ U) - ALPHA * ex) < tol * ALPHA * abs(ex)
    ex = rect_int_lin_lin(a, a2, *box)
    assert abs(U @ (K @ U2) + ALPHA * ex) < tol * ALPHA * abs(ex)
    ex = rect_int_lin_lin(b, b2, *box)
    assert abs(V @ (K @ V2) + ALPHA * ex) < tol * ALPHA * abs(ex)


@pytest.mark.parametrize("shift_cells", [1, 3, 6])
def test_interface_matching_meshes(shift_cells):
    """Matching lattices with an offset in h Z: the cross block equals -M_B,fix on the
    matched nodes, i.e. alpha x consistent surface mass (SURVEY 8(c) pins)."""
    # rail 8x2 cells of 0.1 on top, stock 2x2 cells of 0.1 -> identical triangulations
    f = I.kuhn_box_union((0, 0, 0), (0.1, 0.1, 0.1), (8, 2, 1), [(0, 8, 0, 2, 0, 1)],
                         lambda ax, s, c: np.full(c.shape[0], 4 if (ax == 2 and s == 1) else 1, np.int32))
    m = I.kuhn_box_union((0, 0, 0.1), (0.1, 0.1, 0.1), (2, 2, 1), [(0, 2, 0, 2, 0, 1)],
                         lambda ax, s, c: np.full(c.shape[0], 4 if (ax == 2 and s == 0) else 1, np.int32))
    o = O.Oracle(f, m, 50.0, 3.6e6, ALPHA)
    x0 = 0.1 * shift_cells
    rp, col, val, bG, area = o.interface((x0, 0.0, 0.0), 0.0)
    K = _csr(rp, col, val, o.n).toarray()
    nf = o.nf
    # match each stock-bottom node to the rail-top node at the same position
    bot = np.nonzero(np.abs(m.xyz[:, 2] - 0.1) < 1e-12)[0]
    top = np.nonzero(np.abs(f.xyz[:, 2] - 0.1) < 1e-12)[0]
    match = {}
    for j in bot:
        p = m.xyz[j, :2] + np.array([x0, 0.0])
        d = np.linalg.norm(f.xyz[top, :2] - p, axis=1)
        match[j] = top[np.argmin(d)]
        assert d.min() < 1e-12
    for j in bot:
        for j2 in bot:
            c = K[match[j], nf + j2]
            mb = K[match[j], match[j2]]
            assert abs(c + mb) < 1e-12 * ALPHA
    # consistent surface mass: diagonal of an interior stock-bottom node = 6 * S/6 * alpha
    S = 0.1 * 0.1 / 2
    centre = [j for j in bot if abs(m.xyz[j, 0] - 0.1) < 1e-12 and abs(m.xyz[j, 1] - 0.1) < 1e-12][0]
    assert abs(K[match[centre], nf + centre] - ALPHA * 6 * S / 6) < 1e-12 * ALPHA
    assert abs(K[nf + centre, nf + centre] + ALPHA * 6 * S / 6) < 1e-12 * ALPHA


def test_interface_partial_overlap_single_pair():
    """One rail triangle and one stock triangle overlapping in a known triangle: the
    integrals of products of linear fields equal the P1 mass formula
    int_tau g h = |tau|/12 (sum g_i h_i + sum g_i sum h_i) on the overlap tau."""
    tag_top = lambda ax, s, c: np.full(c.shape[0], 4 if (ax == 2 and s == 1) else 0, np.int32)
    tag_bot = lambda ax, s, c: np.full(c.shape[0], 4 if (ax == 2 and s == 0) else 0, np.int32)
    f = I.kuhn_box_union((0, 0, 0), (1.0, 1.0, 1.0), (1, 1, 1), [(0, 1, 0, 1, 0, 1)], tag_top)
    m = I.kuhn_box_union((0, 0, 1.0), (1.0, 1.0, 1.0), (1, 1, 1), [(0, 1, 0, 1, 0, 1)], tag_bot)
    o = O.Oracle(f, m, 1.0, 1.0, 1.0)
    x0 = 0.5
    rp, col, val, bG, area = o.interface((x0, 0.0, 0.0), 0.0)
    # overlap of [0,1]^2 with [.5,1.5]x[0,1] = [.5,1]x[0,1] (both split along the diagonal)
    assert abs(area - 0.5) < 1e-15
    K = _csr(rp, col, val, o.n)
    # linear u on the fixed part, v on the moving part: int over [.5,1]x[0,1]
    a, b = (1.0, 2.0, -1.0), (3.0, -1.0, 0.5)
    U = np.zeros(o.n)
    U[:o.nf] = a[0] + a[1] * f.xyz[:, 0] + a[2] * f.xyz[:, 1]
    V = np.zeros(o.n)
    xm = m.xyz + np.array([x0, 0, 0])
    V[o.nf:] = b[0] + b[1] * xm[:, 0] + b[2] * xm[:, 1]
    # split the rectangle [.5,1]x[0,1] into two triangles and use the P1 mass formula
    tris = [np.array([[0.5, 0], [1, 0], [1, 1]]), np.array([[0.5, 0], [1, 1], [0.5, 1]])]
    tot = 0.0
    for t in tris:
        ar = 0.5 * abs((t[1, 0] - t[0, 0]) * (t[2, 1] - t[0, 1]) - (t[1, 1] - t[0, 1]) * (t[2, 0] - t[0, 0]))
        g = a[0] + a[1] * t[:, 0] + a[2] * t[:, 1]
        h = b[0] + b[1] * t[:, 0] + b[2] * t[:, 1]
        tot += ar / 12.0 * (g @ h + g.sum() * h.sum())
    assert abs(U @ (K @ V) - tot) < 1e-14 * abs(tot)
