"""Pins of the oracle's stationary solve (readings R19, R28): the state of
the machine at rest, 0 = (A + B_env) T + b_env (uncoupled parts), optionally with the
interface coupling and friction of a time t.  Pinned by closed-form 1-D steady states (the
exact solution is piecewise linear, which P1 elements reproduce exactly), uniform states,
and the global heat balance (boundary outflow = friction input)."""
import numpy as np
import pytest

import oracle as O
from paper_1707_03581_b200 import inputs as I

from test_oracle_stepping import two_slab_closed_form


def _slab_pair(jitter):
    """Rail slab 0.3 x 0.2 x 0.1 with Robin on the floor (tag 3) and on its top face (tag 1),
    insulated sides; a separate stock box above with Robin on its top only (tag 2).  No
    interface faces."""
    def rail_tags(axis, side, c):
        t = np.full(c.shape[0], I.TAG_INSULATED, dtype=np.int32)
        if axis == 2:
            t[:] = I.TAG_FLOOR if side == 0 else I.TAG_ENV
        return t

    def stock_tags(axis, side, c):
        t = np.full(c.shape[0], I.TAG_INSULATED, dtype=np.int32)
        if axis == 2 and side == 1:
            t[:] = I.TAG_COOL
        return t
    f = I.kuhn_box_union((0, 0, 0), (0.05, 0.05, 0.025), (6, 4, 4), [(0, 6, 0, 4, 0, 4)], rail_tags, jitter, 3)
    m = I.kuhn_box_union((0, 0, 0.2), (0.06, 0.05, 0.05), (5, 4, 2), [(0, 5, 0, 4, 0, 2)], stock_tags, jitter, 4)
    return f, m


@pytest.mark.parametrize("jitter", [0.0, 0.1])
@pytest.mark.parametrize("solver", ["cg", "cholesky"])
def test_linear_profile_between_two_robin_faces(jitter, solver):
    """1-D conduction through the rail slab between Robin (50, 24) below and Robin (10, 30) on
    top: T(z) = a + b z with nu b = ab (a - Tb) and -nu b = at (a + b H - Tt); the stock,
    cooled only on top, sits at T2 = 18 everywhere."""
    f, m = _slab_pair(jitter)
    nu, H = 50.0, 0.1
    ab, Tb, at, Tt = 50.0, 24.0, 10.0, 30.0
    robin = [I.Robin(0, I.TAG_FLOOR, ab, Tb), I.Robin(0, I.TAG_ENV, at, Tt), I.Robin(1, I.TAG_COOL, 200.0, 18.0)]
    o = O.Oracle(f, m, nu, 3.6e6, 1000.0, robin=robin)
    T, st = o.stationary(np.full(o.n, 20.0), 0.0, I.Scenario(0.0, 0.0, 1.0, 0.0), False, solver=solver)
    a, b = np.linalg.solve(np.array([[ab, -nu], [at, nu + at * H]]), np.array([ab * Tb, at * Tt]))
    expect = np.concatenate([a + b * f.xyz[:, 2], np.full(m.n_nodes, 18.0)])
    assert abs(T - expect).max() < 1e-10, abs(T - expect).max()
    if solver == "cg":
        assert st[2] < 1e-11


@pytest.mark.parametrize("jitter", [0.0, 0.1])
def test_two_slab_uncoupled_is_uniform(jitter):
    """Without coupling (reading R19) each slab relaxes to its only Robin temperature."""
    f, m = I.two_slab_pair(jitter=jitter)
    robin = [I.Robin(0, I.TAG_FLOOR, 50.0, 24.0), I.Robin(1, I.TAG_COOL, 200.0, 18.0)]
    o = O.Oracle(f, m, 50.0, 3.6e6, 1000.0, robin=robin)
    T, _ = o.stationary(np.full(o.n, 21.0), 0.0, I.Scenario(0.0, 0.0, 1.0, 500.0), False)
    expect = np.where(np.arange(o.n) < o.nf, 24.0, 18.0)
    assert abs(T - expect).max() < 1e-10


@pytest.mark.parametrize("jitter", [0.0, 0.1])
@pytest.mark.parametrize("eta", [0.0, 500.0])
def test_two_slab_coupled_closed_form(jitter, eta):
    """With coupling and friction (reading R28): the analytic two-slab profile with contact
    conductance alpha and eta/2 into each side (derived in test_oracle_stepping from P:23-45)."""
    f, m = I.two_slab_pair(jitter=jitter)
    robin = [I.Robin(0, I.TAG_FLOOR, 50.0, 24.0), I.Robin(1, I.TAG_COOL, 200.0, 18.0)]
    o = O.Oracle(f, m, 50.0, 3.6e6, 1000.0, robin=robin)
    T, _ = o.stationary(np.full(o.n, 24.0), 0.0, I.Scenario(0.0, 0.0, 1.0, eta), True)
    Tbot, T1, T2, Ttop = two_slab_closed_form(0.1, 0.1, 50.0, 1000.0, eta, 50.0, 24.0, 200.0, 18.0)
    z = np.concatenate([f.xyz[:, 2], m.xyz[:, 2]])
    expect = np.where(np.arange(o.n) < o.nf, Tbot + (T1 - Tbot) * z / 0.1, T2 + (Ttop - T2) * (z - 0.1) / 0.1)
    assert abs(T - expect).max() < 1e-10


@pytest.mark.parametrize("coupled", [False, True])
def test_global_heat_balance(coupled):
    """At steady state the Robin outflow balances the friction input: 1^T (B_env T + b_env)
    + eta |Gamma_R| = 0 (1^T A = 0 and 1^T K_G = 0 by the row-sum pins); uncoupled, per part."""
    cfg = I.make_config("small")
    o = O.Oracle.from_config(cfg)
    sc = cfg.scenarios[0]
    t = 3.0
    T, st = o.stationary(np.full(o.n, cfg.T0), t, sc, coupled)
    rp, col, A, B, ML, benv = o.volume()
    BT = np.zeros(o.n)
    for i in range(o.n):
        BT[i] = B[rp[i]:rp[i + 1]] @ T[col[rp[i]:rp[i + 1]]]
    flux = BT + benv
    scale = np.abs(benv).sum()
    if coupled:
        s_t, eta_t = I.scenario_scalars(sc, t)
        area = o.interface((s_t * sc.dir[0], s_t * sc.dir[1], s_t * sc.dir[2]), eta_t)[4]
        assert abs(flux.sum() + eta_t * area) < 1e-9 * scale
    else:
        assert abs(flux[:o.nf].sum()) < 1e-9 * scale and abs(flux[o.nf:].sum()) < 1e-9 * scale


def test_implicit_euler_with_huge_step_approaches_stationary():
    """(M_L - dt K) T = M_L T0 + dt b tends to -K T = b as dt -> infinity: one IE step with
    dt = 1e9 s from the stationary state moves it by O(rho Cp h^2 / (nu dt))."""
    cfg = I.make_config("small")
    o = O.Oracle.from_config(cfg)
    sc = I.Scenario(0.375, 0.0, 60.0, 500.0)
    Ts, _ = o.stationary(np.full(o.n, cfg.T0), 7.0, sc, True)
    Tie, _ = o.step(np.full(o.n, cfg.T0), 6.0, 1e9, 1, sc)
    assert abs(Tie - Ts).max() < 1e-4 * abs(Ts - cfg.T0).max()
