"""Pins of the oracle's implicit-Euler stepping (reading R3: everything at
t_{n+1}) against invariants and closed forms: uniform fixed point, energy balance (north
star), the analytic two-slab steady state, dense Cholesky = CG.
"""
import math

import numpy as np
import pytest

import oracle as O
from paper_1707_03581_b200 import inputs as I


def _face_integral_linear(mesh, values, tags_alpha):
    """sum over Robin faces of alpha * int_face g dS for a nodal linear g (exact: area x mean)."""
    x = mesh.xyz
    f = mesh.bfaces
    S = 0.5 * np.linalg.norm(np.cross(x[f[:, 1]] - x[f[:, 0]], x[f[:, 2]] - x[f[:, 0]]), axis=1)
    al = np.array([tags_alpha.get(int(t), 0.0) for t in mesh.bface_tag])
    return float(np.sum(al * S * values[f].mean(axis=1)))


def test_cholesky_equals_cg_cfg0():
    c = I.make_config("cfg0")
    o = O.Oracle.from_config(c)
    T0 = np.full(o.n, c.T0)
    Tc, sc = o.step(T0, 0.0, c.dt, 5, c.scenarios[0], solver="cg")
    Td, sd = o.step(T0, 0.0, c.dt, 5, c.scenarios[0], solver="cholesky")
    assert np.all(sc[:, 2] < 2e-12)                      # true residual at exit
    # the CG stopping rule bounds the residual, not the error: error <= kappa * 1e-12
    assert abs(Tc - Td).max() / abs(Td).max() < 1e-10
    assert np.all(sd[:, 2] < 1e-14)


def test_step_equals_dense_library_solve():
    """One IE step = numpy.linalg.solve of (M_L - dt K(t1)) x = M_L T0 + dt (b_env + b_G(t1))
    with the scalars at t1 = t + dt (reading R3)."""
    c = I.make_config("cfg0")
    o = O.Oracle.from_config(c)
    sc = c.scenarios[0]
    t, dt = 3.0, 2.0
    T0 = I.initial_field(c)[0]
    T1, st = o.step(T0, t, dt, 1, sc, solver="cholesky")
    s1, eta1 = I.scenario_scalars(sc, t + dt)
    rp, col, A, B, ML, benv = o.volume()
    irp, icol, ival, bG, area = o.interface((s1, 0, 0), eta1)
    n = o.n
    K = np.zeros((n, n))
    for i in range(n):
        K[i, col[rp[i]:rp[i + 1]]] += A[rp[i]:rp[i + 1]] + B[rp[i]:rp[i + 1]]
        K[i, icol[irp[i]:irp[i + 1]]] += ival[irp[i]:irp[i + 1]]
    x = np.linalg.solve(np.diag(ML) - dt * K, ML * T0 + dt * (benv + bG))
    assert abs(x - T1).max() / abs(x).max() < 1e-13


@pytest.mark.parametrize("jitter", [0.0, 0.1])
def test_uniform_state_is_fixed_point(jitter):
    """All T_i = T0, eta = 0: T stays T0 to CG tolerance while the stock moves."""
    f, m = I.rail_pair((32, 8, 4), (10, 6, 3), jitter=jitter)
    robin = [I.Robin(0, 1, 10.0, 24.0), I.Robin(1, 1, 10.0, 24.0), I.Robin(0, 3, 50.0, 24.0),
             I.Robin(1, 2, 200.0, 24.0)]
    o = O.Oracle(f, m, 50.0, 3.6e6, 1000.0, robin=robin)
    T, st = o.step(np.full(o.n, 24.0), 0.0, 1.0, 10, I.Scenario(0.375, 0.375, 20.0, 0.0))
    assert abs(T - 24.0).max() < 1e-9


@pytest.mark.parametrize("jitter", [0.0, 0.1])
def test_energy_balance_robin_off(jitter):
    """With all Robin boundaries off: sum M_L (T^{n+1} - T^n) = dt eta(t_{n+1}) |Gamma_R|
    per step, because the alpha (T_mov - T_fix) exchange cancels (north star).  eta varies
    in time, so the time level of the friction term is pinned too."""
    f, m = I.rail_pair((32, 8, 4), (10, 6, 3), jitter=jitter)
    o = O.Oracle(f, m, 50.0, 3.6e6, 1000.0)
    ML = o.volume()[4]
    sc = I.Scenario(0.375, 0.375, 20.0, 500.0, 0.5, 7.0)
    T = np.full(o.n, 24.0)
    t, dt = 0.0, 0.5
    for n in range(6):
        T1, st = o.step(T, t + n * dt, dt, 1, sc)
        eta = sc.eta0 * (1.0 + sc.eta_amp * math.sin(2.0 * math.pi * (t + (n + 1) * dt) / sc.eta_period))
        dE = float(ML @ (T1 - T))
        assert abs(dE - dt * eta * 0.05) < 1e-7 * dt * eta * 0.05
        T = T1


def test_energy_balance_robin_on():
    """sum M_L dT = dt (eta |Gamma_R| + sum_i alpha_i int (T_i - T^{n+1}) dS) per step."""
    c = I.make_config("small")
    o = O.Oracle.from_config(c)
    ML = o.volume()[4]
    sc = c.scenarios[0]
    T = I.initial_field(c)[0]
    dt = c.dt
    nf = c.fixed.n_nodes
    xyz = np.concatenate([c.fixed.xyz, c.moving.xyz])
    for n in range(3):
        T1, st = o.step(T, n * dt, dt, 1, sc)
        eta = sc.eta0 * (1.0 + sc.eta_amp * math.sin(2.0 * math.pi * ((n + 1) * dt) / sc.eta_period))
        flux = dt * eta * 0.05
        for part, mesh, sl in ((0, c.fixed, slice(0, nf)), (1, c.moving, slice(nf, None))):
            for r in c.robin:
                if r.part != part:
                    continue
                Ta = r.T_ref + xyz[sl] @ np.array(r.grad)
                flux += dt * _face_integral_linear(mesh, Ta - T1[sl], {r.tag: r.alpha})
        dE = float(ML @ (T1 - T))
        assert abs(dE - flux) < 1e-7 * abs(flux)
        T = T1


def two_slab_closed_form(H1, H2, nu, alpha, eta, ab, Tb, at, Tt):
    """Steady 1-D two-slab profile: rail [0,H1] with Robin (ab,Tb) at the bottom,
    stock [H1,H1+H2] with Robin (at,Tt) on top, contact conductance alpha and friction
    eta/2 into each side.  Unknowns T_bot, T_1 (rail top), T_2 (stock bottom), T_top."""
    # -nu g1 = ab (Tb - Tbot) ; nu g1 = alpha (T2 - T1) + eta/2 ; -nu g2 = alpha (T1 - T2) + eta/2
    # nu g2 = at (Tt - Ttop) ; g1 = (T1 - Tbot)/H1 ; g2 = (Ttop - T2)/H2
    M = np.array([[nu / H1 + ab, -nu / H1, 0, 0],            # -nu (T1-Tbot)/H1 = ab (Tb - Tbot)
                  [-nu / H1, nu / H1 + alpha, -alpha, 0],     # nu (T1-Tbot)/H1 - alpha T2 + alpha T1 = eta/2
                  [0, -alpha, nu / H2 + alpha, -nu / H2],     # -nu (Ttop-T2)/H2 - alpha T1 + alpha T2 = eta/2
                  [0, 0, -nu / H2, nu / H2 + at]], float)     # nu (Ttop-T2)/H2 + at Ttop = at Tt
    rhs = np.array([ab * Tb, eta / 2, eta / 2, at * Tt])
    return np.linalg.solve(M, rhs)


def test_two_slab_closed_form_values():
    """The closed form reproduces the profile of the golden fixture."""
    import os
    sol = two_slab_closed_form(0.1, 0.1, 50.0, 1000.0, 500.0, 50.0, 24.0, 200.0, 18.0)
    path = os.path.join(os.path.dirname(__file__), "golden", "two_slab_profile.txt")
    gold = [float(x) for line in open(path) if not line.startswith("#") for x in line.split()]
    np.testing.assert_allclose(sol, gold, rtol=0, atol=1e-12)


@pytest.mark.parametrize("jitter", [0.0, 0.1])
def test_two_slab_steady_state(jitter):
    """IE with dt = 1e7 s converges to the analytic piecewise-linear steady state, which the
    P1 discretisation reproduces exactly (consistent boundary integrals, patch test)."""
    f, m = I.two_slab_pair(jitter=jitter)
    robin = [I.Robin(0, I.TAG_FLOOR, 50.0, 24.0), I.Robin(1, I.TAG_COOL, 200.0, 18.0)]
    o = O.Oracle(f, m, 50.0, 3.6e6, 1000.0, robin=robin)
    T, st = o.step(np.full(o.n, 24.0), 0.0, 1e7, 6, I.Scenario(0.0, 0.0, 1.0, 500.0))
    Tbot, T1, T2, Ttop = two_slab_closed_form(0.1, 0.1, 50.0, 1000.0, 500.0, 50.0, 24.0, 200.0, 18.0)
    z = np.concatenate([f.xyz[:, 2], m.xyz[:, 2]])
    expect = np.where(np.arange(o.n) < o.nf, Tbot + (T1 - Tbot) * z / 0.1, T2 + (Ttop - T2) * (z - 0.1) / 0.1)
    assert abs(T - expect).max() < 1e-10


def test_implicit_euler_stable_far_beyond_explicit_limit():
    """explicit diffusion needs dt <= rho Cp dx^2 / nu; IE stays bounded at 1e4x."""
    c = I.make_config("small")
    o = O.Oracle.from_config(c)
    h = 0.2 / 8 / 2
    dt = 1e4 * c.rho_cp * h * h / c.nu
    T, st = o.step(np.full(o.n, 24.0), 0.0, dt, 3, c.scenarios[0])
    assert np.isfinite(T).all() and T.min() > 17.0 and T.max() < 60.0


@pytest.mark.parametrize("order", [1, 2])
def test_extrapolated_start(order):
    """or_set_guess (reading R17: the CG start is not part of the method): CG from the
    extrapolated states reaches the dense-Cholesky solution of every step to the same bound as
    from T^n, with fewer iterations; the history carries across calls only from the state the
    previous call returned (15 + 15 steps = 30 steps bitwise), and a different state or dt
    restarts it (bitwise equal to a fresh oracle)."""
    c = I.make_config("cfg0")
    sc = c.scenarios[0]
    T0 = np.full(c.n_dof, c.T0)
    n = 30
    Td, _ = O.Oracle.from_config(c).step(T0, 0.0, c.dt, n, sc, solver="cholesky")
    T_0, s_0 = O.Oracle.from_config(c).step(T0, 0.0, c.dt, n, sc)
    og = O.Oracle.from_config(c, order)
    T_g, s_g = og.step(T0, 0.0, c.dt, n, sc)
    assert abs(T_0 - Td).max() / abs(Td).max() < 1e-10
    assert abs(T_g - Td).max() / abs(Td).max() < 1e-10
    assert s_g[:, 0].sum() <= s_0[:, 0].sum()
    assert np.all(s_g[:, 2] < 2e-12)                     # true residual at exit
    cs = I.make_config("small", jitter=0.1)              # large enough to save iterations
    Ts0 = np.full(cs.n_dof, cs.T0)
    _, a = O.Oracle.from_config(cs).step(Ts0, 0.0, cs.dt, 30, cs.scenarios[0])
    _, b = O.Oracle.from_config(cs, order).step(Ts0, 0.0, cs.dt, 30, cs.scenarios[0])
    assert b[:, 0].sum() < a[:, 0].sum()
    o2 = O.Oracle.from_config(c, order)
    Ta, _ = o2.step(T0, 0.0, c.dt, n // 2, sc)
    Tb, _ = o2.step(Ta, n // 2 * c.dt, c.dt, n - n // 2, sc)
    assert np.array_equal(Tb, T_g)
    # restart: another state, then another dt
    T1 = I.initial_field(c)[0]
    Tc, _ = o2.step(T1, 0.0, c.dt, 5, sc)
    Tf, _ = O.Oracle.from_config(c, order).step(T1, 0.0, c.dt, 5, sc)
    assert np.array_equal(Tc, Tf)
    Te, _ = o2.step(Tc, 5 * c.dt, 0.5 * c.dt, 4, sc)
    Tf2, _ = O.Oracle.from_config(c, order).step(Tc, 5 * c.dt, 0.5 * c.dt, 4, sc)
    assert np.array_equal(Te, Tf2)
    with pytest.raises(ValueError):
        og.set_guess(3)


def test_ie_residual_rows():
    """or_ie_residual_rows (the checker of test_cfg2_full_run_invariants) against a dense
    numpy build of the same system from the oracle's exported matrices (R3):
    (i) the residual of a dense-Cholesky step vanishes to rounding; (ii) for a perturbed state
    T1 + delta the residual rows equal (M_L - dt K) delta, row by row, on a subset of rows; (iii)
    bnorm = ||M_L T0 + dt (b_env + b_G)||_2."""
    c = I.make_config("cfg0")
    o = O.Oracle.from_config(c)
    sc = c.scenarios[0]
    t, dt = 3.0, 2.0
    T0 = I.initial_field(c)[0]
    T1, _ = o.step(T0, t, dt, 1, sc, solver="cholesky")
    s1, eta1 = I.scenario_scalars(sc, t + dt)
    off = (s1 * sc.dir[0], s1 * sc.dir[1], s1 * sc.dir[2])
    rows = np.arange(o.n, dtype=np.int64)
    res, bnorm = o.residual_rows(dt, off, eta1, T0, T1, rows)
    rp, col, A, B, ML, benv = o.volume()
    irp, icol, ival, bG, area = o.interface(off, eta1)
    n = o.n
    K = np.zeros((n, n))
    for i in range(n):
        K[i, col[rp[i]:rp[i + 1]]] += A[rp[i]:rp[i + 1]] + B[rp[i]:rp[i + 1]]
        K[i, icol[irp[i]:irp[i + 1]]] += ival[irp[i]:irp[i + 1]]
    Kt = np.diag(ML) - dt * K
    b = ML * T0 + dt * (benv + bG)
    assert abs(bnorm - np.linalg.norm(b)) <= 1e-14 * np.linalg.norm(b)
    assert np.linalg.norm(res) <= 1e-13 * bnorm
    delta = np.sin(np.arange(n) * 0.37) * 0.01
    sub = np.arange(0, n, 7, dtype=np.int64)
    res2, _ = o.residual_rows(dt, off, eta1, T0, T1 + delta, sub)
    ref = (Kt @ (T1 + delta) - b)[sub]
    assert np.abs(res2 - ref).max() <= 1e-12 * np.abs(Kt @ delta).max()
    assert np.abs(res2 - (Kt @ delta)[sub]).max() <= 1e-10 * np.abs(Kt @ delta).max()
