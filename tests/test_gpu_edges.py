"""Edge cases of the CUDA path through the C ABI: no interface at all, partial contact (the
stock overhanging the rail end), zero steps, argument errors, and the implicit-Euler limit
dt -> infinity against the analytic two-slab profile."""
import numpy as np
import pytest

import oracle as O
from paper_1707_03581_b200 import inputs as I

pytestmark = pytest.mark.gpu
TOL = 1e-9


@pytest.fixture(scope="module", autouse=True)
def _built():
    import __graft_entry__ as g
    g.build()


def rel(a, b):
    return float(np.abs(a - b).max() / np.abs(b).max())


def _slabs_without_interface():
    from test_oracle_stationary import _slab_pair
    return _slab_pair(0.1)


def test_no_interface_faces():
    """Two parts without any interface face: decoupled conduction, parity vs Cholesky."""
    from paper_1707_03581_b200.thermo import Thermo
    f, m = _slabs_without_interface()
    robin = [I.Robin(0, I.TAG_FLOOR, 50.0, 24.0), I.Robin(0, I.TAG_ENV, 10.0, 30.0),
             I.Robin(1, I.TAG_COOL, 200.0, 18.0)]
    sc = I.Scenario(0.0, 0.0, 1.0, 500.0)
    th = Thermo(f, m, 50.0, 3.6e6, 1000.0, [sc], 21.0, (4, 4), robin)
    assert th.stats()["n_iface_rows"] == 0
    th.step(0.0, 20.0, 7)
    o = O.Oracle(f, m, 50.0, 3.6e6, 1000.0, robin=robin)
    Tr, _ = o.step(np.full(o.n, 21.0), 0.0, 20.0, 7, sc, solver="cholesky")
    assert rel(th.get_T(), Tr) <= TOL
    assert th.stats()["iface_area"] == 0.0


def test_partial_contact_overhang():
    """cfg 0 geometry with the stock pushed 0.15 m past the rail end: |Gamma_R| = 0.1 x 0.2."""
    from paper_1707_03581_b200.thermo import Thermo
    cfg = I.make_config("cfg0")
    sc = I.Scenario(0.9, 0.0, 60.0, 500.0)
    cfg.scenarios = [sc]
    th = Thermo.from_config(cfg)
    th.step(0.0, cfg.dt, 10)
    Tr, _ = O.Oracle.from_config(cfg).step(np.full(cfg.n_dof, cfg.T0), 0.0, cfg.dt, 10, sc, solver="cholesky")
    assert rel(th.get_T(), Tr) <= TOL
    assert abs(th.stats()["iface_area"] - 0.02) < 1e-14


def test_zero_steps_and_argument_errors():
    from paper_1707_03581_b200.thermo import Thermo, ThermoError
    cfg = I.make_config("cfg0")
    th = Thermo.from_config(cfg)
    T0 = th.get_T()
    th.step(0.0, cfg.dt, 0)                       # no-op
    assert np.array_equal(th.get_T(), T0) and th.stats()["steps_done"] == 0
    for bad in (lambda: th.step(0.0, 0.0, 1), lambda: th.step(0.0, -1.0, 1), lambda: th.step(float("nan"), 1.0, 1),
                lambda: th.get_T(scen=1), lambda: th.get_T(part=2), lambda: th.set_solver(0.0, 0),
                lambda: th.set_method("mrsdc", 9, 2, 1)):
        with pytest.raises((ThermoError, KeyError)):
            bad()
    assert np.array_equal(th.get_T(), T0)         # failed calls leave the state alone


def test_huge_step_reaches_two_slab_profile():
    """Implicit Euler with dt = 1e7 s: the coupled two-slab steady state with
    contact conductance and friction, computed analytically (test_oracle_stepping)."""
    from test_oracle_stepping import two_slab_closed_form
    from paper_1707_03581_b200.thermo import Thermo
    f, m = I.two_slab_pair(jitter=0.1)
    robin = [I.Robin(0, I.TAG_FLOOR, 50.0, 24.0), I.Robin(1, I.TAG_COOL, 200.0, 18.0)]
    th = Thermo(f, m, 50.0, 3.6e6, 1000.0, [I.Scenario(0.0, 0.0, 1.0, 500.0)], 24.0, (4, 4), robin)
    th.step(0.0, 1e7, 6)
    Tbot, T1, T2, Ttop = two_slab_closed_form(0.1, 0.1, 50.0, 1000.0, 500.0, 50.0, 24.0, 200.0, 18.0)
    z = np.concatenate([f.xyz[:, 2], m.xyz[:, 2]])
    expect = np.where(np.arange(th.n) < th.nf, Tbot + (T1 - Tbot) * z / 0.1, T2 + (Ttop - T2) * (z - 0.1) / 0.1)
    assert np.abs(th.get_T() - expect).max() < 1e-9


def test_async_host_copies_overlap_safely():
    """thermo_get_T_async: each copy holds the state of the moment it was enqueued, even when the
    following steps overwrite the double-buffered state while the copies are in flight."""
    import torch
    from paper_1707_03581_b200.thermo import Thermo
    cfg = I.make_config("small", jitter=0.1)
    ref = Thermo.from_config(cfg)
    expect = []
    for k in range(4):
        ref.step(k * cfg.dt, cfg.dt, 1)
        expect.append(ref.get_T())
    th = Thermo.from_config(cfg)
    hosts = [torch.empty(cfg.n_dof, dtype=torch.float64, pin_memory=True) for _ in range(4)]
    for k in range(4):
        th.step(k * cfg.dt, cfg.dt, 1)
        th.get_T_async(hosts[k].data_ptr())
    th.set_T(np.zeros(cfg.n_dof))          # overwrites the current buffer: must wait for its copy
    th.sync()
    for k in range(4):
        assert np.array_equal(hosts[k].numpy(), expect[k]), k


@pytest.mark.parametrize("s0", [0.375, 0.5, 0.0])
def test_coincident_edges_and_vertices(s0):
    """Static stock whose x-edges fall exactly on rail lattice lines (cfg 0: rail h_x = 1/16,
    offsets multiples of it): degenerate overlaps (shared edges / vertices, zero-area slivers,
    reading R7) -- parity vs Cholesky and the exact contact area 0.25 x 0.2."""
    from paper_1707_03581_b200.thermo import Thermo
    cfg = I.make_config("cfg0")
    sc = I.Scenario(s0, 0.0, 60.0, 500.0)
    cfg.scenarios = [sc]
    th = Thermo.from_config(cfg)
    th.step(0.0, cfg.dt, 6)
    Tr, _ = O.Oracle.from_config(cfg).step(np.full(cfg.n_dof, cfg.T0), 0.0, cfg.dt, 6, sc, solver="cholesky")
    assert rel(th.get_T(), Tr) <= TOL
    assert abs(th.stats()["iface_area"] - 0.05) < 1e-14


def _single_tet(pts, tags):
    """One positively oriented tetrahedron with its four outward faces and their tags."""
    x = np.array(pts, dtype=np.float64)
    t = [0, 1, 2, 3]
    if np.linalg.det(np.stack([x[1] - x[0], x[2] - x[0], x[3] - x[0]])) < 0:
        t = [0, 2, 1, 3]
    faces = np.array([[t[1], t[2], t[3]], [t[0], t[3], t[2]], [t[0], t[1], t[3]], [t[0], t[2], t[1]]], np.int32)
    return I.Mesh(xyz=x, tets=np.array([t], np.int32), bfaces=faces,
                  bface_tag=np.array([tags[tuple(sorted(f))] for f in faces.tolist()], np.int32))


def test_smallest_pair_one_tet_each():
    """SURVEY 4.1's smallest real case: one tetrahedron per part (8 DoF), a triangular contact
    patch partially covered and moving, Robin floor and cooled top; GPU vs the oracle's dense
    Cholesky over a few steps (the degenerate end of every kernel: one slice, one chunk, one
    triangle per surface)."""
    # fixed tet: top face (nodes 0, 1, 2) in z = 0.1 is the contact surface, the rest is floor
    fixed = _single_tet([(0, 0, 0.1), (1, 0, 0.1), (0, 1, 0.1), (0, 0, 0)],
                        {(0, 1, 2): 4, (0, 1, 3): 3, (0, 2, 3): 3, (1, 2, 3): 3})
    # moving tet: bottom face (nodes 0, 1, 2) in z = 0.1, the others cooled
    moving = _single_tet([(0.1, 0.1, 0.1), (0.6, 0.1, 0.1), (0.1, 0.6, 0.1), (0.1, 0.1, 0.4)],
                         {(0, 1, 2): 4, (0, 1, 3): 2, (0, 2, 3): 2, (1, 2, 3): 2})
    cfg = I.make_config("cfg0")
    cfg.fixed, cfg.moving = fixed, moving
    cfg.robin = [I.Robin(0, 3, 50.0, 24.0), I.Robin(1, 2, 200.0, 18.0)]
    cfg.scenarios = [I.Scenario(0.2, 0.2, 8.0, 500.0, 0.5, 3.0)]   # partly off the fixed triangle
    from paper_1707_03581_b200.thermo import Thermo
    th = Thermo.from_config(cfg)
    th.step(0.0, 1.0, 6)
    Tr, st = O.run_config(cfg, nsteps=6, solver="cholesky")
    assert rel(th.get_T(), Tr) <= TOL
    assert th.stats()["failed_step"] == -1
