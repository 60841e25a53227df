"""GPU parity: the CUDA path through the C ABI against the CPU oracle on the same seeded
inputs (max-norm relative error <= 1e-9 after the run, BASELINE.json north star), plus the
invariants of the method evaluated on the GPU output.

All calls go through paper_1707_03581_b200.thermo (ctypes -> libthermo.so).
"""
import math

import numpy as np
import pytest

import oracle as O
from paper_1707_03581_b200 import inputs as I

pytestmark = pytest.mark.gpu

TOL = 1e-9   # north star: max-norm relative error after the full run


@pytest.fixture(scope="module", autouse=True)
def _built():
    import __graft_entry__ as g
    g.build()
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"


def _thermo(cfg, **kw):
    from paper_1707_03581_b200.thermo import Thermo
    return Thermo.from_config(cfg, **kw)


def rel(a, b):
    return float(np.abs(a - b).max() / np.abs(b).max())


def test_cfg0_full_run_vs_dense_cholesky():
    """BASELINE config 0, 100 steps: GPU CG vs oracle dense Cholesky."""
    cfg = I.make_config("cfg0")
    th = _thermo(cfg)
    th.step(0.0, cfg.dt, cfg.nsteps)
    Tg = th.get_T()
    Tr, st = O.run_config(cfg, solver="cholesky")
    assert rel(Tg, Tr) <= TOL
    s = th.stats()
    assert s["steps_done"] == cfg.nsteps and s["failed_step"] == -1
    assert abs(s["iface_area"] - 0.05) < 1e-14


@pytest.mark.parametrize("name,jitter", [("small", 0.0), ("small", 0.1), ("medium", 0.1)])
def test_parity_vs_oracle_cg(name, jitter):
    """Several slices + a ragged tail, jittered non-matching meshes, a non-uniform seeded
    start field, time-varying friction; full configured run length."""
    cfg = I.make_config(name, jitter=jitter)
    T0 = I.initial_field(cfg)[0]
    th = _thermo(cfg)
    th.set_guess(0)   # x0 = T^n as in the oracle (reading R17), so iteration counts compare
    th.set_T(T0)
    th.step(0.0, cfg.dt, cfg.nsteps)
    Tg = th.get_T()
    Tr, st = O.run_config(cfg, T_init=T0)
    assert rel(Tg, Tr) <= TOL
    it = th.step_iters()[:, 0]
    # same stopping rule and start on both sides: iteration counts agree to +-1
    assert np.abs(it - st[:, 0]).max() <= 1


@pytest.mark.parametrize("order", [1, 2])
def test_extrapolated_guess_parity_and_fewer_iterations(order):
    """thermo_set_guess: CG from the extrapolated state reaches the same IE solution (same
    stopping rule) in fewer iterations; the history restarts after thermo_set_T and after a
    dt change (no stale state enters the guess)."""
    cfg = I.make_config("medium", jitter=0.1)
    n1 = 24
    runs = {}
    for g in (0, order):
        th = _thermo(cfg)
        th.set_guess(g)
        th.step(0.0, cfg.dt, n1 // 2)
        th.step(n1 // 2 * cfg.dt, cfg.dt, n1 - n1 // 2)   # history carried across calls
        runs[g] = (th.get_T(), th.step_iters()[:, 0].copy(), th)
    Tr, st = O.run_config(cfg, nsteps=n1)
    assert rel(runs[0][0], Tr) <= TOL
    assert rel(runs[order][0], Tr) <= TOL
    # the second call's steps all have history: fewer iterations in total
    assert runs[order][1].sum() < runs[0][1].sum(), (runs[order][1], runs[0][1])
    # the oracle with the same start (or_set_guess, history across its calls as well) takes
    # the same iterations and lands on the same field to rounding
    o = O.Oracle.from_config(cfg, order)
    Ta, _ = o.step(np.full(o.n, cfg.T0), 0.0, cfg.dt, n1 // 2, cfg.scenarios[0])
    Tg, sg = o.step(Ta, n1 // 2 * cfg.dt, cfg.dt, n1 - n1 // 2, cfg.scenarios[0])
    assert np.abs(runs[order][1] - sg[:, 0]).max() <= 1
    assert rel(runs[order][0], Tg) <= 1e-12
    th = runs[order][2]
    # restart: new state, then a different dt -- both must match the oracle from that state
    T1 = I.initial_field(cfg, seed=5)[0]
    th.set_T(T1)
    t1 = 3 * 0.5 * cfg.dt
    th.step(0.0, 0.5 * cfg.dt, 3)
    th.step(t1, 0.25 * cfg.dt, 3)
    o = O.Oracle.from_config(cfg)
    Ta, _ = o.step(T1, 0.0, 0.5 * cfg.dt, 3, cfg.scenarios[0])
    Tb, _ = o.step(Ta, t1, 0.25 * cfg.dt, 3, cfg.scenarios[0])
    assert rel(th.get_T(), Tb) <= TOL


def test_guess_argument_errors():
    from paper_1707_03581_b200.thermo import ThermoError
    cfg = I.make_config("cfg0")
    th = _thermo(cfg)
    for bad in (-1, 3):
        with pytest.raises(ThermoError):
            th.set_guess(bad)


def test_parts_and_device_copy():
    import torch
    cfg = I.make_config("small")
    th = _thermo(cfg)
    th.step(0.0, cfg.dt, 3)
    full = th.get_T()
    assert np.array_equal(th.get_T(part=0), full[:cfg.fixed.n_nodes])
    assert np.array_equal(th.get_T(part=1), full[cfg.fixed.n_nodes:])
    out = torch.empty(cfg.n_dof, dtype=torch.float64, device="cuda")
    th.get_T(out=out)
    torch.cuda.synchronize()
    assert np.array_equal(out.cpu().numpy(), full)


def test_deterministic_and_step_splitting():
    """Deterministic reductions: two runs are bitwise equal, and 10 steps in one call equal
    5 + 5 steps in two calls."""
    cfg = I.make_config("small", jitter=0.1)
    a = _thermo(cfg)
    a.step(0.0, cfg.dt, 10)
    b = _thermo(cfg)
    b.step(0.0, cfg.dt, 5)
    b.step(5 * cfg.dt, cfg.dt, 5)
    c = _thermo(cfg)
    c.step(0.0, cfg.dt, 10)
    assert np.array_equal(a.get_T(), c.get_T())
    assert np.array_equal(a.get_T(), b.get_T())


def test_uniform_state_fixed_point_gpu():
    cfg = I.make_config("small", jitter=0.1)
    cfg.robin = [I.Robin(0, 1, 10.0, 24.0), I.Robin(1, 1, 10.0, 24.0), I.Robin(0, 3, 50.0, 24.0),
                 I.Robin(1, 2, 200.0, 24.0)]
    cfg.scenarios = [I.Scenario(0.375, 0.375, 20.0, 0.0)]
    th = _thermo(cfg)
    th.step(0.0, 1.0, 10)
    assert np.abs(th.get_T() - 24.0).max() < 1e-9


def test_energy_balance_gpu():
    """Robin off: sum M_L dT = dt eta(t_{n+1}) |Gamma_R| per step (north star invariant)."""
    cfg = I.make_config("medium", jitter=0.1)
    cfg.robin = []
    ML = O.Oracle.from_config(cfg).volume()[4]
    sc = cfg.scenarios[0]
    th = _thermo(cfg)
    T = th.get_T()
    for n in range(4):
        th.step(n * cfg.dt, cfg.dt, 1)
        T1 = th.get_T()
        eta = sc.eta0 * (1 + sc.eta_amp * math.sin(2 * math.pi * (n + 1) * cfg.dt / sc.eta_period))
        dE = float(ML @ (T1 - T))
        assert abs(dE - cfg.dt * eta * 0.05) < 1e-7 * cfg.dt * eta * 0.05
        T = T1


def test_noconv_reports_and_keeps_state():
    from paper_1707_03581_b200.thermo import ThermoError, THERMO_ENOCONV
    cfg = I.make_config("small")
    th = _thermo(cfg)
    th.step(0.0, cfg.dt, 2)
    T2 = th.get_T()
    th.set_solver(1e-12, 1)
    with pytest.raises(ThermoError) as e:
        th.step(2 * cfg.dt, cfg.dt, 3)
    assert e.value.code == THERMO_ENOCONV
    s = th.stats()
    assert s["failed_step"] == 0 and s["failed_relres"] > 1e-12
    assert np.array_equal(th.get_T(), T2)



@pytest.mark.parametrize("pair", [(2, 8), (4, 9), (7, 10)])
@pytest.mark.parametrize("name", ["small", "medium"])
def test_fused_variant_bitwise_equals_unfused(monkeypatch, name, pair):
    """The one-barrier-per-iteration kernel (update of iteration k folded into the sweep of
    k + 1, p formed from the z, q', p windows) computes the same numbers in the same order as
    the two-phase kernel of the same chunk size: bitwise equal fields and iteration counts."""
    cfg = I.make_config(name, jitter=0.1)
    T0 = I.initial_field(cfg)[0]
    out = []
    for v in pair:
        monkeypatch.setenv("THERMO_CG_VARIANT", str(v))
        th = _thermo(cfg)
        th.set_T(T0)
        th.step(0.0, cfg.dt, cfg.nsteps)
        out.append((th.get_T(), th.step_iters()[:, 0].copy()))
    assert np.array_equal(out[0][1], out[1][1])
    assert np.array_equal(out[0][0], out[1][0])


@pytest.mark.parametrize("name", ["cfg0", "medium"])
def test_interface_overlap_mode(monkeypatch, name):
    """Overlap mode (interface kernels of step n+1 on a side stream into the second buffer set
    while step n solves on the remaining SMs): same result as the serial schedule to rounding
    (only the CTA count of the reductions differs), bitwise reproducible, split calls equal one
    call, and both match the oracle."""
    cfg = I.make_config(name, jitter=0.1 if name != "cfg0" else None)
    # (the resident solve with its ahead mode is the default at these sizes and replaces the
    # overlap mode there; the overlap mode serves the L2-resident sizes above it, e.g. cfg 1)
    monkeypatch.setenv("THERMO_CG_RESIDENT", "0")
    runs = {}
    for mode in ("0", "1"):
        monkeypatch.setenv("THERMO_OVERLAP", mode)
        a = _thermo(cfg)
        a.step(0.0, cfg.dt, 12)
        b = _thermo(cfg)
        b.step(0.0, cfg.dt, 5)
        b.step(5 * cfg.dt, cfg.dt, 7)
        assert np.array_equal(a.get_T(), b.get_T())
        runs[mode] = a.get_T()
        assert a.stats()["failed_step"] == -1
    assert rel(runs["1"], runs["0"]) < 1e-12
    Tr, _ = O.run_config(cfg, nsteps=12)
    assert rel(runs["1"], Tr) <= TOL
    # one step per call (the speculated assembly of the next step is used) = one call; a call
    # that does not continue the time line (or changes dt) discards the speculation
    monkeypatch.setenv("THERMO_OVERLAP", "1")
    c1 = _thermo(cfg)
    for n in range(12):
        c1.step(n * cfg.dt, cfg.dt, 1)
    assert np.array_equal(c1.get_T(), runs["1"])
    d = _thermo(cfg)
    d.step(0.0, cfg.dt, 3)
    d.step(7.0 * cfg.dt, cfg.dt, 2)          # jump in time: speculation for t = 3 dt unused
    d.step(9.0 * cfg.dt, 0.5 * cfg.dt, 2)    # other dt
    d.stationary(0.0, with_interface=True)   # joins the side stream, reuses the first buffer set
    d.step(0.0, cfg.dt, 2)
    o = O.Oracle.from_config(cfg)
    Ta, _ = o.step(np.full(o.n, cfg.T0), 0.0, cfg.dt, 3, cfg.scenarios[0])
    Tb, _ = o.step(Ta, 7.0 * cfg.dt, cfg.dt, 2, cfg.scenarios[0])
    Tc, _ = o.step(Tb, 9.0 * cfg.dt, 0.5 * cfg.dt, 2, cfg.scenarios[0])
    Ts, _ = o.stationary(Tc, 0.0, cfg.scenarios[0], with_interface=True)
    Td, _ = o.step(Ts, 0.0, cfg.dt, 2, cfg.scenarios[0])
    assert rel(d.get_T(), Td) <= TOL


def test_speculated_interface_equals_fresh_assembly(monkeypatch):
    """One step per call in overlap mode uses the interface the previous call assembled
    speculatively for t + nsteps dt.  Its step time must be the expression the next call
    evaluates (ts + 1 dt), so the speculation is bitwise the fresh assembly -- checked with a
    step size that is not a power of two (dt = 0.3: t + 2 dt != (t + dt) + dt in the last bits)."""
    cfg = I.make_config("cfg0")
    dt = 0.3
    monkeypatch.setenv("THERMO_CG_RESIDENT", "0")   # the overlap mode's path (see above)
    out = []
    for spec in ("1", "0"):
        monkeypatch.setenv("THERMO_OVERLAP", "1")
        monkeypatch.setenv("THERMO_SPEC", spec)
        th = _thermo(cfg)
        t = 0.0
        for n in range(40):
            th.step(t, dt, 1)
            t = t + dt
        out.append(th.get_T())
    assert np.array_equal(out[0], out[1])


@pytest.mark.parametrize("stages", [3, 5])
@pytest.mark.parametrize("variant", [1, 3, 5])
def test_two_consumer_groups_any_stage_cap(monkeypatch, variant, stages):
    """Kernels with two consumer groups take alternate ring slots; a stage count that is not a
    multiple of the group count once let a group pass a stage's mbarrier one phase early (stale
    stage, launch failure on cfg 3).  The ring is now rounded to a multiple of the groups."""
    cfg = I.make_config("medium", jitter=0.1)
    monkeypatch.setenv("THERMO_CG_VARIANT", str(variant))
    monkeypatch.setenv("THERMO_CG_STAGES", str(stages))
    a = _thermo(cfg)
    a.step(0.0, cfg.dt, 8)
    Tr, _ = O.run_config(cfg, nsteps=8)
    assert rel(a.get_T(), Tr) <= TOL


@pytest.mark.parametrize("variant", [0, 1, 2, 3, 4, 8, 9])
def test_cg_kernel_variants_agree(monkeypatch, variant):
    """Every sweep kind (register streaming, TMA matrix ring, TMA ring + shared-memory vector
    windows with 16-bit local columns) forms identical row sums; only the CTA-level order of
    the dot-product partials differs, so results agree to rounding and all match the oracle."""
    cfg = I.make_config("medium", jitter=0.1)
    monkeypatch.setenv("THERMO_CG_VARIANT", str(variant))
    a = _thermo(cfg)
    a.step(0.0, cfg.dt, cfg.nsteps)
    monkeypatch.setenv("THERMO_CG_VARIANT", "0")
    b = _thermo(cfg)
    b.step(0.0, cfg.dt, cfg.nsteps)
    assert rel(a.get_T(), b.get_T()) < 1e-12
    Tr, _ = O.run_config(cfg)
    assert rel(a.get_T(), Tr) <= TOL


@pytest.mark.slow
@pytest.mark.parametrize("name,nsteps", [("cfg2", 4), ("cfg3", 2)])
def test_stand_scale_short_horizon(name, nsteps):
    """BASELINE configs 2 and 3 at full size (1.28 M / 10.0 M DoF, jittered L-shape, the
    launch configuration bench.py times): a short horizon from a seeded non-uniform field,
    every DoF against the oracle (its full 3600 / 200-step runs are out of a test's reach)."""
    cfg = I.make_config(name)
    T0 = I.initial_field(cfg)[0]
    th = _thermo(cfg)
    th.set_T(T0)
    t0 = 7.0
    th.step(t0, cfg.dt, nsteps)
    Tg = th.get_T()
    o = O.Oracle.from_config(cfg)
    Tr, st = o.step(T0, t0, cfg.dt, nsteps, cfg.scenarios[0])
    assert rel(Tg, Tr) <= TOL
    assert abs(th.stats()["iface_area"] - 0.08) < 1e-12


@pytest.mark.slow
def test_cfg2_full_run_invariants():
    """BASELINE config 2 for its full 3600 steps on the GPU: every step converged, the
    interface area stays 0.08 m^2, and sampled rows of the last step satisfy the oracle's
    own implicit-Euler equations (row residuals assembled by the oracle, one by one)."""
    cfg = I.make_config("cfg2")
    th = _thermo(cfg)
    th.step(0.0, cfg.dt, cfg.nsteps - 1)
    Tprev = th.get_T()
    th.step((cfg.nsteps - 1) * cfg.dt, cfg.dt, 1)
    Tlast = th.get_T()
    s = th.stats()
    assert s["steps_done"] == cfg.nsteps and s["last_relres"] <= 1e-12
    assert abs(s["iface_area"] - 0.08) < 1e-12
    assert np.isfinite(Tlast).all() and 17.0 < Tlast.min() and Tlast.max() < 40.0
    o = O.Oracle.from_config(cfg)
    tp = cfg.nsteps * cfg.dt
    sv, eta = I.scenario_scalars(cfg.scenarios[0], tp)
    rng = np.random.default_rng(3)
    rows = np.concatenate([rng.integers(0, o.n, 2000), np.arange(o.n - 50, o.n)])
    res, bnorm = o.residual_rows(cfg.dt, (sv, 0.0, 0.0), eta, Tprev, Tlast, rows)
    assert np.abs(res).max() <= 1e-10 * bnorm


@pytest.mark.parametrize("stock_cells", [(5, 3, 4), (5, 3, 3)])
def test_one_row_tail_slice(stock_cells):
    """N = 225 leaves a last slice with a single row (31 padding lanes) -- the regression case
    of the window kernel's own-row index; N = 201 leaves 9 rows.  Parity vs dense Cholesky."""
    from paper_1707_03581_b200.thermo import Thermo
    f, m = I.two_slab_pair(stock_cells=stock_cells, jitter=0.1)
    robin = [I.Robin(0, I.TAG_FLOOR, 50.0, 24.0), I.Robin(1, I.TAG_COOL, 200.0, 18.0)]
    sc = I.Scenario(0.0, 0.0, 1.0, 500.0)
    th = Thermo(f, m, 50.0, 3.6e6, 1000.0, [sc], 24.0, (4, 4), robin)
    th.step(0.0, 5.0, 8)
    o = O.Oracle(f, m, 50.0, 3.6e6, 1000.0, robin=robin)
    Tr, _ = o.step(np.full(o.n, 24.0), 0.0, 5.0, 8, sc, solver="cholesky")
    assert rel(th.get_T(), Tr) <= TOL


@pytest.mark.parametrize("name,jitter", [("cfg0", None), ("small", 0.1)])
def test_interface_rows_vs_oracle_matrices(name, jitter):
    """Per-kernel check of the interface assembly: the GPU's interface rows
    (-dt K_G(t) entries) and friction sources (eta/2 int phi) at several stock
    positions against the oracle's independently clipped and integrated matrices, entry by entry."""
    cfg = I.make_config(name, jitter=jitter)
    th = _thermo(cfg)
    o = O.Oracle.from_config(cfg)
    sc = cfg.scenarios[0]
    dt = 0.7
    for t in (0.0, 3.3, 11.0, 17.25, 41.0):
        rows, cnt, col, val, b = th.get_interface(t, dt)
        s, eta = I.scenario_scalars(sc, t)
        rp, icol, ival, bG, area = o.interface(np.array(sc.dir) * s, eta)
        scale = max(np.abs(ival).max() * dt, 1e-300)
        worst = 0.0
        for k, r in enumerate(rows):
            g = {}
            for q in range(cnt[k]):
                g[int(col[k, q])] = g.get(int(col[k, q]), 0.0) + val[k, q]
            ref = {int(c): -dt * v for c, v in zip(icol[rp[r]:rp[r + 1]], ival[rp[r]:rp[r + 1]])}
            for c in set(g) | set(ref):
                worst = max(worst, abs(g.get(c, 0.0) - ref.get(c, 0.0)))
            assert abs(b[k] - bG[r]) <= 1e-13 * max(abs(bG).max(), 1e-300), (t, k)
        assert worst <= 1e-13 * scale, (t, worst / scale)
        # rows outside the interface carry no interface terms in the oracle either
        others = np.setdiff1d(np.arange(o.n), rows)
        assert np.all(rp[others + 1] - rp[others] == 0) or np.abs(ival).max() == 0


def test_interface_rows_batched_scenarios():
    """The same per-kernel check for a batched context: the rows of scenarios 1 and 2 (their own
    stock positions and friction laws, blockIdx.y = scenario) against the oracle."""
    from paper_1707_03581_b200.thermo import Thermo
    cfg = I.make_config("small", jitter=0.1)
    scen = [I.Scenario(0.375, 0.375, 20.0 + 7 * k, 100.0 + 150.0 * k, 0.3 * k, 9.0) for k in range(3)]
    th = Thermo.from_config(cfg, scenarios=scen)
    o = O.Oracle.from_config(cfg)
    dt, t = 0.5, 6.5
    for k in (1, 2):
        rows, cnt, col, val, b = th.get_interface(t, dt, scen=k)
        s, eta = I.scenario_scalars(scen[k], t)
        rp, icol, ival, bG, area = o.interface(np.array(scen[k].dir) * s, eta)
        scale = np.abs(ival).max() * dt
        for j, r in enumerate(rows):
            g = {}
            for q in range(cnt[j]):
                g[int(col[j, q])] = g.get(int(col[j, q]), 0.0) + val[j, q]
            ref = {int(c): -dt * v for c, v in zip(icol[rp[r]:rp[r + 1]], ival[rp[r]:rp[r + 1]])}
            for c in set(g) | set(ref):
                assert abs(g.get(c, 0.0) - ref.get(c, 0.0)) <= 1e-13 * scale, (k, j, c)
            assert abs(b[j] - bG[r]) <= 1e-13 * np.abs(bG).max(), (k, j)
