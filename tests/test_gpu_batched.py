"""Batched scenarios (BASELINE.json config 4): S scenarios with different
motion periods and friction laws advanced together through one context; every column is
checked against an independent oracle run of that scenario (max-norm relative <= 1e-9)."""
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


def _scen(k):
    return I.Scenario(0.375, 0.375, 20.0 + k, 100.0 + 15.0 * k, 0.3 * (k % 2), 7.0 + k)


@pytest.mark.parametrize("S", [2, 3, 5])
def test_batched_columns_match_oracle(S):
    from paper_1707_03581_b200.thermo import Thermo
    cfg = I.make_config("small", jitter=0.1)
    scen = [_scen(k) for k in range(S)]
    th = Thermo.from_config(cfg, scenarios=scen)
    T0 = I.initial_field(cfg)[0]
    for k in range(S):
        th.set_T(T0 + 0.1 * k, scen=k)
    th.step(0.0, cfg.dt, 20)
    o = O.Oracle.from_config(cfg)
    for k in range(S):
        Tr, st = o.step(T0 + 0.1 * k, 0.0, cfg.dt, 20, scen[k])
        assert rel(th.get_T(scen=k), Tr) <= TOL, k
    it = th.step_iters()
    assert it.shape == (20, S) and it.min() > 0


@pytest.mark.parametrize("guess", [0, 2])
def test_batched_equals_single_runs(guess):
    """Column k of a batched run equals a single-scenario run of scenario k (same row sums;
    only the dot-product reduction trees differ), with CG started from T^n or from the
    extrapolated states on both sides."""
    from paper_1707_03581_b200.thermo import Thermo
    cfg = I.make_config("medium", jitter=0.1)
    scen = [_scen(k) for k in range(4)]
    tb = Thermo.from_config(cfg, scenarios=scen)
    tb.set_guess(guess)
    tb.step(0.0, 1.0, 6)
    for k in (0, 3):
        ts = Thermo.from_config(cfg, scenarios=[scen[k]])
        ts.set_guess(guess)
        ts.step(0.0, 1.0, 6)
        # both stop at rtol 1e-12; the reduction trees differ (and so may the last iteration
        # count), so they agree to the solver tolerance, not bitwise (reading R17)
        assert rel(tb.get_T(scen=k), ts.get_T()) < 1e-11
        # same CG iterations per step (+-1): the batched dot products are those of column k
        ib = tb.step_iters().reshape(6, -1)[:, k]
        isg = ts.step_iters().reshape(6, -1)[:, 0]
        assert np.abs(ib.astype(int) - isg.astype(int)).max() <= 1, (ib, isg)


def test_cfg4_sampled_scenarios():
    """Config 4 (cfg 1 meshes, 64 scenarios, dt = 1 s): a short horizon, sampled columns
    against the oracle."""
    from paper_1707_03581_b200.thermo import Thermo
    cfg = I.make_config("cfg4")
    th = Thermo.from_config(cfg)
    n = 5
    th.step(0.0, cfg.dt, n)
    o = O.Oracle.from_config(cfg)
    for k in (0, 37, 63):
        Tr, st = o.step(np.full(o.n, cfg.T0), 0.0, cfg.dt, n, cfg.scenarios[k])
        assert rel(th.get_T(scen=k), Tr) <= TOL, k


@pytest.mark.parametrize("S", [3, 20])
def test_windowed_spmm_kernel_matches_gather_kernel(monkeypatch, S):
    """The default windowed-SpMM batched kernel (cg_spmm.cu: column groups of 16, padding
    columns for S = 20) against the gather kernel (THERMO_CGB=1, cg_batched.cu) and the oracle."""
    from paper_1707_03581_b200.thermo import Thermo
    cfg = I.make_config("medium", jitter=0.1)
    scen = [_scen(k) for k in range(S)]
    out = {}
    for mode in ("spmm", "1"):
        if mode == "1":
            monkeypatch.setenv("THERMO_CGB", mode)
        else:
            monkeypatch.delenv("THERMO_CGB", raising=False)
        th = Thermo.from_config(cfg, scenarios=scen)
        th.step(0.0, 1.0, 6)
        assert th.stats()["solve_kind"] == (3 if mode == "spmm" else -1)
        out[mode] = np.stack([th.get_T(scen=k) for k in range(S)])
    for k in range(S):
        assert rel(out["spmm"][k], out["1"][k]) < 1e-11, k
    for k in (0, S - 1):
        Tr, _ = O.Oracle.from_config(cfg).step(np.full(cfg.n_dof, cfg.T0), 0.0, 1.0, 6, scen[k])
        assert rel(out["spmm"][k], Tr) <= 1e-9


def test_spmm_kernel_reproducible_cfg4(monkeypatch):
    """Regression test for the stage reuse race of the windowed-SpMM kernel (a bulk copy
    refilling a ring stage could overtake a consumer's outstanding shared-memory loads without
    the producer's proxy fence; about one run in three then had one stale row).  configs[4],
    200 steps in calls of 5 from x0 = T^n at rtol 2e-13, three runs, each after a throw-away
    context has left its freed memory behind: bitwise equal to each other, and to the gather
    kernel within 1e-12."""
    from paper_1707_03581_b200.thermo import Thermo
    cfg = I.make_config("cfg4")

    def run(kind, n=200, block=5):
        if kind == 1:
            monkeypatch.setenv("THERMO_CGB", "1")
        else:
            monkeypatch.delenv("THERMO_CGB", raising=False)
        th = Thermo.from_config(cfg)
        th.set_guess(0)
        th.set_solver(rtol=2e-13)
        assert th.stats()["solve_kind"] == (3 if kind == 2 else -1)
        for b in range(n // block):
            th.step(b * block * cfg.dt, cfg.dt, block)
        T = np.stack([th.get_T(scen=k) for k in range(cfg.n_scen)])
        th.close()
        return T

    ref = run(1)
    outs = []
    for _ in range(3):
        junk = Thermo.from_config(cfg)
        junk.step(0.0, cfg.dt, 2)
        junk.close()
        outs.append(run(2))
    for T in outs:
        assert np.array_equal(T, outs[0])
        assert rel(T, ref) < 1e-12


def test_sdc_method_moves_context_to_gather_kernel():
    """set_method('sdc') on a batched context running the windowed-SpMM kernel moves its state
    to the gather kernel's layout: the state is unchanged, and continuing with implicit Euler
    matches a context that ran on the gather kernel throughout."""
    import os
    from paper_1707_03581_b200.thermo import Thermo
    cfg = I.make_config("medium", jitter=0.1)
    scen = [_scen(k) for k in range(20)]
    a = Thermo.from_config(cfg, scenarios=scen)
    a.set_guess(0)
    assert a.stats()["solve_kind"] == 3
    a.step(0.0, 1.0, 3)
    before = np.stack([a.get_T(scen=k) for k in range(20)])
    a.set_method("sdc", 3, 1, 1)
    assert a.stats()["solve_kind"] == -1
    after = np.stack([a.get_T(scen=k) for k in range(20)])
    assert np.array_equal(before, after)
    a.set_method("ie")
    a.step(3.0, 1.0, 3)
    os.environ["THERMO_CGB"] = "1"
    try:
        b = Thermo.from_config(cfg, scenarios=scen)
    finally:
        del os.environ["THERMO_CGB"]
    b.set_guess(0)
    b.step(0.0, 1.0, 6)
    for k in (0, 19):
        assert rel(a.get_T(scen=k), b.get_T(scen=k)) < 1e-11
