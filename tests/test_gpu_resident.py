"""GPU tests of the latency path for paper-scale problems (16,626 DoF; the look-ahead
factor P:189-194): the resident-operator solve (csrc/cg_resident.cu: operator and vectors in
shared memory, one grid barrier per CG iteration) and the ahead mode (the interfaces of the next
16 step times assembled in one launch set, csrc/thermo.cu).  Both are the default where the
operator fits; every other GPU suite therefore already runs through them on the small
configurations -- here: that they are selected, parity against the oracle and against the
streaming kernel, bitwise reproducibility, and the ahead mode's slot bookkeeping (batches,
split calls, time jumps, step-size changes, operator rebuilds).
"""
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
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"


def _thermo(cfg, **kw):
    from paper_1707_03581_b200.thermo import Thermo
    return Thermo.from_config(cfg, **kw)


def rel(a, b):
    return float(np.abs(a - b).max() / np.abs(b).max())


@pytest.mark.parametrize("name,jitter", [("cfg0", None), ("small", 0.1), ("medium", 0.1), ("paper", 0.1)])
def test_resident_solve_selected_parity_and_reproducible(monkeypatch, name, jitter):
    """Default path on small problems = the resident kernel: whole field vs the oracle, vs the
    streaming grid kernel (same iteration counts +-1), and bitwise equal from run to run."""
    cfg = I.make_config(name, jitter=jitter)
    T0 = I.initial_field(cfg)[0]
    n = 12

    def run():
        th = _thermo(cfg)
        th.set_T(T0)
        th.step(0.0, cfg.dt, n)
        return th, th.get_T(), th.step_iters()[:, 0].copy()

    th, Tr1, it1 = run()
    st = th.stats()
    assert st["latency_path"] == 2 and st["failed_step"] == -1, st
    _, Tr2, it2 = run()
    assert np.array_equal(Tr1, Tr2) and np.array_equal(it1, it2)
    monkeypatch.setenv("THERMO_CG_RESIDENT", "0")
    ths, Ts, its = run()
    assert ths.stats()["latency_path"] != 2
    assert rel(Tr1, Ts) < 1e-12
    assert np.abs(it1 - its).max() <= 1
    o = O.Oracle.from_config(cfg)
    To, _ = o.step(T0, 0.0, cfg.dt, n, cfg.scenarios[0])
    assert rel(Tr1, To) <= TOL


def test_resident_not_selected_beyond_its_size_limit():
    """85,694 DoF (580 rows per CTA): the streaming kernel stays the default."""
    th = _thermo(I.make_config("cfg1"))
    assert th.stats()["latency_path"] == 0


def test_resident_forced_on_cfg1_matches_streaming_kernel(monkeypatch):
    """THERMO_CG_RESIDENT=1 on cfg 1 (operator = 182 KB of shared memory per CTA, blocks balanced by
    entries so that the rail-top interface rows spread over many CTAs): same fields."""
    cfg = I.make_config("cfg1")
    a = _thermo(cfg)
    a.step(0.0, cfg.dt, 6)
    monkeypatch.setenv("THERMO_CG_RESIDENT", "1")
    b = _thermo(cfg)
    assert b.stats()["latency_path"] == 2
    b.step(0.0, cfg.dt, 6)
    assert rel(b.get_T(), a.get_T()) < 1e-12
    assert np.abs(a.step_iters() - b.step_iters()).max() <= 1


@pytest.mark.parametrize("name", ["cfg0", "small"])
def test_ahead_mode_batches_split_calls_and_jumps(monkeypatch, name):
    """Ahead mode: 40 steps in one call (three batches of 16 slots) = 40 one-step calls (the slots
    left over by a call are the next call's) = the same run with the interface assembled step by
    step (THERMO_AHEAD=0), all bitwise; a jump in time, another step size and a stationary solve
    in between discard the assembled slots -- checked against the oracle."""
    cfg = I.make_config(name, jitter=0.1 if name != "cfg0" else None)
    n = 40
    a = _thermo(cfg)
    a.step(0.0, cfg.dt, n)
    b = _thermo(cfg)
    for k in range(n):
        b.step(k * cfg.dt, cfg.dt, 1)
    c = _thermo(cfg)
    c.step(0.0, cfg.dt, 7)
    c.step(7 * cfg.dt, cfg.dt, 20)
    c.step(27 * cfg.dt, cfg.dt, 13)
    monkeypatch.setenv("THERMO_AHEAD", "0")
    d = _thermo(cfg)
    d.step(0.0, cfg.dt, n)
    monkeypatch.delenv("THERMO_AHEAD")
    Ta = a.get_T()
    assert np.array_equal(Ta, b.get_T()) and np.array_equal(Ta, c.get_T()) and np.array_equal(Ta, d.get_T())
    assert np.array_equal(a.step_iters(), d.step_iters())
    e = _thermo(cfg)
    e.step(0.0, cfg.dt, 3)
    e.step(7.0 * cfg.dt, cfg.dt, 2)          # jump in time: the slots for t = 4 dt ... are not this call's
    e.step(9.0 * cfg.dt, 0.5 * cfg.dt, 2)    # other dt: operator rebuild, slots stale
    e.stationary(0.0, with_interface=True)
    e.step(0.0, cfg.dt, 2)
    o = O.Oracle.from_config(cfg)
    Tx, _ = o.step(np.full(o.n, cfg.T0), 0.0, cfg.dt, 3, cfg.scenarios[0])
    Tx, _ = o.step(Tx, 7.0 * cfg.dt, cfg.dt, 2, cfg.scenarios[0])
    Tx, _ = o.step(Tx, 9.0 * cfg.dt, 0.5 * cfg.dt, 2, cfg.scenarios[0])
    Tx, _ = o.stationary(Tx, 0.0, cfg.scenarios[0], with_interface=True)
    Tx, _ = o.step(Tx, 0.0, cfg.dt, 2, cfg.scenarios[0])
    assert rel(e.get_T(), Tx) <= TOL


def test_ahead_mode_slot_times_are_the_callers_expressions(monkeypatch):
    """A slot is used only if its step time equals the step's bitwise.  With dt = 0.3 (not a power
    of two) the time of step k of one call, t + (k + 1) dt, and of one-step call k, (t + k dt) + dt,
    differ in the last bits for some k: each call pattern must give exactly what it gives with the
    interface assembled step by step."""
    cfg = I.make_config("cfg0")
    dt = 0.3
    out = {}
    for ahead in ("16", "0"):
        monkeypatch.setenv("THERMO_AHEAD", ahead)
        a = _thermo(cfg)
        a.step(0.0, dt, 25)
        b = _thermo(cfg)
        for k in range(25):
            b.step(k * dt, dt, 1)
        out[ahead] = (a.get_T(), b.get_T())
    assert np.array_equal(out["16"][0], out["0"][0])
    assert np.array_equal(out["16"][1], out["0"][1])


def test_ahead_mode_operator_rebuild_invalidates_slots(monkeypatch):
    """New Robin data between two calls rebuilds the volume operator and its Jacobi diagonal: the
    interface rows' diagonals assembled ahead are stale and must be assembled again."""
    cfg = I.make_config("small", jitter=0.1)
    out = {}
    for ahead in ("16", "0"):
        monkeypatch.setenv("THERMO_AHEAD", ahead)
        th = _thermo(cfg)
        th.step(0.0, cfg.dt, 3)
        th.set_bc(0, 1, 25.0, 21.0)
        th.step(3 * cfg.dt, cfg.dt, 3)
        out[ahead] = th.get_T()
    assert np.array_equal(out["16"], out["0"])


def test_ahead_mode_with_streaming_kernel_cfg2(monkeypatch):
    """Sizes without the overlap mode (N > 2^18) run the ahead mode with the streaming grid kernel
    (the interface rows' Jacobi diagonal comes with the step's slot): bitwise the step-by-step
    assembly, at a fraction of its interface time per step."""
    cfg = I.make_config("cfg2")
    out = {}
    for ahead in ("16", "0"):
        monkeypatch.setenv("THERMO_AHEAD", ahead)
        th = _thermo(cfg)
        th.set_timing(True)
        th.step(0.0, cfg.dt, 2)
        th.step(2 * cfg.dt, cfg.dt, 18)     # 2 slots of the first batch left over + a second batch
        st = th.stats()
        assert st["latency_path"] == 0 and st["failed_step"] == -1
        out[ahead] = (th.get_T(), st["ms_iface"] / 18, th.step_iters().copy())
    assert np.array_equal(out["16"][0], out["0"][0])
    assert np.array_equal(out["16"][2], out["0"][2])
    assert out["16"][1] < 0.7 * out["0"][1], (out["16"][1], out["0"][1])
