"""Pins of the oracle's single-rate SDC (the "single-rate SDC" of the
work-precision study P:730-736; reading R29: every term implicit, the interface operator
reassembled at each node): reduction to implicit Euler, the order K + 1 up to the
quadrature order M, and convergence of the sweeps to the collocation solution."""
import numpy as np
import pytest

import oracle as O
from paper_1707_03581_b200 import inputs as I


def _setup(alpha=True):
    cfg = I.make_config("small")
    if not alpha:
        cfg.alpha_iface = 0.0
    return cfg, O.Oracle.from_config(cfg)


@pytest.mark.parametrize("K", [0, 1, 3])
def test_one_node_is_implicit_euler(K):
    """M = 1: the only node is t_{n+1}; the predictor is one implicit-Euler step and every
    sweep reproduces it (I = dt F(T^k, t_{n+1}) cancels the -dt K T^k term)."""
    cfg, o = _setup()
    sc = I.Scenario(0.375, 0.375, 60.0, 500.0, 0.5, 20.0)
    T0 = I.initial_field(cfg)[0]
    Tie, _ = o.step(T0, 1.0, 0.5, 6, sc)
    Tsdc, st = o.step_sdc(T0, 1.0, 0.5, 6, sc, M=1, K=K)
    assert np.abs(Tsdc - Tie).max() <= 1e-10 * np.abs(Tie).max()
    assert (st[:, 0] == 1 + K).all()


def _orders(o, T0, sc, M, K, ref):
    errs = []
    for dt, n in ((1.0, 4), (0.5, 8), (0.25, 16)):
        T, _ = o.step_sdc(T0, 0.0, dt, n, sc, M=M, K=K)
        errs.append(np.abs(T - ref).max())
    return [np.log2(errs[i] / errs[i + 1]) for i in range(2)], errs


def test_order_k_plus_one_up_to_m():
    """Static stock, smooth friction eta(t): the predictor is first order, every sweep adds
    at least one order up to the quadrature order M = 3.  (On this stiff problem
    one sweep already reaches order 3; the bound min(M, K + 1) is what the method promises.)"""
    cfg, o = _setup()
    sc = I.Scenario(0.375, 0.0, 4.0, 2000.0, 0.8, 3.0)
    T0 = I.initial_field(cfg)[0]
    ref, _ = o.step_sdc(T0, 0.0, 4.0 / 128, 128, sc, M=3, K=4)
    for K in (0, 1, 2):
        orders, errs = _orders(o, T0, sc, 3, K, ref)
        lo = min(3, K + 1)
        assert lo - 0.2 < orders[-1] < 3.3, (K, orders, errs)
        if K == 0:
            assert abs(orders[-1] - 1) < 0.2


def test_sweeps_converge_to_collocation():
    """The SDC residual r^k falls with every sweep."""
    cfg, o = _setup()
    sc = I.Scenario(0.375, 0.05, 8.0, 800.0, 0.5, 3.0)
    T0 = I.initial_field(cfg)[0]
    res = []
    for K in (1, 2, 3, 8):
        _, st = o.step_sdc(T0, 0.0, 0.5, 1, sc, M=3, K=K)
        res.append(st[0, 2])
    assert res[1] < 0.1 * res[0] and res[2] < 0.1 * res[1], res   # until the CG-tolerance floor
    assert res[-1] < 1e-9 * np.abs(o.volume()[4] * T0).max()


def test_uniform_state_is_fixed_point():
    """No friction, all Robin temperatures equal to T0: the uniform state stays (every F = 0)."""
    cfg = I.make_config("small")
    cfg.robin = [I.Robin(r.part, r.tag, r.alpha, cfg.T0) for r in cfg.robin]
    o = O.Oracle.from_config(cfg)
    sc = I.Scenario(0.375, 0.375, 60.0, 0.0)
    T, _ = o.step_sdc(np.full(o.n, cfg.T0), 0.0, 2.0, 3, sc, M=3, K=2)
    assert np.abs(T - cfg.T0).max() < 1e-10
