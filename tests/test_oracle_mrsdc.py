"""Pins of the oracle's multi-rate SDC: quadrature tables, the reduction to
IMEX Euler, and the measured order min(M, P, k+1) on smooth problems.

Reading R24: P:510 prints s^_{m,p} = sum_q s_{m,p,q}; the consistency
I_{m-1}^m = sum_p I_{m,p-1}^p requires the sum over the sub-intervals p, i.e.
s^_{m,q} = sum_p s_{m,p,q} (summing over q instead gives the sub-interval length).
"""
import os

import numpy as np
import pytest

import oracle as O
from paper_1707_03581_b200 import inputs as I


def test_weights_closed_forms():
    # M = 1: the single node integrates over the whole step
    tau, taue, s, sh, st, se = O.mrsdc_weights(1, 1, 0.0, 2.0)
    np.testing.assert_allclose(tau, [2.0])
    np.testing.assert_allclose(s, [[2.0]])
    # M = 2 on [0, 1] (nodes .5, 1): the golden fixture
    tau, taue, s, sh, st, se = O.mrsdc_weights(2, 1, 0.0, 1.0)
    np.testing.assert_allclose(tau, [0.5, 1.0])
    gold = {"q": [], "s": []}
    for line in open(os.path.join(os.path.dirname(__file__), "golden", "sdc_weights_M2.txt")):
        if line.strip() and not line.startswith("#"):
            k, *v = line.split()
            gold[k].append([float(x) for x in v])
    np.testing.assert_allclose(s, gold["s"], atol=1e-15)
    np.testing.assert_allclose(np.cumsum(s, axis=0), gold["q"], atol=1e-15)   # q_m = sum_{m' <= m} s_m


@pytest.mark.parametrize("M,P", [(3, 2), (5, 8), (4, 3), (2, 5)])
def test_weights_consistency_and_exactness(M, P):
    t0, dt = 1.5, 0.8
    tau, taue, s, sh, st, se = O.mrsdc_weights(M, P, t0, dt)
    # nodes: equidistant, no-left, tau_M = t_{n+1}, tau_{m,P} = tau_m
    np.testing.assert_allclose(tau, t0 + dt * np.arange(1, M + 1) / M)
    np.testing.assert_allclose(taue[:, -1], tau)
    # consistency (reading R24)
    np.testing.assert_allclose(st.sum(axis=1), s, atol=1e-14)
    np.testing.assert_allclose(se.sum(axis=1), sh, atol=1e-14)
    # exactness on polynomials: standard weights to degree M-1, embedded to degree P-1
    edges = np.concatenate([[t0], tau])
    for d in range(M):
        exact = (edges[1:] ** (d + 1) - edges[:-1] ** (d + 1)) / (d + 1)
        np.testing.assert_allclose(s @ tau ** d, exact, rtol=1e-12, atol=1e-14)
    for m in range(M):
        emb = taue[m]
        sub = np.concatenate([[edges[m]], emb])
        for d in range(P):
            np.testing.assert_allclose(sh[m] @ emb ** d, (edges[m + 1] ** (d + 1) - edges[m] ** (d + 1)) / (d + 1),
                                       rtol=1e-12, atol=1e-14)
            np.testing.assert_allclose(se[m] @ emb ** d, (sub[1:] ** (d + 1) - sub[:-1] ** (d + 1)) / (d + 1),
                                       rtol=1e-11, atol=1e-14)
        for d in range(M):
            np.testing.assert_allclose(st[m] @ tau ** d, (sub[1:] ** (d + 1) - sub[:-1] ** (d + 1)) / (d + 1),
                                       rtol=1e-11, atol=1e-14)


def test_mrsdc_11_predictor_is_imex_euler():
    """M = P = 1, no sweep: M T1 = M T* + dt f^E(T0, t_n) with (M - dt (A+B)) T* = M T0 + dt g
    (Algorithm 1), computed here with a dense library solve."""
    cfg = I.make_config("cfg0")
    o = O.Oracle.from_config(cfg)
    sc = I.Scenario(0.375, 0.375, 60.0, 500.0, 0.5, 7.0)
    T0 = I.initial_field(cfg)[0]
    t, dt = 2.0, 0.7
    T1, st = o.step_mrsdc(T0, t, dt, 1, sc, 1, 1, 0)
    rp, col, A, B, ML, benv = o.volume()
    n = o.n
    K = np.zeros((n, n))
    for i in range(n):
        K[i, col[rp[i]:rp[i + 1]]] += A[rp[i]:rp[i + 1]] + B[rp[i]:rp[i + 1]]
    Ts = np.linalg.solve(np.diag(ML) - dt * K, ML * T0 + dt * benv)
    s0, eta0 = I.scenario_scalars(sc, t)   # f^E at the left end t_n (explicit)
    irp, icol, ival, bG, area = o.interface((s0, 0, 0), eta0)
    KG = np.zeros((n, n))
    for i in range(n):
        KG[i, icol[irp[i]:irp[i + 1]]] += ival[irp[i]:irp[i + 1]]
    expect = Ts + dt * (KG @ T0 + bG) / ML
    assert np.abs(T1 - expect).max() / np.abs(expect).max() < 1e-12


def _order(o, T0, sc, M, P, K, ref):
    errs = []
    for dt, n in ((0.5, 4), (0.25, 8), (0.125, 16)):
        T, _ = o.step_mrsdc(T0, 0.0, dt, n, sc, M, P, K)
        errs.append(np.abs(T - ref).max())
    return [np.log2(errs[i] / errs[i + 1]) for i in range(2)]


def test_order_without_coupling_is_sdc_order():
    """f^E = 0 (alpha = eta = 0): MRSDC reduces to SDC of the implicit part, order min(M, k+1)."""
    cfg = I.make_config("small")
    cfg.alpha_iface = 0.0
    o = O.Oracle.from_config(cfg)
    sc = I.Scenario(0.375, 0.0, 4.0, 0.0)
    T0 = I.initial_field(cfg)[0]
    ref, _ = o.step_mrsdc(T0, 0.0, 2.0 / 64, 64, sc, 3, 2, 6)
    for K, expect in ((0, 1), (1, 2), (2, 3)):
        orders = _order(o, T0, sc, 3, 2, K, ref)
        assert abs(orders[-1] - expect) < 0.15, (K, orders)


def test_order_with_coupling_min_m_p_k():
    """Coupled problem with smooth f^E (static stock, eta(t) smooth): order min(M, P, k+1)
    (P:580): (3,2): 1, 2, 2 for k = 0, 1, 2; (3,8): at least k + 1."""
    cfg = I.make_config("small")
    o = O.Oracle.from_config(cfg)
    sc = I.Scenario(0.375, 0.0, 4.0, 2000.0, 0.8, 1.5)
    T0 = I.initial_field(cfg)[0]
    ref, _ = o.step_mrsdc(T0, 0.0, 2.0 / 128, 128, sc, 3, 2, 6)
    for K, expect in ((0, 1), (1, 2), (2, 2)):
        orders = _order(o, T0, sc, 3, 2, K, ref)
        assert abs(orders[-1] - expect) < 0.15, (K, orders)
    for K in (1, 2):
        orders = _order(o, T0, sc, 3, 8, K, ref)
        assert orders[-1] > K + 1 - 0.2, (K, orders)


def test_residual_decays_to_collocation():
    """Property (i): the SDC residual decreases with every sweep toward the
    collocation solution."""
    cfg = I.make_config("small")
    o = O.Oracle.from_config(cfg)
    sc = I.Scenario(0.375, 0.05, 8.0, 800.0, 0.5, 3.0)
    T0 = I.initial_field(cfg)[0]
    res = []
    for K in (1, 2, 3, 5, 8):
        _, st = o.step_mrsdc(T0, 0.0, 0.5, 1, sc, 3, 2, K)
        res.append(st[0, 2])
    assert all(res[i + 1] < res[i] for i in range(len(res) - 1)), res
    ML = o.volume()[4]
    assert res[-1] < 1e-9 * float(np.max(ML * np.abs(T0)))
