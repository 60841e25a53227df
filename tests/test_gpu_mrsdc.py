"""MRSDC on the GPU against the oracle's Algorithms 1-2 on the same inputs."""
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


@pytest.mark.parametrize("name,jitter,M,P,K", [("small", 0.1, 3, 2, 0), ("small", 0.1, 3, 2, 2),
                                               ("medium", 0.1, 3, 2, 1), ("small", 0.0, 2, 4, 1),
                                               ("cfg0", 0.0, 1, 1, 0)])
def test_mrsdc_parity(name, jitter, M, P, K):
    from paper_1707_03581_b200.thermo import Thermo
    cfg = I.make_config(name, jitter=jitter)
    T0 = I.initial_field(cfg)[0]
    th = Thermo.from_config(cfg)
    th.set_method("mrsdc", M, P, K)
    th.set_T(T0)
    nsteps = 6
    th.step(1.0, cfg.dt, nsteps)
    Tg = th.get_T()
    o = O.Oracle.from_config(cfg)
    Tr, st = o.step_mrsdc(T0, 1.0, cfg.dt, nsteps, cfg.scenarios[0], M, P, K)
    assert rel(Tg, Tr) <= TOL
    s = th.stats()
    assert s["steps_done"] == nsteps and s["failed_step"] == -1


def test_method_switch_and_validation():
    from paper_1707_03581_b200.thermo import Thermo, ThermoError
    cfg = I.make_config("small")
    th = Thermo.from_config(cfg)
    th.set_method("mrsdc", 3, 2, 1)
    th.step(0.0, cfg.dt, 2)
    th.set_method("ie")
    th.step(2 * cfg.dt, cfg.dt, 2)
    o = O.Oracle.from_config(cfg)
    T, _ = o.step_mrsdc(np.full(o.n, cfg.T0), 0.0, cfg.dt, 2, cfg.scenarios[0], 3, 2, 1)
    T, _ = o.step(T, 2 * cfg.dt, cfg.dt, 2, cfg.scenarios[0])
    assert rel(th.get_T(), T) <= TOL
    with pytest.raises(ThermoError):
        th.set_method("mrsdc", 0, 2, 1)
    with pytest.raises(ThermoError):
        th.set_method("mrsdc", 3, 9, 1)


@pytest.mark.slow
def test_mrsdc_stand_scale_one_step():
    """BASELINE configs[2] geometry (1.28 M DoF, jittered L-shape stand): one MRSDC(3,2) k = 1
    step through the C ABI against the oracle's Algorithms 1-2."""
    from paper_1707_03581_b200.thermo import Thermo
    cfg = I.make_config("cfg2")
    th = Thermo.from_config(cfg)
    th.set_method("mrsdc", 3, 2, 1)
    th.step(3.0, cfg.dt, 1)
    o = O.Oracle.from_config(cfg)
    Tr, _ = o.step_mrsdc(np.full(o.n, cfg.T0), 3.0, cfg.dt, 1, cfg.scenarios[0], 3, 2, 1)
    assert rel(th.get_T(), Tr) <= TOL


def _scen(k):
    return I.Scenario(0.375, 0.375, 20.0 + 7 * k, 100.0 + 150.0 * k, 0.3 * k, 9.0)


@pytest.mark.parametrize("method,M,P,K", [("mrsdc", 3, 2, 1), ("mrsdc", 3, 2, 2), ("sdc", 3, 1, 1),
                                          ("sdc", 2, 1, 0)])
def test_batched_sdc_methods_every_column_vs_oracle(method, M, P, K):
    """Batched SDC methods (S = 3 scenarios with their own motion and friction laws, advanced
    together): every column against an independent oracle run of its scenario (Algorithms 1-2 /
    single-rate SDC), and the same as a single-scenario GPU run to the solver
    tolerance."""
    from paper_1707_03581_b200.thermo import Thermo
    cfg = I.make_config("small", jitter=0.1)
    scen = [_scen(k) for k in range(3)]
    T0 = I.initial_field(cfg)[0]
    tb = Thermo.from_config(cfg, scenarios=scen)
    tb.set_method(method, M, P, K)
    for k in range(3):
        tb.set_T(T0, scen=k)
    nsteps = 5
    tb.step(1.0, cfg.dt, nsteps)
    assert tb.stats()["failed_step"] == -1
    for k, sc in enumerate(scen):
        o = O.Oracle.from_config(cfg)
        if method == "mrsdc":
            Tr, _ = o.step_mrsdc(T0, 1.0, cfg.dt, nsteps, sc, M, P, K)
        else:
            Tr, _ = o.step_sdc(T0, 1.0, cfg.dt, nsteps, sc, M, K)
        assert rel(tb.get_T(scen=k), Tr) <= TOL, k
        ts = Thermo.from_config(cfg, scenarios=[sc])
        ts.set_method(method, M, P, K)
        ts.set_T(T0)
        ts.step(1.0, cfg.dt, nsteps)
        assert rel(tb.get_T(scen=k), ts.get_T()) <= 1e-11, k


def test_batched_work_precision_harness():
    """tools/work_precision_batched.py on a small batch: every method class runs
    batched; errors fall with dt for each class, the corrected SDC methods beat implicit Euler at
    equal dt, and one batched run advances all variants together."""
    import importlib.util
    import os
    path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools",
                        "work_precision_batched.py")
    spec = importlib.util.spec_from_file_location("wpb", path)
    wpb = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(wpb)
    rows, head = wpb.work_precision(S=4, t_end=8.0, dts=(2.0, 1.0), sweeps=(1, 2))
    by = {}
    for r in rows:
        by.setdefault(r["method"], {})[r["dt"]] = r["err_max"]
    assert set(by) == {"implicit Euler", "SDC(3) k=1", "SDC(3) k=2", "MRSDC(3,2) k=1", "MRSDC(3,2) k=2"}
    for m, e in by.items():
        assert e[1.0] < e[2.0], (m, e)
    for m in ("SDC(3) k=2", "MRSDC(3,2) k=2"):
        assert by[m][1.0] < by["implicit Euler"][1.0], (m, by)
