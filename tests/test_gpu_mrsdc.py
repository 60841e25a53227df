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
    cfgb = I.make_config("small")
    cfgb.scenarios = cfgb.scenarios * 2
    tb = Thermo.from_config(cfgb)
    with pytest.raises(ThermoError):
        tb.set_method("mrsdc", 3, 2, 1)


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
