"""Single-rate SDC on the GPU (method 2: P:354-413 with the interface implicit, reading R29)
against the oracle's or_step_sdc on the same inputs."""
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


@pytest.mark.parametrize("name,jitter,M,K", [("small", 0.1, 3, 0), ("small", 0.1, 3, 2), ("medium", 0.1, 3, 1),
                                             ("small", 0.0, 2, 3), ("cfg0", 0.0, 1, 0)])
def test_sdc_parity(name, jitter, M, K):
    from paper_1707_03581_b200.thermo import Thermo
    cfg = I.make_config(name, jitter=jitter)
    T0 = I.initial_field(cfg)[0]
    th = Thermo.from_config(cfg)
    th.set_method("sdc", M, 1, K)
    th.set_T(T0)
    nsteps = 5
    th.step(1.0, cfg.dt, nsteps)
    o = O.Oracle.from_config(cfg)
    Tr, st = o.step_sdc(T0, 1.0, cfg.dt, nsteps, cfg.scenarios[0], M, K)
    assert rel(th.get_T(), Tr) <= TOL
    s = th.stats()
    assert s["steps_done"] == nsteps and s["failed_step"] == -1


def test_one_node_sdc_equals_implicit_euler_on_gpu():
    """M = 1 with sweeps reproduces the GPU implicit-Euler path (to CG tolerance)."""
    from paper_1707_03581_b200.thermo import Thermo
    cfg = I.make_config("small", jitter=0.1)
    T0 = I.initial_field(cfg)[0]
    a, b = Thermo.from_config(cfg), Thermo.from_config(cfg)
    a.set_T(T0)
    b.set_T(T0)
    a.step(0.0, cfg.dt, 4)
    b.set_method("sdc", 1, 1, 2)
    b.step(0.0, cfg.dt, 4)
    assert rel(b.get_T(), a.get_T()) <= TOL
