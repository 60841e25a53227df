"""Full-run parity at the stand scale (BASELINE.json configs[2]: 1.28 M DoF, 3600 steps;
configs[3]: 10 M DoF, 200 steps) and for the batch (configs[4]: 64 scenarios, 500 steps): the
GPU temperatures after the configured run against the oracle's, stored by
tools/make_golden_fullrun.py (which calls only oracle/) at a seeded sample of DoF (every
interface node + 20k uniform) for configs 2-3 and as whole fields of sampled scenarios for
config 4.  North-star bar: max-norm relative error <= 1e-9 after the full run."""
import json
import os

import numpy as np
import pytest

from paper_1707_03581_b200 import inputs as I

pytestmark = [pytest.mark.gpu, pytest.mark.slow]
GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@pytest.fixture(scope="module", autouse=True)
def _built():
    import __graft_entry__ as g
    g.build()


@pytest.mark.parametrize("name", ["cfg2", "cfg3"])
def test_full_run_vs_oracle_samples(name):
    path = os.path.join(GOLDEN, f"fullrun_{name}.npz")
    if not os.path.exists(path):
        pytest.skip(f"{path} not generated (tools/make_golden_fullrun.py {name})")
    from paper_1707_03581_b200.thermo import Thermo
    g = np.load(path)
    meta = json.loads(str(g["meta"]))
    cfg = I.make_config(name)
    assert meta["n_dof"] == cfg.n_dof and meta["dt"] == cfg.dt
    th = Thermo.from_config(cfg)
    th.step(meta["t0"], cfg.dt, meta["nsteps"])
    T = th.get_T()
    ref = g["values"]
    err = np.abs(T[g["rows"]] - ref).max() / np.abs(ref).max()
    assert err <= 1e-9, err
    # whole-field properties the oracle recorded (range and sum)
    assert abs(T.max() - meta["T_max"]) <= 1e-9 * abs(meta["T_max"])
    assert abs(T.min() - meta["T_min"]) <= 1e-9 * abs(meta["T_max"])
    assert abs(T.sum() - meta["T_sum"]) <= 1e-9 * abs(meta["T_sum"])


def test_cfg4_full_run_vs_oracle_scenarios():
    path = os.path.join(GOLDEN, "fullrun_cfg4.npz")
    if not os.path.exists(path):
        pytest.skip(f"{path} not generated (tools/make_golden_fullrun.py cfg4)")
    from paper_1707_03581_b200.thermo import Thermo
    g = np.load(path)
    meta = json.loads(str(g["meta"]))
    cfg = I.make_config("cfg4")
    assert meta["n_dof"] == cfg.n_dof and meta["n_scen"] == cfg.n_scen
    th = Thermo.from_config(cfg)
    th.step(meta["t0"], cfg.dt, meta["nsteps"])
    for k, ref in zip(g["scen"], g["values"]):
        T = th.get_T(scen=int(k))
        err = np.abs(T - ref).max() / np.abs(ref).max()
        assert err <= 1e-9, (int(k), err)
