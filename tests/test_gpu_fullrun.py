"""Full-run parity of the PRODUCT path against a start-agnostic oracle, on every stored DoF.

References (tests/golden/fullrun_<cfg>.npz, written by tools/make_golden_fullrun.py, which
calls only oracle/): the implicit-Euler solution after the configured
run of BASELINE.json configs[1..4], with the oracle's textbook Jacobi-PCG started at x0 = T^n
and driven to a relative residual of 1e-14 (true residual checked at every step's exit), so
the reference does not depend on any CG start and its own solver error is negligible.

The GPU side runs the library's defaults (quadratic-extrapolation CG start, rtol 1e-12 --
the configuration bench.py times), plus the x0 = T^n start as a second mode.  From x0 = T^n
CG stops with a larger error per step (the start is further from the solution, so the last
iteration's error is larger for the same residual bound) and over the 3600 steps of configs[2]
the drift reaches 1.62e-9 at rtol 1e-12 (measured); that mode is therefore run at rtol 2e-13.  North-star
bar: max-norm relative error <= 1e-9 after the full run (reading R18), over
  cfg1, cfg2   every DoF
  cfg3         1.3 M stored DoF (every boundary node, every interface-adjacent node, a seeded
               uniform sample) and the whole-field max / min / sum
  cfg4         every DoF of all 64 scenarios.
The stored values are rounded to 2^-36 (<= 7.3e-12 absolute, tests/golden_codec.py)."""
import json
import os

import numpy as np
import pytest

import golden_codec as G
from paper_1707_03581_b200 import inputs as I

pytestmark = [pytest.mark.gpu, pytest.mark.slow]
GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
TOL = 1e-9
MODES = {"default": (None, None), "x0_Tn": (0, 2e-13)}   # (CG start, rtol)


@pytest.fixture(scope="module", autouse=True)
def _built():
    import __graft_entry__ as g
    g.build()


def _golden(name):
    path = os.path.join(GOLDEN, f"fullrun_{name}.npz")
    if not os.path.exists(path):
        pytest.skip(f"{path} not generated (tools/make_golden_fullrun.py {name})")
    g = np.load(path)
    return g, json.loads(str(g["meta"]))


def _run(cfg, mode, nsteps):
    from paper_1707_03581_b200.thermo import Thermo
    th = Thermo.from_config(cfg)
    guess, rtol = MODES[mode]
    if guess is not None:
        th.set_guess(guess)
    if rtol is not None:
        th.set_solver(rtol=rtol)
    th.step(0.0, cfg.dt, nsteps)
    return th


@pytest.mark.parametrize("mode", list(MODES))
@pytest.mark.parametrize("name", ["cfg1", "cfg2", "cfg3"])
def test_full_run_vs_start_agnostic_oracle(name, mode):
    g, meta = _golden(name)
    cfg = I.make_config(name)
    assert meta["n_dof"] == cfg.n_dof and meta["dt"] == cfg.dt and meta["t0"] == 0.0
    assert "x0 = T^n" in meta["solver"] and meta["max_true_rel_residual"] <= 1e-13
    th = _run(cfg, mode, meta["nsteps"])
    T = th.get_T()
    if "field" in g.files:
        ref = G.unpack_field(g["field"], cfg.n_dof)
        err = np.abs(T - ref).max() / np.abs(ref).max()
    else:
        rows = G.unpack_rows(g["rows"], meta["n_rows"])
        ref = G.unpack_field(g["values"], meta["n_rows"])
        err = np.abs(T[rows] - ref).max() / np.abs(ref).max()
        # whole-field properties the oracle recorded (range and sum)
        assert abs(T.max() - meta["T_max"]) <= TOL * abs(meta["T_max"])
        assert abs(T.min() - meta["T_min"]) <= TOL * abs(meta["T_max"])
        assert abs(T.sum() - meta["T_sum"]) <= TOL * abs(meta["T_sum"])
    print(f"{name} {mode}: max-norm rel err {err:.3e} over the stored DoF")
    assert err <= TOL, err


@pytest.mark.parametrize("mode", list(MODES))
def test_cfg4_full_run_every_scenario(mode):
    g, meta = _golden("cfg4")
    cfg = I.make_config("cfg4")
    S = cfg.n_scen
    assert meta["n_dof"] == cfg.n_dof and meta["n_scen"] == S
    ref = G.unpack_field(g["field"], S * cfg.n_dof).reshape(S, cfg.n_dof)
    th = _run(cfg, mode, meta["nsteps"])
    worst = 0.0
    for k in range(S):
        T = th.get_T(scen=k)
        err = np.abs(T - ref[k]).max() / np.abs(ref[k]).max()
        worst = max(worst, err)
        assert err <= TOL, (k, err)
    print(f"cfg4 {mode}: worst scenario max-norm rel err {worst:.3e}")
