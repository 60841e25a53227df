"""Print the full-run parity errors of the GPU path against the stored oracle runs
(tests/golden/fullrun_*.npz): python tools/fullrun_errors.py

Each GPU CG start (thermo_set_guess: 0 = T^n, 2 = quadratic extrapolation, the default) is
compared with the oracle run of the same start (fullrun_<cfg>.npz / fullrun_<cfg>_g2.npz), and
for context also with the other one: over thousands of steps the solver-tolerance errors of two
different starts drift apart by ~1e-9 (reading R17)."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_1707_03581_b200 import inputs as I  # noqa: E402
from paper_1707_03581_b200.thermo import Thermo  # noqa: E402


def golden(name, guess):
    path = os.path.join("tests", "golden", f"fullrun_{name}{'_g%d' % guess if guess else ''}.npz")
    return np.load(path) if os.path.exists(path) else None


for name in ("cfg2", "cfg3", "cfg4"):
    cfg = I.make_config(name)
    for gpu_guess in (0, 2):
        ref = golden(name, gpu_guess)
        if ref is None:
            continue
        meta = json.loads(str(ref["meta"]))
        th = Thermo.from_config(cfg)
        th.set_guess(gpu_guess)
        th.step(meta["t0"], cfg.dt, meta["nsteps"])
        for ref_guess in (gpu_guess, 2 - gpu_guess):
            g = golden(name, ref_guess)
            if g is None:
                continue
            tag = f"GPU start {gpu_guess} vs oracle start {ref_guess}{' (same start)' if ref_guess == gpu_guess else ''}"
            if "rows" in g:
                T = th.get_T()
                m = json.loads(str(g["meta"]))
                err = np.abs(T[g["rows"]] - g["values"]).max() / np.abs(g["values"]).max()
                print(f"{name}: {m['nsteps']} steps, {len(g['rows'])} sampled DoF, {tag}: max rel err {err:.2e}, "
                      f"sum rel err {abs(T.sum() - m['T_sum']) / abs(m['T_sum']):.2e}", flush=True)
            else:
                errs = [np.abs(th.get_T(scen=int(k)) - v).max() / np.abs(v).max() for k, v in zip(g["scen"], g["values"])]
                print(f"{name}: {meta['nsteps']} steps, scenarios {[int(k) for k in g['scen']]}, {tag}: "
                      f"max rel err {max(errs):.2e}", flush=True)
        th.close()
