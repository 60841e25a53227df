"""Print the full-run parity errors of the GPU path against the stored oracle runs
(tests/golden/fullrun_*.npz): python tools/fullrun_errors.py"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_1707_03581_b200 import inputs as I  # noqa: E402
from paper_1707_03581_b200.thermo import Thermo  # noqa: E402

for name in ("cfg2", "cfg3", "cfg4"):
    g = np.load(os.path.join("tests", "golden", f"fullrun_{name}.npz"))
    meta = json.loads(str(g["meta"]))
    cfg = I.make_config(name)
    th = Thermo.from_config(cfg)
    th.step(meta["t0"], cfg.dt, meta["nsteps"])
    if "rows" in g:
        T = th.get_T()
        err = np.abs(T[g["rows"]] - g["values"]).max() / np.abs(g["values"]).max()
        print(f"{name}: {meta['nsteps']} steps, {len(g['rows'])} sampled DoF, max rel err {err:.2e}, "
              f"sum rel err {abs(T.sum() - meta['T_sum']) / abs(meta['T_sum']):.2e}", flush=True)
    else:
        errs = [np.abs(th.get_T(scen=int(k)) - v).max() / np.abs(v).max() for k, v in zip(g["scen"], g["values"])]
        print(f"{name}: {meta['nsteps']} steps, scenarios {list(g['scen'])}, max rel err {max(errs):.2e}", flush=True)
    th.close()
