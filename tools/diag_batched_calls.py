"""Diagnostic: reproducibility of the batched kernels -- the same run twice, and one multi-step
call against one-step calls (bitwise for a deterministic kernel)."""
import os
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_1707_03581_b200 import inputs as I  # noqa: E402
from paper_1707_03581_b200.thermo import Thermo  # noqa: E402

cfg = I.make_config(sys.argv[1] if len(sys.argv) > 1 else "cfg4")
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
S = cfg.n_scen
for mode in ("0", "1"):
    os.environ["THERMO_CGB"] = "2" if mode == "0" else "1"
    runs = []
    for rep in range(2):
        a = Thermo.from_config(cfg)
        a.step(0.0, cfg.dt, n)
        runs.append(np.stack([a.get_T(scen=k) for k in range(S)]))
    b = Thermo.from_config(cfg)
    for k in range(n):
        b.step(k * cfg.dt, cfg.dt, 1)
    B = np.stack([b.get_T(scen=k) for k in range(S)])
    print(f"kernel {'SpMM' if mode == '0' else 'gather'}: run vs rerun max |dT| {np.abs(runs[0] - runs[1]).max():.3e}, "
          f"{n}-step call vs one-step calls {np.abs(runs[0] - B).max():.3e}", flush=True)
