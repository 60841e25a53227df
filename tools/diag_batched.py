"""Batched kernels A/B (diagnostic): the windowed SpMM kernel against the gather kernel on
configs[4], field difference per scenario every `every` steps; iterations and reported residuals
of the first step where a scenario diverges."""
import os
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_1707_03581_b200 import inputs as I  # noqa: E402
from paper_1707_03581_b200.thermo import Thermo  # noqa: E402

cfg = I.make_config("cfg4")
n = int(sys.argv[1]) if len(sys.argv) > 1 else 500
every = int(sys.argv[2]) if len(sys.argv) > 2 else 25
ths = {}
for mode in ("0", "1"):
    os.environ["THERMO_CGB"] = "2" if mode == "0" else "1"
    ths[mode] = Thermo.from_config(cfg)
t = 0.0
for blk in range(n // every):
    for mode, th in ths.items():
        th.step(t, cfg.dt, every)
    t += every * cfg.dt
    A = np.stack([ths["0"].get_T(scen=k) for k in range(cfg.n_scen)])
    B = np.stack([ths["1"].get_T(scen=k) for k in range(cfg.n_scen)])
    d = np.abs(A - B).max(axis=1) / np.abs(B).max(axis=1)
    ia = ths["0"].step_iters().reshape(every, -1)
    ib = ths["1"].step_iters().reshape(every, -1)
    bad = np.flatnonzero(d > 1e-10)
    print(f"steps {(blk + 1) * every}: max diff {d.max():.2e} (scen {d.argmax()}), iters new/old sum "
          f"{ia.sum()}/{ib.sum()}, scenarios > 1e-10: {bad.tolist()[:10]}", flush=True)
    if bad.size:
        k = bad[0]
        print("  scenario", k, "iters new", ia[:, k].tolist(), "old", ib[:, k].tolist(), flush=True)
        break
