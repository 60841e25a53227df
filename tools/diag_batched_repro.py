import os, sys
import numpy as np
sys.path.insert(0, ".")
from paper_1707_03581_b200 import inputs as I
from paper_1707_03581_b200.thermo import Thermo
cfg = I.make_config("cfg4")
nf = cfg.fixed.n_nodes
for n in (1, 2, 3, 5):
    runs = []
    for rep in range(3):
        a = Thermo.from_config(cfg)
        a.step(0.0, cfg.dt, n)
        runs.append(np.stack([a.get_T(scen=k) for k in range(64)]))
        it = a.step_iters().reshape(n, -1)
    for rep in (1, 2):
        d = np.abs(runs[0] - runs[rep])
        if d.max() > 0:
            k, i = np.unravel_index(d.argmax(), d.shape)
            sc = np.flatnonzero(d.max(axis=1) > 0)
            print(f"n={n} rep{rep}: max {d.max():.2e} scen {k} row {i} ({'fixed' if i < nf else 'moving'}), scenarios differing {sc.tolist()[:20]}, rows differing {int((d > 0).sum())}")
        else:
            print(f"n={n} rep{rep}: identical")
