"""Diagnostic: true relative residual of every batched implicit-Euler step in [n0, n1) of
configs[4] for both batched kernels (SpMM: THERMO_CGB=0, gather: 1), via the oracle's residual
rows; each kernel's residual is taken with its own previous state."""
import os
import sys

import numpy as np

sys.path.insert(0, ".")
import oracle as O  # noqa: E402
from paper_1707_03581_b200 import inputs as I  # noqa: E402
from paper_1707_03581_b200.thermo import Thermo  # noqa: E402

cfg = I.make_config("cfg4")
n0, n1 = int(sys.argv[1]), int(sys.argv[2])
scen = [int(x) for x in sys.argv[3:]] or [48, 56]
ths = {}
for mode in ("0", "1"):
    os.environ["THERMO_CGB"] = "2" if mode == "0" else "1"
    ths[mode] = Thermo.from_config(cfg)
    ths[mode].step(0.0, cfg.dt, n0)
o = O.Oracle.from_config(cfg)
rows = np.arange(cfg.n_dof, dtype=np.int64)
for n in range(n0, n1):
    T0 = {(m, k): ths[m].get_T(scen=k) for m in ths for k in scen}
    for th in ths.values():
        th.step(n * cfg.dt, cfg.dt, 1)
    t1 = (n + 1) * cfg.dt
    out = []
    for k in scen:
        sc = cfg.scenarios[k]
        s, eta = I.scenario_scalars(sc, t1)
        r = {}
        for m in ths:
            res, bn = o.residual_rows(cfg.dt, np.array(sc.dir) * s, eta, T0[(m, k)], ths[m].get_T(scen=k), rows)
            r[m] = np.linalg.norm(res) / bn
        d = np.abs(ths["0"].get_T(scen=k) - ths["1"].get_T(scen=k)).max()
        out.append(f"s{k}: new {r['0']:.1e} old {r['1']:.1e} |dT| {d:.1e}")
    print(f"step {n + 1}: " + "; ".join(out), flush=True)
