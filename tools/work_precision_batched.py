"""Batched work-precision harness: S scenario variants (friction levels,
motion periods) advanced together by the batched implicit-Euler path, one batched run per
step size, errors against a fine-step Richardson reference of the same batch.  The analogue of
the paper's error-vs-look-ahead study for many digital twins at once: every
variant reaches t_end after the same device time, so the look-ahead factor
eta = t_end / device time holds for all of them simultaneously.

    python tools/work_precision_batched.py [S] [t_end]
"""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1707_03581_b200 import inputs as I  # noqa: E402
from paper_1707_03581_b200.thermo import Thermo  # noqa: E402

S = int(sys.argv[1]) if len(sys.argv) > 1 else 64
t_end = float(sys.argv[2]) if len(sys.argv) > 2 else 60.0
cfg = I.make_config("cfg4", n_scen=S)
th = Thermo.from_config(cfg)
stream = torch.cuda.current_stream()
T0 = np.stack([th.get_T(scen=s) for s in range(S)])


def run(dt):
    for s in range(S):
        th.set_T(T0[s], scen=s)
    n = int(round(t_end / dt))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    th.step(0.0, dt, n)
    e1.record(stream)
    torch.cuda.synchronize()
    return np.stack([th.get_T(scen=s) for s in range(S)]), e0.elapsed_time(e1) * 1e-3


# reference: Richardson extrapolation of the two finest implicit-Euler runs (first order)
fine = 1.0 / 64
Ta, _ = run(fine)
Tb, _ = run(fine / 2)
Tref = 2.0 * Tb - Ta
scale = np.abs(Tref - T0).max(axis=1)                   # largest temperature change per variant
rows = []
for dt in (4.0, 2.0, 1.0, 0.5, 0.25, 0.125):
    T, sec = run(dt)
    err = np.abs(T - Tref).max(axis=1) / scale
    rows.append({"dt": dt, "err_median": float(np.median(err)), "err_max": float(err.max()),
                 "err_min": float(err.min()), "seconds": sec, "lookahead": t_end / sec,
                 "dof_steps_per_s": cfg.n_dof * S * (t_end / dt) / sec})
print(f"# batched work-precision: {S} variants of cfg4 (eta_k = 100 + 15k W/m^2, period 20 + k s) on the "
      f"cfg1 meshes ({cfg.n_dof} DoF each), implicit Euler, t_end = {t_end} s; reference = Richardson of "
      f"dt = {fine} and {fine / 2} s; error = max-norm over DoF / max |T_ref - T0|, per variant")
print(f"{'dt [s]':>8s} {'median err':>12s} {'max err':>12s} {'device s':>10s} {'look-ahead':>11s} "
      f"{'DoF-steps/s':>12s}")
for r in rows:
    print(f"{r['dt']:8.3f} {r['err_median']:12.3e} {r['err_max']:12.3e} {r['seconds']:10.4f} "
          f"{r['lookahead']:11.1f} {r['dof_steps_per_s']:12.3e}")
print(json.dumps(rows))
