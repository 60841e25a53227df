"""Work-precision of implicit Euler, single-rate SDC(3) and MRSDC(3,2) on the B200 (synthetic
analogue of the paper's Fig. 7): time-discretisation error at t_end against the
look-ahead factor eta = simulated time / device time.

    python tools/work_precision.py [config] [t_end]

The reference solution is MRSDC(3,2) with 3 sweeps at a step 16x smaller than the finest
tested step.  Errors are max-norm over all DoF, relative to the largest temperature change
max|T_ref - T0|.  Device time is measured with CUDA events around thermo_step.
"""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1707_03581_b200 import inputs as I
from paper_1707_03581_b200.thermo import Thermo

name = sys.argv[1] if len(sys.argv) > 1 else "cfg1"
t_end = float(sys.argv[2]) if len(sys.argv) > 2 else 60.0
cfg = I.make_config(name)
th = Thermo.from_config(cfg)
T0 = th.get_T()
stream = torch.cuda.current_stream()


def run(method, dt, M=3, P=2, K=1):
    th.set_T(T0)
    if method == "ie":
        th.set_method("ie")
    else:
        th.set_method(method, M, P, K)
    n = int(round(t_end / dt))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    th.step(0.0, dt, n)
    e1.record(stream)
    torch.cuda.synchronize()
    return th.get_T(), e0.elapsed_time(e1) * 1e-3


dts = [4.0, 2.0, 1.0, 0.5, 0.25]
Tref, tref = run("mrsdc", dts[-1] / 16, 3, 2, 3)
scale = float(np.abs(Tref - T0).max())
rows = []
for dt in dts:
    T, sec = run("ie", dt)
    rows.append({"method": "implicit Euler", "dt": dt, "err": float(np.abs(T - Tref).max() / scale),
                 "seconds": sec, "lookahead": t_end / sec})
for K in (0, 1, 2):
    for dt in dts:
        T, sec = run("mrsdc", dt, 3, 2, K)
        rows.append({"method": f"MRSDC(3,2) k={K}", "dt": dt, "err": float(np.abs(T - Tref).max() / scale),
                     "seconds": sec, "lookahead": t_end / sec})
for K in (0, 1, 2):
    for dt in dts:
        T, sec = run("sdc", dt, 3, 1, K)
        rows.append({"method": f"SDC(3) k={K}", "dt": dt, "err": float(np.abs(T - Tref).max() / scale),
                     "seconds": sec, "lookahead": t_end / sec})
print(f"# work-precision on {name} ({cfg.n_dof} DoF), t_end = {t_end} s, reference MRSDC(3,2) k=3 "
      f"dt = {dts[-1] / 16} s ({tref:.2f} s), error relative to max|T_ref - T0| = {scale:.4f} K")
print(f"{'method':20s} {'dt [s]':>8s} {'rel. error':>12s} {'device s':>10s} {'look-ahead':>12s}")
for r in rows:
    print(f"{r['method']:20s} {r['dt']:8.3f} {r['err']:12.3e} {r['seconds']:10.4f} {r['lookahead']:12.1f}")
print(json.dumps(rows))
