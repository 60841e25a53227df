"""Batched work-precision harness: the paper's three method classes --
implicit Euler, single-rate SDC(3) and MRSDC(3,2) with k = 0, 1, 2 sweeps (P:722-747,
Fig. 7) -- each run on S scenario variants (friction levels, motion periods) advanced
together by the batched path, one batched run per method and step size.  Errors against a
reference of the same batch: MRSDC(3,2) with 3 sweeps at a step 16x smaller than the finest
tested step.  Every variant of a run reaches t_end after the same device time, so the
look-ahead factor eta = t_end / device time holds for all of them at once.

    python tools/work_precision_batched.py [S] [t_end]
"""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1707_03581_b200 import inputs as I  # noqa: E402
from paper_1707_03581_b200.thermo import Thermo  # noqa: E402


def work_precision(S=64, t_end=60.0, dts=(4.0, 2.0, 1.0, 0.5, 0.25), sweeps=(0, 1, 2), cfg_name="cfg4"):
    """Rows {method, dt, err_median, err_max, seconds, lookahead, dof_steps_per_s} and the header."""
    cfg = I.make_config(cfg_name, n_scen=S)
    th = Thermo.from_config(cfg)
    stream = torch.cuda.current_stream()
    T0 = np.stack([th.get_T(scen=s) for s in range(S)])

    def run(method, dt, M=3, P=2, K=1):
        for s in range(S):
            th.set_T(T0[s], scen=s)
        th.set_method(method, M, P, K) if method != "ie" else th.set_method("ie")
        n = int(round(t_end / dt))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        th.step(0.0, dt, n)
        e1.record(stream)
        torch.cuda.synchronize()
        return np.stack([th.get_T(scen=s) for s in range(S)]), e0.elapsed_time(e1) * 1e-3

    Tref, tref = run("mrsdc", dts[-1] / 16, 3, 2, 3)
    scale = np.abs(Tref - T0).max(axis=1)                   # largest temperature change per variant
    rows = []

    def record(label, method, dt, M=3, P=2, K=1):
        T, sec = run(method, dt, M, P, K)
        err = np.abs(T - Tref).max(axis=1) / scale
        rows.append({"method": label, "dt": dt, "err_median": float(np.median(err)), "err_max": float(err.max()),
                     "seconds": sec, "lookahead": t_end / sec,
                     "dof_steps_per_s": cfg.n_dof * S * (t_end / dt) / sec})

    for dt in dts:
        record("implicit Euler", "ie", dt)
    for K in sweeps:
        for dt in dts:
            record(f"SDC(3) k={K}", "sdc", dt, 3, 1, K)
    for K in sweeps:
        for dt in dts:
            record(f"MRSDC(3,2) k={K}", "mrsdc", dt, 3, 2, K)
    head = (f"# batched work-precision: {S} variants of {cfg_name} (eta_k = 100 + 15k W/m^2, period 20 + k s) on the "
            f"cfg1 meshes ({cfg.n_dof} DoF each), t_end = {t_end} s, every method batched over all variants; "
            f"reference MRSDC(3,2) k=3 dt = {dts[-1] / 16} s ({tref:.2f} s); error = max-norm over DoF / "
            f"max |T_ref - T0|, per variant (median and max over the variants)")
    return rows, head


if __name__ == "__main__":
    S = int(sys.argv[1]) if len(sys.argv) > 1 else 64
    t_end = float(sys.argv[2]) if len(sys.argv) > 2 else 60.0
    rows, head = work_precision(S, t_end)
    print(head)
    print(f"{'method':18s} {'dt [s]':>7s} {'median err':>11s} {'max err':>11s} {'device s':>9s} {'look-ahead':>11s} "
          f"{'DoF-steps/s':>12s}")
    for r in rows:
        print(f"{r['method']:18s} {r['dt']:7.3f} {r['err_median']:11.3e} {r['err_max']:11.3e} {r['seconds']:9.4f} "
              f"{r['lookahead']:11.1f} {r['dof_steps_per_s']:12.3e}")
    print(json.dumps(rows))
