"""Batched-kernel probe: device time per CG iteration of configs[4] (64 scenarios) with the
phase split (THERMO_CG_TRACE=1 prints phase 0 / S / U per iteration of the last solve).

    THERMO_CG_TRACE=1 python tools/probe_batched.py [K] [S]
"""
import os
import sys

sys.path.insert(0, ".")
from paper_1707_03581_b200 import inputs as I  # noqa: E402
import paper_1707_03581_b200.thermo as _T  # noqa: E402
from paper_1707_03581_b200.thermo import Thermo  # noqa: E402

if os.environ.get("DIAG_LIB"):   # another build of libthermo.so (A/B on one box)
    _T.load(os.environ["DIAG_LIB"])

K = int(sys.argv[1]) if len(sys.argv) > 1 else 5
S = int(sys.argv[2]) if len(sys.argv) > 2 else 64
cfg = I.make_config("cfg4", n_scen=S)
th = Thermo.from_config(cfg)
th.set_timing(True)
if int(os.environ.get("THERMO_CGB_DEBUG", "0")) & 15:   # measurement modes do not converge: fixed iterations
    th.set_solver(1e-12, 20)
    try:
        th.step(0.0, cfg.dt, 1)
    except Exception as e:
        print("debug run:", str(e)[:80])
    sys.exit(0)
th.step(0.0, cfg.dt, 3)
th.step(3.0, cfg.dt, K)
st = th.stats()
it = th.step_iters().reshape(K, -1).max(axis=1)
print(f"cfg4 S={S}: kind {st['solve_kind']}, solve {st['ms_solve'] / K:.3f} ms/step, iface {st['ms_iface'] / K:.3f} ms/step, "
      f"{it.mean():.1f} iterations/step, {st['ms_solve'] / it.sum() * 1e3:.1f} us/iteration", flush=True)
