"""Stationary-solve probe: iterations, true residual and device time of
thermo_stationary on a configuration (uncoupled and coupled), e.g. python tools/probe_stationary.py cfg3"""
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_1707_03581_b200 import inputs as I  # noqa: E402
from paper_1707_03581_b200.thermo import Thermo  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
cfg = I.make_config(name)
for coupled in (False, True):
    th = Thermo.from_config(cfg)
    th.set_solver(rtol=1e-12, maxit=50000)
    s = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(s)
    th.stationary(0.0, coupled)
    e1.record(s)
    torch.cuda.synchronize()
    st = th.stats()
    ms = e0.elapsed_time(e1)
    print(f"{name} stationary coupled={coupled}: {st['max_iters']} iterations (incl. true-residual restarts), "
          f"true rel res {st['last_relres']:.2e}, {ms:.1f} ms ({ms / max(st['max_iters'], 1) * 1e3:.1f} us/iter)",
          flush=True)
    th.close()
