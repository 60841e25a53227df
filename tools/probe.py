"""Quick timing probe: python tools/probe.py cfg1 100  (device-timed, not the bench)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1707_03581_b200 import inputs as I
from paper_1707_03581_b200.thermo import Thermo

name = sys.argv[1] if len(sys.argv) > 1 else "cfg1"
K = int(sys.argv[2]) if len(sys.argv) > 2 else 20
t0 = time.time()
cfg = I.make_config(name)
t1 = time.time()
th = Thermo.from_config(cfg)
torch.cuda.synchronize()
t2 = time.time()
st = th.stats()
print(f"{name}: N={cfg.n_dof} nnz={st['nnz_volume']} pad={st['nnz_volume_padded']} n_if={st['n_iface_rows']} cap={st['iface_capacity']} gen={t1-t0:.1f}s create={t2-t1:.1f}s", flush=True)
if os.environ.get("GUESS"):
    th.set_guess(int(os.environ["GUESS"]))
th.set_timing(True)
th.step(0.0, cfg.dt, 3)
s = torch.cuda.current_stream()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(s)
th.step(3 * cfg.dt, cfg.dt, K)
e1.record(s)
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / K
it = th.step_iters()[:, 0]
N, Z = cfg.n_dof, st["nnz_volume"]
bytes_it = 12 * Z + 108 * N
gbs = (it.mean() * bytes_it + 12 * Z + 40 * N) / (ms * 1e-3) / 1e9
print(f"{name}: {ms:.3f} ms/step, iters/step {it.mean():.1f} (min {it.min()} max {it.max()}), "
      f"DoF-steps/s {N / (ms * 1e-3):.3e}, alg GB/s {gbs:.0f}, per-iter {ms / it.mean() * 1e3:.1f} us", flush=True)
st = th.stats()
print(f"{name}: CG iterations of the timed steps (launches 4..{3 + K}): {[int(x) for x in it]}", flush=True)
print(f"{name}: iface {st['ms_iface'] / K * 1e3:.1f} us/step, solve {st['ms_solve'] / K:.3f} ms/step "
      f"({st['ms_solve'] / K / it.mean() * 1e3:.1f} us/iter), grid {st['solve_grid']}x{st['solve_block']}", flush=True)
