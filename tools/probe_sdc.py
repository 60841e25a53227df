"""Device time per step of the SDC methods on a config: python tools/probe_sdc.py cfg1 mrsdc 3 2 1 [steps]"""
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_1707_03581_b200 import inputs as I
from paper_1707_03581_b200.thermo import Thermo

name, method, M, P, K = sys.argv[1], sys.argv[2], int(sys.argv[3]), int(sys.argv[4]), int(sys.argv[5])
n = int(sys.argv[6]) if len(sys.argv) > 6 else 20
cfg = I.make_config(name)
th = Thermo.from_config(cfg)
th.set_method(method, M, P, K)
th.step(0.0, 1.0, 2)
s = torch.cuda.current_stream()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
t0 = time.perf_counter()
e0.record(s)
th.step(2.0, 1.0, n)
e1.record(s)
torch.cuda.synchronize()
wall = time.perf_counter() - t0
st = th.stats()
print(f"{name} {method}({M},{P}) k={K}: {e0.elapsed_time(e1) / n:.3f} ms/step device, {wall / n * 1e3:.3f} ms/step wall, "
      f"CG iterations/step {st['total_iters'] / max(1, st['last_nsteps']):.1f}")
