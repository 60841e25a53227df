"""Latency probe for paper-scale problems (16,626 DoF; look-ahead factor P:189-194):
device time per implicit-Euler step and per CG iteration of small configurations with the
resident-operator solve (default where the operator fits in shared memory), the single-cluster
solve (THERMO_CG_CLUSTER=1) and the persistent streaming grid kernel (THERMO_CG_CLUSTER=0), one
step per call as a digital twin would run.

    python tools/probe_latency.py [K]
"""
import os
import sys

import torch

sys.path.insert(0, ".")
from paper_1707_03581_b200 import inputs as I  # noqa: E402
from paper_1707_03581_b200.thermo import Thermo  # noqa: E402

K = int(sys.argv[1]) if len(sys.argv) > 1 else 50
for name, jit in (("cfg0", None), ("small", 0.1), ("medium", 0.1), ("paper", 0.1), ("cfg1", None)):
    for mode in ("resident", "cluster", "grid"):
        os.environ.pop("THERMO_CG_CLUSTER", None)
        if mode != "resident":
            os.environ["THERMO_CG_CLUSTER"] = "1" if mode == "cluster" else "0"
        cfg = I.make_config(name, jitter=jit)
        th = Thermo.from_config(cfg)
        th.step(0.0, cfg.dt, 5)
        s = torch.cuda.current_stream()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(s)
        th.step(5 * cfg.dt, cfg.dt, K)   # one call of K steps: device time per step (no per-step events)
        e1.record(s)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / K
        e0.record(s)
        for n in range(K):               # one step per call (a digital twin stepping in real time)
            th.step((5 + K + n) * cfg.dt, cfg.dt, 1)
        e1.record(s)
        torch.cuda.synchronize()
        ms1 = e0.elapsed_time(e1) / K
        th.set_timing(True)              # per-step events for the solve / interface split
        th.step((5 + 2 * K) * cfg.dt, cfg.dt, K)
        st = th.stats()
        its = st["total_iters"] / K
        print(f"{name:7s} N={cfg.n_dof:6d} {mode:8s} (path {st['latency_path']}): {ms * 1e3:7.1f} us/step ({st['ms_solve'] / K * 1e3:6.1f} solve, "
              f"{st['ms_solve'] / max(st['total_iters'], 1) * 1e3:5.2f} us/iter, {its:4.1f} iters), "
              f"{ms1 * 1e3:7.1f} us/step one step per call; look-ahead {cfg.dt / (ms * 1e-3):7.0f}", flush=True)
        th.close()
os.environ.pop("THERMO_CG_CLUSTER", None)
