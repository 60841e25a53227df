"""End-to-end probe: where the one-step-per-call loop with a host copy of every step's fields
loses time against the device-only run (bench.py's e2e loop).

    python tools/probe_e2e.py [K] [config]          (default: 20, cfg4)
prints ms per step of (a) one K-step call, (b) K one-step calls, (c) K one-step calls each followed
by thermo_get_T_all_async, and the D2H rate of the pinned host buffer.
"""
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_1707_03581_b200 import inputs as I  # noqa: E402
import os  # noqa: E402
import paper_1707_03581_b200.thermo as _T  # noqa: E402
from paper_1707_03581_b200.thermo import Thermo  # noqa: E402

if os.environ.get("DIAG_LIB"):   # another build of libthermo.so (A/B on one box)
    _T.load(os.environ["DIAG_LIB"])

K = int(sys.argv[1]) if len(sys.argv) > 1 else 20
name = sys.argv[2] if len(sys.argv) > 2 else "cfg4"
cfg = I.make_config(name)
stream = torch.cuda.current_stream()
th = Thermo.from_config(cfg, stream=stream.cuda_stream)
t = 0.0
th.step(t, cfg.dt, 5)
t += 5 * cfg.dt
hosts = [torch.empty(th.S * cfg.n_dof, dtype=torch.float64, pin_memory=True) for _ in range(2)]


def timed(fn):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    w0 = time.perf_counter()
    e0.record(stream)
    fn()
    e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / K, (time.perf_counter() - w0) * 1e3 / K


def one_call():
    global t
    th.step(t, cfg.dt, K)
    t += K * cfg.dt


def k_calls():
    global t
    for _ in range(K):
        th.step(t, cfg.dt, 1)
        t += cfg.dt


def k_calls_copy():
    global t
    for k in range(K):
        th.step(t, cfg.dt, 1)
        th.get_T_all_async(hosts[k & 1].data_ptr())
        t += cfg.dt
    th.sync()


for label, fn in (("one K-step call", one_call), ("K one-step calls", k_calls),
                  ("K one-step calls + get_T_all_async", k_calls_copy)):
    fn()   # warm
    ev, wall = timed(fn)
    it = th.step_iters()
    print(f"{name} {label:38s}: {ev:.3f} ms/step (events), {wall:.3f} ms/step (wall); iterations of the last call {it.ravel()[:12].tolist()}", flush=True)
dev = torch.empty(th.S * cfg.n_dof, dtype=torch.float64, device="cuda")
torch.cuda.synchronize()
w0 = time.perf_counter()
for k in range(10):
    hosts[k & 1].copy_(dev, non_blocking=True)
torch.cuda.synchronize()
dtm = (time.perf_counter() - w0) / 10
print(f"D2H of {dev.numel() * 8 / 1e6:.1f} MB into pinned memory: {dtm * 1e3:.3f} ms, {dev.numel() * 8 / dtm / 1e9:.1f} GB/s")
