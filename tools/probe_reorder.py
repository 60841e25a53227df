"""Numbering-independence probe: device time per CG iteration of the lattice-ordered config
against the same config with its nodes randomly renumbered (inputs.permute_config), which the
library renumbers internally (reverse Cuthill-McKee; THERMO_REORDER=2: rooted at the interface) at create.

    python tools/probe_reorder.py cfg2 cfg3 [K]
"""
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_1707_03581_b200 import inputs as I  # noqa: E402
from paper_1707_03581_b200.thermo import Thermo  # noqa: E402


def run(cfg, K):
    t0 = time.time()
    th = Thermo.from_config(cfg)
    torch.cuda.synchronize()
    t_create = time.time() - t0
    st0 = th.stats()
    th.set_timing(True)
    th.step(0.0, cfg.dt, 3)
    th.step(3 * cfg.dt, cfg.dt, K)
    st = th.stats()
    it = st["total_iters"]
    th.close()
    return {"create_s": t_create, "reordered": st0["reordered"], "probe_runs": st0["order_max_runs"],
            "probe_window": st0["order_max_window"], "kind": st0["solve_kind"], "variant": st0["solve_variant"],
            "runs": st0["solve_max_runs"], "window": st0["solve_window"],
            "us_per_iter": st["ms_solve"] / it * 1e3, "iters_per_step": it / K,
            "ms_per_step": (st["ms_solve"] + st["ms_iface"]) / K}


args = [a for a in sys.argv[1:] if a.startswith("cfg")]
K = int(sys.argv[-1]) if sys.argv[-1].isdigit() else 10
for name in args:
    cfg = I.make_config(name)
    a = run(cfg, K)
    pcfg, _ = I.permute_config(cfg, seed=99)
    b = run(pcfg, K)
    print(f"{name} lattice order : {a}", flush=True)
    print(f"{name} random + RCM  : {b}", flush=True)
    print(f"{name} per-iteration ratio (random + RCM / lattice): {b['us_per_iter'] / a['us_per_iter']:.3f}", flush=True)
