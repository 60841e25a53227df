#!/usr/bin/env python
"""bench.py -- BASELINE.json metric: coupled implicit DoF-steps/s (fp64) and SpMV/CG HBM GB/s.

Workload: BASELINE.json configs[3], the roofline configuration
(fixed L-shape stand 7,968,341 DoF + stock 2,050,401 DoF = 10,018,742 DoF, jittered Kuhn
tetrahedra, implicit Euler dt = 1 s, CG to relative residual 1e-12, Jacobi preconditioner,
fp64).  One "step" = one implicit-Euler time step of the whole hot path: interface
re-integration + right-hand side (a3) + Jacobi-PCG solve (a4) + commit (a6).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl thermo|reference]

Rank 0 prints one JSON line.  Multi-GPU: the single-run IE step does not shard (DESIGN.md:
"replicas only"); under torchrun each rank advances its own replica, `value` is the
whole-job DoF-steps/s over the max-over-ranks device time, scaling "weak".  The batched
configuration (--config cfg4, 64 scenarios) shards its scenarios over the ranks with no
data-path collective (paper_1707_03581_b200/dist.py); scaling "strong" (total work fixed).
--impl reference times the CPU oracle (oracle/, the reference arm for this tier) on a
bounded sample of the same workload on the host cores.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "coupled implicit DoF-steps/s (fp64) and SpMV/CG HBM GB/s vs 8 TB/s peak"
UNIT = "DoF-steps/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="thermo", choices=["thermo", "reference"])
    ap.add_argument("--config", default="cfg3")
    ap.add_argument("--e2e-steps", type=int, default=10)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    return ap.parse_args()


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def ncu_traffic(cfg_name):
    """Per-launch DRAM bytes of the CG kernel from the committed ncu --set full capture."""
    path = os.path.join(ROOT, "profiles", "ncu_cg_summary.json")
    try:
        with open(path) as f:
            d = json.load(f)
        e = d[cfg_name]
        return e
    except Exception:
        return None


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), "--query-gpu=" + self.FIELDS,
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        time.sleep(0.3)
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.2)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in self.rows:
            for n, v in zip(names, r[3:7]):
                if v.strip().lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(self.rows)}


def dist_setup():
    from paper_1707_03581_b200.dist import env_world
    return env_world()


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_baseline(cfg, steps=1):
    """The oracle as it stands (plain C; its CG loops on all host cores via OpenMP, assembly and
    interface serial) on a bounded sample: `steps` full IE steps of the same workload;
    create/assembly excluded from the timed region."""
    import oracle as O
    t0 = time.time()
    o = O.Oracle.from_config(cfg)
    t_create = time.time() - t0
    T = np.full(o.n, cfg.T0)
    t0 = time.perf_counter()
    T, st = o.step(T, 0.0, cfg.dt, steps, cfg.scenarios[0])
    dt = time.perf_counter() - t0
    thr = O.threads()
    return {"value": cfg.n_dof * steps / dt, "unit": UNIT, "cores": thr, "kind": "oracle",
            "cpu_model": cpu_model(), "nproc": os.cpu_count(),
            "sample": f"{steps} full implicit-Euler step(s) of {cfg.name} ({cfg.n_dof} DoF, scenario 0), C oracle "
                      f"with its CG loops on {thr} OpenMP threads ({os.cpu_count()} host cores, {cpu_model()}), "
                      f"CG iterations {int(st[:, 0].sum())}, assembly ({t_create:.0f} s) untimed",
            "seconds": dt}


def workload_name(name):
    return {"cfg0": "configs[0]", "cfg1": "configs[1]", "cfg2": "configs[2]", "cfg3": "configs[3]",
            "cfg4": "configs[4]"}.get(name, name)


def run_reference(args):
    world, rank, local = dist_setup()
    if rank != 0:
        return
    from paper_1707_03581_b200 import inputs as I
    cfg = I.make_config(args.config)
    steps = max(1, min(args.steps, 2))
    cb = cpu_baseline(cfg, steps)
    line = {"impl": "reference", "metric": METRIC, "value": cb["value"], "unit": UNIT, "n_gpus": args.gpus,
            "steps": steps, "warmup": 0, "ms_per_step": cb["seconds"] / steps * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"BASELINE {workload_name(cfg.name)} ({cfg.name}): {cfg.description}",
                       "n_dof": cfg.n_dof,
                       "dt": cfg.dt, "sample": f"{steps} of the requested {args.steps} steps (bounded)"},
            "cpu_baseline": {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample", "cpu_model", "nproc")},
            "e2e": {"value": cb["value"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def run_thermo(args):
    import torch
    world, rank, local = dist_setup()
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_1707_03581_b200 import dist as D
    from paper_1707_03581_b200 import inputs as I
    from paper_1707_03581_b200.thermo import Thermo

    W = max(3, args.warmup)
    K = args.steps
    cfg_all = I.make_config(args.config)
    sharded = cfg_all.n_scen > 1 and world > 1     # batched mode: scenarios split over ranks
    cfg = D.shard_config(cfg_all, rank, world) if sharded else cfg_all
    stream = torch.cuda.current_stream()
    th = Thermo.from_config(cfg, stream=stream.cuda_stream)
    th.set_timing(True)
    t = 0.0
    th.step(t, cfg.dt, W)
    t += W * cfg.dt
    st0 = th.stats()
    # the state after the warm-up: the e2e loop below restarts from it, so that both timed regions
    # cover the same step times (the cost of a step varies with the stock's position and speed)
    t_w = t
    snap = torch.empty(th.S * cfg.n_dof, dtype=torch.float64, pin_memory=True)
    th.get_T_all_async(snap.data_ptr())
    th.sync()
    snap_np = snap.numpy()

    def barrier():
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()

    # ---- timed region: K implicit-Euler steps, inputs resident in HBM
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    with ClockSampler(local) as clk:
        e0.record(stream)
        th.step(t, cfg.dt, K)
        e1.record(stream)
        torch.cuda.synchronize()
    barrier()
    t += K * cfg.dt
    ms = e0.elapsed_time(e1)
    st = th.stats()
    iters = th.step_iters().max(axis=1)      # loop iterations of the (batched) solve per step
    ms_max = D.max_over_ranks(ms, device="cuda")

    # ---- e2e through the C ABI with host buffers: per step, H2D of the step's time scalars
    # (inside thermo_step) + D2H of the whole temperature field of every scenario into pinned
    # host memory (thermo_get_T_async: the copy of step k overlaps step k + 1; two host
    # buffer sets alternate); thermo_sync waits for the last copies inside the timed region
    KE = max(1, args.e2e_steps)
    # (all scenarios of a batched context in one transfer: thermo_get_T_all_async)
    hosts = [torch.empty(th.S * cfg.n_dof, dtype=torch.float64, pin_memory=True) for _ in range(2)]
    th.set_timing(False)   # (the per-step CUDA events served the roofline split of the timed region above)
    for s_ in range(th.S):   # back to the state after the warm-up (same step times as the timed region)
        th.set_T(snap_np[s_ * cfg.n_dof:(s_ + 1) * cfg.n_dof], scen=s_)
    t = t_w
    for k in range(3):   # untimed: the extrapolation history restarts after set_T; the first host
        th.step(t, cfg.dt, 1)   # copies allocate the library's staging buffers
        th.get_T_all_async(hosts[k & 1].data_ptr())
        t += cfg.dt
    th.sync()
    barrier()
    e2, e3 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e2.record(stream)
    e2e_iters = 0.0
    for k in range(KE):
        th.step(t, cfg.dt, 1)
        # the step's CG iterations (reported next to the e2e value), read BEFORE the field copy is
        # queued: a small device-to-host copy issued behind the 80-MB transfer waits for it on the
        # copy engine (1.3 ms per step on configs[3])
        e2e_iters += float(th.step_iters().max())
        th.get_T_all_async(hosts[k & 1].data_ptr())
        t += cfg.dt
    th.sync()
    e3.record(stream)
    torch.cuda.synchronize()
    ms_e2e = D.max_over_ranks(e2.elapsed_time(e3), device="cuda")

    if rank != 0:
        if world > 1:
            torch.distributed.barrier()
            torch.distributed.destroy_process_group()
        return
    N, Z, S = cfg.n_dof, st["nnz_volume"], th.S
    units = N * cfg_all.n_scen if sharded else world * N * S     # DoF-steps per step, whole job
    value = units * K / (ms_max * 1e-3)
    # roofline of the dominant kernel (the persistent CG solve, one launch per step):
    # SURVEY 8(d) per-iteration bytes 12 Z + 108 N, plus 12 Z + 40 N for r0 = b - K~ x0;
    # batched: 12 Z + 4 N + S 104 N per iteration (SURVEY 8(d) cfg 4 row), 12 Z + S 40 N phase 0
    if S == 1:
        per_iter, phase0 = 12 * Z + 108 * N, 12 * Z + 40 * N
    else:
        per_iter, phase0 = 12 * Z + 4 * N + S * 104 * N, 12 * Z + S * 40 * N
    alg_bytes = float(iters.sum()) * per_iter + K * phase0
    achieved = alg_bytes / (st["ms_solve"] * 1e-3) / 1e9
    peak, peak_kind = peaks()
    prof = ncu_traffic(args.config)
    traffic, dram = None, {}
    if prof:
        traffic = prof.get("dram_bytes_per_launch")
        if prof.get("cg_iterations") and S == 1:
            # actual DRAM bytes per CG iteration (ncu, one launch) x this run's iterations / time
            per_it = traffic / (prof["cg_iterations"] + 0.82)   # phase 0 ~ 0.82 iteration (trace)
            gbs = per_it * (float(iters.sum()) + 0.82 * K) / (st["ms_solve"] * 1e-3) / 1e9
            dram = {"actual_dram_gbs_est": gbs, "actual_dram_frac_est": gbs / peak,
                    "actual_bytes_per_iter_ncu": per_it, "algorithmic_bytes_per_iter": per_iter}
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K, "warmup": W,
        "ms_per_step": ms_max / K, "higher_is_better": True, "scaling": "strong" if sharded else "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"BASELINE {workload_name(cfg_all.name)} ({cfg_all.name}): {cfg_all.description}",
                   "n_dof": N, "n_scenarios": cfg_all.n_scen, "nnz_volume": Z, "dt": cfg.dt, "rtol": 1e-12,
                   "l2": f"inputs > L2 ({per_iter / 1e9:.2f} GB algorithmic per CG iteration)" if per_iter > 126e6
                         else "working set fits L2 (no flush; small config)",
                   "parallelism": (f"scenarios sharded over {world} ranks" if sharded else
                                   "replicas only" if world > 1 else "single GPU"),
                   "cg_iters_per_step": float(iters.mean())},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": traffic,
                     "kernel": ("k_cg_step (persistent Jacobi-PCG, one launch per step)" if S == 1 else
                                "k_sbcg_step (persistent batched Jacobi-PCG, windowed SpMM over column groups "
                                "of 16 scenarios, one launch per step)" if st.get("solve_kind") == 3 else
                                "k_cgb_step (persistent batched Jacobi-PCG over all scenarios, one launch per step)"),
                     "peak_kind": peak_kind, "achieved_vs_8TBs": achieved / 8000.0,
                     "solve_share_of_step": st["ms_solve"] / ms,
                     "iface_share_of_step": st["ms_iface"] / ms, **dram},
        "e2e": {"value": units * KE / (ms_e2e * 1e-3), "unit": UNIT, "cg_iters_per_step": e2e_iters / KE,
                "h2d_bytes_per_step": 32 * S,
                "d2h_bytes_per_step": 8 * N * S},
        "gpu_launches": K * st["launches_per_step"],
        "clocks": clk.summary(),
    }
    th.close()
    if not args.no_cpu_baseline and world == 1:
        cb = cpu_baseline(cfg, 1)
        line["cpu_baseline"] = {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample", "cpu_model", "nproc")}
    print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.barrier()
        torch.distributed.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_thermo(args)


if __name__ == "__main__":
    main()
