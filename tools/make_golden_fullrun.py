"""Write full-run oracle references for the stand-scale configurations (BASELINE.json
configs[2] and configs[3]) under tests/golden/.  Calls only the CPU oracle (oracle/), never
the CUDA path: the stored values are the oracle's temperatures after the configured number of
implicit-Euler steps from the uniform start T0, sampled at a fixed seeded set of DoF (every
interface row plus a uniform sample) -- the GPU full run is compared against them in
tests/test_gpu_fullrun.py.

    python tools/make_golden_fullrun.py cfg2 [nsteps]      (~1.7 h single thread)
    python tools/make_golden_fullrun.py cfg3 [nsteps]      (~1.5 h)
    python tools/make_golden_fullrun.py cfg4 [nsteps]      (scenarios 0, 37, 63 of the batch, whole fields)

GUESS=k in the environment selects the oracle's CG start (or_set_guess: 0 = T^n, 2 = quadratic
extrapolation, the CUDA path's default); k > 0 writes fullrun_<cfg>_g<k>.npz.
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle as O  # noqa: E402
from paper_1707_03581_b200 import inputs as I  # noqa: E402

GUESS = int(os.environ.get("GUESS", "0"))
SUFFIX = f"_g{GUESS}" if GUESS else ""
START = "x0 = T^n" if GUESS == 0 else f"x0 = extrapolation of order {GUESS} (or_set_guess)"


def sample_rows(cfg, n_uniform=20000, seed=1707):
    """Every node on an interface face of either part plus a seeded uniform sample."""
    nf = cfg.fixed.n_nodes
    rows = set()
    for mesh, off in ((cfg.fixed, 0), (cfg.moving, nf)):
        sel = mesh.bface_tag == cfg.iface_tag
        rows.update((mesh.bfaces[sel].ravel() + off).tolist())
    r = I.uniform01(seed, np.arange(n_uniform, dtype=np.int64), 0)
    rows.update((r * cfg.n_dof).astype(np.int64).tolist())
    return np.array(sorted(rows), dtype=np.int64)


def batched(cfg, nsteps, scen=(0, 37, 63)):
    """Config 4: independent oracle runs of sampled scenarios of the batch, whole fields."""
    t1 = time.time()
    vals, iters = [], 0
    for k in scen:
        o = O.Oracle.from_config(cfg, GUESS)   # fresh history per scenario
        T, st = o.step(np.full(o.n, cfg.T0), 0.0, cfg.dt, nsteps, cfg.scenarios[k])
        vals.append(T)
        iters += int(st[:, 0].sum())
        print(f"{cfg.name}: scenario {k} done, {time.time() - t1:.0f} s", flush=True)
    out = os.path.join(ROOT, "tests", "golden", f"fullrun_{cfg.name}{SUFFIX}.npz")
    meta = {"config": cfg.name, "nsteps": nsteps, "dt": cfg.dt, "t0": 0.0, "T0": cfg.T0, "n_dof": cfg.n_dof,
            "n_scen": cfg.n_scen, "scenarios": list(scen), "solver": f"oracle Jacobi-PCG, rtol 1e-12, {START}",
            "script": "tools/make_golden_fullrun.py", "oracle_seconds": time.time() - t1,
            "cg_iterations_total": iters}
    np.savez_compressed(out, scen=np.array(scen), values=np.stack(vals), meta=json.dumps(meta))
    print(json.dumps(meta))


def main():
    name = sys.argv[1]
    cfg = I.make_config(name)
    nsteps = int(sys.argv[2]) if len(sys.argv) > 2 else cfg.nsteps
    if cfg.n_scen > 1:
        return batched(cfg, nsteps)
    t0 = time.time()
    o = O.Oracle.from_config(cfg, GUESS)
    t1 = time.time()
    T = np.full(o.n, cfg.T0)
    sc = cfg.scenarios[0]
    iters = []
    chunk = 50
    done = 0
    while done < nsteps:
        k = min(chunk, nsteps - done)
        T, st = o.step(T, done * cfg.dt, cfg.dt, k, sc)
        iters.extend(st[:, 0].tolist())
        done += k
        print(f"{name}: {done}/{nsteps} steps, {time.time() - t1:.0f} s", flush=True)
    rows = sample_rows(cfg)
    out = os.path.join(ROOT, "tests", "golden", f"fullrun_{name}{SUFFIX}.npz")
    meta = {"config": name, "nsteps": nsteps, "dt": cfg.dt, "t0": 0.0, "T0": cfg.T0, "n_dof": cfg.n_dof,
            "solver": f"oracle Jacobi-PCG, rtol 1e-12, {START}", "script": "tools/make_golden_fullrun.py",
            "oracle_seconds": time.time() - t1, "create_seconds": t1 - t0,
            "cg_iterations_total": int(sum(iters)), "T_max": float(T.max()), "T_min": float(T.min()),
            "T_sum": float(T.sum())}
    np.savez_compressed(out, rows=rows, values=T[rows], meta=json.dumps(meta))
    print(json.dumps(meta))


if __name__ == "__main__":
    main()
