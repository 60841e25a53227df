"""Reproducer for the rare deviation of the windowed-SpMM batched kernel.

Runs configs[4] (64 scenarios) with the x0 = T^n start at rtol 2e-13 for NSTEPS steps in calls
of BLOCK steps, R times, each time after a throw-away context has left its freed device memory
behind; compares every block's state with the gather kernel's (deterministic) run and prints the
first block / column group that deviates.

    python tools/diag_spmm_race.py [R] [NSTEPS] [BLOCK]
"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_1707_03581_b200 import inputs as I  # noqa: E402
import paper_1707_03581_b200.thermo as _T  # noqa: E402
from paper_1707_03581_b200.thermo import Thermo  # noqa: E402

if os.environ.get("DIAG_LIB"):   # another build of libthermo.so (A/B on one box)
    _T.load(os.environ["DIAG_LIB"])

R = int(sys.argv[1]) if len(sys.argv) > 1 else 4
NSTEPS = int(sys.argv[2]) if len(sys.argv) > 2 else 500
BLOCK = int(sys.argv[3]) if len(sys.argv) > 3 else 25
cfg = I.make_config("cfg4")
S = cfg.n_scen


def make(kind):
    os.environ["THERMO_CGB"] = str(kind)
    th = Thermo.from_config(cfg)
    th.set_guess(0)
    th.set_solver(rtol=2e-13)
    return th


def run(th):
    snaps, its = [], []
    t = 0.0
    for b in range(NSTEPS // BLOCK):
        th.step(t, cfg.dt, BLOCK)
        t += BLOCK * cfg.dt
        snaps.append(np.stack([th.get_T(scen=k) for k in range(S)]))
        its.append(th.step_iters().reshape(BLOCK, S).copy())
    return snaps, its


t0 = time.time()
ref = make(1)
assert ref.stats()["solve_kind"] != 3
ref_snaps, ref_its = run(ref)
ref.close()
print(f"gather kernel reference: {time.time() - t0:.1f} s", flush=True)
for rep in range(R):
    junk = make(1)   # leaves garbage in the memory the next context allocates
    junk.step(0.0, cfg.dt, 2)
    junk.close()
    th = make(2)
    assert th.stats()["solve_kind"] == 3, "windowed SpMM kernel not selected"
    snaps, its = run(th)
    th.close()
    worst, first = 0.0, None
    for b, (a, r) in enumerate(zip(snaps, ref_snaps)):
        d = np.abs(a - r).max(axis=1) / np.abs(r).max()
        worst = max(worst, float(d.max()))
        if first is None and d.max() > 1e-11:
            groups = sorted(set((np.flatnonzero(d > 1e-11) // 16).tolist()))
            itd = np.flatnonzero((its[b] != ref_its[b]).any(axis=1))
            first = (b, float(d.max()), int(d.argmax()), groups, itd.tolist()[:8])
            k = int(d.argmax())
            e = np.abs(a[k] - r[k])
            top = np.argsort(e)[::-1][:6]
            nf = cfg.fixed.n_nodes
            desc = []
            for i in top:
                if i < nf:
                    nx, ny = 129, 33
                    desc.append(f"F{i}({i % nx},{i // nx % ny},{i // (nx * ny)}) {e[i]:.1e}")
                else:
                    j = i - nf
                    desc.append(f"M{j}({j % 41},{j // 41 % 25},{j // (41 * 25)}) {e[i]:.1e}")
            print(f"   block {b} scen {k}: rows > 0.1 max {int((e > 0.1 * e.max()).sum())}, > 1e-3 max "
                  f"{int((e > 1e-3 * e.max()).sum())}; top: {'; '.join(desc)}", flush=True)
            dg = d[(k // 16) * 16:(k // 16 + 1) * 16]
            print("   group deviations: " + " ".join(f"{x:.1e}" for x in dg), flush=True)
    print(f"rep {rep}: max rel deviation {worst:.2e}; first block > 1e-11: {first}", flush=True)
