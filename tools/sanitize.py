"""Small runs of every CUDA path for compute-sanitizer (memcheck / synccheck / racecheck):

    compute-sanitizer --tool memcheck python tools/sanitize.py

implicit Euler on cfg 0 and the 'small' mesh (fused and two-phase CG kernels, serial and overlapped
interface, extrapolated start), the batched kernel (3 scenarios), MRSDC(3,2), single-rate SDC and
the stationary solve.  Prints one line per case; the sanitizer reports errors itself."""
import os
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_1707_03581_b200 import inputs as I  # noqa: E402
from paper_1707_03581_b200.thermo import Thermo  # noqa: E402


def case(name, env, fn):
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        T = fn()
        print(f"{name}: ok, T range [{T.min():.6f}, {T.max():.6f}]", flush=True)
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


def ie(cfg_name, steps=4, **kw):
    def run():
        cfg = I.make_config(cfg_name, **kw)
        th = Thermo.from_config(cfg)
        th.step(0.0, cfg.dt, steps)
        T = th.get_T()
        th.close()
        return T
    return run


def batched():
    cfg = I.make_config("cfg0")
    sc = [I.Scenario(0.375, 0.375, 20.0 + k, 100.0 + 15.0 * k) for k in range(3)]
    th = Thermo.from_config(cfg, scenarios=sc)
    th.step(0.0, 1.0, 3)
    T = th.get_T(scen=2)
    th.close()
    return T


def sdc(method):
    def run():
        cfg = I.make_config("cfg0")
        th = Thermo.from_config(cfg)
        th.set_method(method, 3, 2, 1)
        th.step(0.0, 1.0, 2)
        T = th.get_T()
        th.close()
        return T
    return run


def stationary():
    cfg = I.make_config("cfg0")
    th = Thermo.from_config(cfg)
    th.stationary(0.0, with_interface=True)
    T = th.get_T()
    th.close()
    return T


case("ie cfg0 default (fused, overlap)", {}, ie("cfg0"))
case("ie cfg0 two-phase, serial", {"THERMO_CG_VARIANT": "2", "THERMO_OVERLAP": "0"}, ie("cfg0"))
case("ie small jittered default", {}, ie("small", jitter=0.1))
case("ie small two-phase W6", {"THERMO_CG_VARIANT": "4", "THERMO_OVERLAP": "0"}, ie("small", jitter=0.1))
case("ie small KIND 0", {"THERMO_CG_VARIANT": "0", "THERMO_OVERLAP": "0"}, ie("small", jitter=0.1))
case("ie small NG=2 3-stage cap", {"THERMO_CG_VARIANT": "3", "THERMO_CG_STAGES": "3", "THERMO_OVERLAP": "0"},
     ie("small", jitter=0.1))
case("batched 3 scenarios", {}, batched)
case("mrsdc(3,2) k=1", {}, sdc("mrsdc"))
case("sdc(3) k=1", {}, sdc("sdc"))
case("stationary coupled", {}, stationary)
print("sanitize runs done", flush=True)
