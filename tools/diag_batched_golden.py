import os, sys
import numpy as np
sys.path.insert(0, ".")
sys.path.insert(0, "tests")
from paper_1707_03581_b200 import inputs as I
from paper_1707_03581_b200.thermo import Thermo
import golden_codec as G, json
cfg = I.make_config("cfg4")
g = np.load("tests/golden/fullrun_cfg4.npz"); meta = json.loads(str(g["meta"]))
ref = G.unpack_field(g["field"], 64 * cfg.n_dof).reshape(64, cfg.n_dof)
res = {}
for mode, chunk in (("0", 500), ("0", 25), ("1", 500), ("0", 100), ("0", 250)):
    os.environ["THERMO_CGB"] = "2" if mode == "0" else "1"
    th = Thermo.from_config(cfg)
    for b in range(500 // chunk): th.step(b * chunk * cfg.dt, cfg.dt, chunk)
    T = np.stack([th.get_T(scen=k) for k in range(64)])
    e = np.abs(T - ref).max(axis=1) / np.abs(ref).max(axis=1)
    print(f"kernel {mode} calls of {chunk}: worst vs oracle {e.max():.2e} (scen {e.argmax()}), scen48 {e[48]:.2e}", flush=True)
