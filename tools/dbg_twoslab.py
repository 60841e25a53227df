import sys
sys.path.insert(0, ".")
import numpy as np
from paper_1707_03581_b200 import inputs as I
from paper_1707_03581_b200.thermo import Thermo
mode = sys.argv[1]
sc = tuple(int(x) for x in sys.argv[2].split(","))
jit = float(sys.argv[3])
f, m = I.two_slab_pair(stock_cells=sc, jitter=jit)
robin = [I.Robin(0, I.TAG_FLOOR, 50.0, 24.0), I.Robin(1, I.TAG_COOL, 200.0, 18.0)]
th = Thermo(f, m, 50.0, 3.6e6, 1000.0, [I.Scenario(0.0, 0.0, 1.0, 500.0)], 24.0, (4, 4), robin)
print("N", th.n, "n_if", th.stats()["n_iface_rows"], flush=True)
if mode == "ie":
    th.step(0.0, 1.0, 3)
elif mode == "stat0":
    th.stationary(0.0, False)
else:
    th.stationary(0.0, True)
print(mode, "ok", th.get_T()[:4], th.stats()["max_iters"], flush=True)
