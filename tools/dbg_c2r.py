import os, sys
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import numpy as np, torch
import oracle_lib as O
import paper_1506_07933_b200 as D
from gpu_util import make_plan, rel_l2, run_world
for dims in ([1, 16], [4, 16], [2, 16, 16], [16, 16, 16], [1, 8], [1, 32], [1, 64]):
    x = O.seeded(dims, False, "f64")
    y, _ = O.execute(x, dims, "slab", [1], "r2c", "forward", "f64")
    hy = np.abs(y.reshape(-1, y.shape[-1]))
    try:
        z = run_world(make_plan("slab", dims, [1], "c2r", "backward", "f64"), y)
        print(dims, "ok", rel_l2(z, x))
    except D.Error as e:
        print(dims, str(e)[60:], "true max", hy.max(), "true dc imag", np.abs(y.reshape(-1, y.shape[-1])[:, [0, -1]].imag).max())
