"""Debug aid: run a set of small configs through the emulated world and print
rel-L2 errors against the oracle (set DFFTB_NO_TMA=1 to force the direct
kernels).  Not part of the test suite."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import oracle_lib as O  # noqa: E402
from gpu_util import make_plan, rel_l2, run_world  # noqa: E402

CFGS = [
    ("slab", [16, 16, 16], [1], "r2c", "f64"),
    ("slab", [16, 16, 16], [1], "r2c", "f32"),
    ("slab", [16, 16, 16], [2], "r2c", "f64"),
    ("slab", [8, 8, 16], [8], "r2c", "f64"),
    ("pencil", [32, 16, 8], [2, 2], "r2c", "f64"),
    ("slab", [32, 32, 32], [1], "r2c", "f64"),
    ("slab", [32, 32, 32], [1], "c2c", "f64"),
]
for decomp, dims, grid, kind, prec in CFGS:
    x = O.seeded(dims, kind == "c2c", prec)
    y_ref, _ = O.execute(x, dims, decomp, grid, kind, "forward", prec)
    y = run_world(make_plan(decomp, dims, grid, kind, "forward", prec), x)
    bk = "c2r" if kind == "r2c" else "c2c"
    try:
        z = run_world(make_plan(decomp, dims, grid, bk, "backward", prec), y_ref)
        ez = rel_l2(z, x)
    except Exception as e:  # noqa: BLE001
        ez = str(e)[:220]
    print(decomp, dims, grid, kind, prec, "fwd", rel_l2(y, y_ref), "bwd", ez, flush=True)
