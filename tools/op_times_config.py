"""Per-op device times (ExecContext.last_ops) of one fwd+inv of a
configuration on one GPU:
python tools/op_times_config.py 256,256,256 r2c f64 slab"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1506_07933_b200 as D  # noqa: E402

dims = tuple(int(v) for v in sys.argv[1].split(","))
kind, prec, decomp = sys.argv[2], sys.argv[3], sys.argv[4]
kf = D.TransformKind.R2C if kind == "r2c" else D.TransformKind.C2C
kb = D.TransformKind.C2R if kind == "r2c" else D.TransformKind.C2C
if decomp == "slab":
    fwd = D.plan_slab(dims, 1, kf, D.Direction.Forward, precision=prec)
    bwd = D.plan_slab(dims, 1, kb, D.Direction.Backward, precision=prec)
else:
    fwd = D.plan_pencil(dims, (1, 1), kf, D.Direction.Forward, precision=prec)
    bwd = D.plan_pencil(dims, (1, 1), kb, D.Direction.Backward, precision=prec)
ctx = D.make_context(fwd)
x = D.DistTensor.seeded(fwd.input, 0, complex_field=kind == "c2c")
for _ in range(3):
    y = D.execute(fwd, x, ctx)
    z = D.execute(bwd, y, ctx)
torch.cuda.synchronize()
for name in ("fwd", "bwd"):
    tb = D.TimingBreakdown()
    if name == "fwd":
        y = D.execute(fwd, x, ctx, timers=tb)
    else:
        z = D.execute(bwd, y, ctx, timers=tb)
    print(f"{name} total {tb.total * 1e3:.3f} ms")
    for kind, stream, n, share, start, ms in ctx.last_ops():
        print(f"  {kind:8s} n={n:5d} share {share:.3f} at {start:.3f}: {ms:.3f} ms")
