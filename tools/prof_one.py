"""Short single-GPU workload for ncu: W warm-up fwd+inv steps then one
profiled-region fwd+inv of 512^3 C2C fp64 (pencil 1x1).  Not a benchmark."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1506_07933_b200 as D  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--dims", default="512,512,512")
ap.add_argument("--kind", default="c2c")
ap.add_argument("--prec", default="f64")
ap.add_argument("--warmup", type=int, default=1)
ap.add_argument("--steps", type=int, default=1)
a = ap.parse_args()
dims = tuple(int(x) for x in a.dims.split(","))
kf = D.TransformKind.R2C if a.kind == "r2c" else D.TransformKind.C2C
kb = D.TransformKind.C2R if a.kind == "r2c" else D.TransformKind.C2C
fwd = D.plan_pencil(dims, (1, 1), kf, D.Direction.Forward, precision=a.prec)
bwd = D.plan_pencil(dims, (1, 1), kb, D.Direction.Backward, precision=a.prec)
ctx = D.make_context(fwd)
x = D.DistTensor.seeded(fwd.input, 0, complex_field=a.kind == "c2c")
y = D.DistTensor.zeros(fwd.output, 0)
z = D.DistTensor.zeros(bwd.output, 0)
for _ in range(a.warmup + a.steps):
    D.execute(fwd, x, ctx, out=y, sync=False)
    D.execute(bwd, y, ctx, out=z, sync=False)
torch.cuda.synchronize()
ctx.check()
print("ok", D.kernel_launch_count())
