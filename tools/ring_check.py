"""Debug aid: one forward (and backward) with and without the L2 ring
(DFFTB_RING), compared bitwise.  python tools/ring_check.py [n]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1506_07933_b200 as D  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
dims = (n, n, n)
fwd = D.plan_pencil(dims, (1, 1), D.TransformKind.C2C, D.Direction.Forward)
bwd = D.plan_pencil(dims, (1, 1), D.TransformKind.C2C, D.Direction.Backward)
ctx = D.make_context(fwd)
x = D.DistTensor.seeded(fwd.input, 0)
os.environ["DFFTB_RING"] = "0"
y0 = D.execute(fwd, x, ctx)
z0 = D.execute(bwd, y0, ctx)
torch.cuda.synchronize()
os.environ["DFFTB_RING"] = "1"
os.environ["DFFTB_OP_TIMES"] = "1"
tb = D.TimingBreakdown()
y1 = D.execute(fwd, x, ctx, timers=tb)
print("fwd equal:", bool(torch.equal(y0.data, y1.data)), flush=True)
z1 = D.execute(bwd, y0, ctx, timers=tb)
print("bwd equal:", bool(torch.equal(z0.data, z1.data)), flush=True)
