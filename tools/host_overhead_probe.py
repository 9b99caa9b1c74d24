import time, sys, os
sys.path.insert(0, os.getcwd())
import torch
import paper_1506_07933_b200 as D
fwd = D.plan_slab((64, 64, 64), 1, D.TransformKind.C2C, D.Direction.Forward)
bwd = D.plan_slab((64, 64, 64), 1, D.TransformKind.C2C, D.Direction.Backward)
ctx = D.make_context(fwd)
x = D.DistTensor.seeded(fwd.input, 0)
y = D.DistTensor.zeros(fwd.output, 0)
z = D.DistTensor.zeros(bwd.output, 0)
for _ in range(10):
    D.execute(fwd, x, ctx, out=y, sync=False); D.execute(bwd, y, ctx, out=z, sync=False)
torch.cuda.synchronize()
N = 2000
t0 = time.perf_counter()
for _ in range(N):
    D.execute(fwd, x, ctx, out=y, sync=False); D.execute(bwd, y, ctx, out=z, sync=False)
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"host per fwd+inv {1e6*(t1-t0)/N:.1f} us; wall incl. drain {1e6*(t2-t0)/N:.1f} us")
# device time: events around a burst launched while the GPU is kept busy (queue full)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda._sleep(200_000_000)  # ~0.1 s of GPU spin so the launches queue up
e0.record()
for _ in range(200):
    D.execute(fwd, x, ctx, out=y, sync=False); D.execute(bwd, y, ctx, out=z, sync=False)
e1.record()
torch.cuda.synchronize()
print(f"device per fwd+inv (queued) {1e3*e0.elapsed_time(e1)/200:.1f} us")
import cProfile, pstats
pr = cProfile.Profile(); pr.enable()
for _ in range(500):
    D.execute(fwd, x, ctx, out=y, sync=False)
pr.disable()
torch.cuda.synchronize()
pstats.Stats(pr).sort_stats("tottime").print_stats(8)
