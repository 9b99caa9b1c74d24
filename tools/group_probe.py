"""Exchange-group-size probe (not a benchmark): 512^3 C2C fp64 fwd+inv on
the GPUs of this torchrun launch with a slab grid (one group of N) and a
pencil 1 x N grid, so the staged exchange runs with N-1 peers per DMA
chunk, as the 4-member groups of the 8-GPU 2x4 grid do.  Prints ms per
fwd+inv (max over ranks); compare DFFTB_DMA=0 (direct peer stores)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_1506_07933_b200 as D  # noqa: E402


def main():
    world = int(os.environ["WORLD_SIZE"])
    rank = int(os.environ["RANK"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dims = (512, 512, 512)
    for name, mk in (("slab", lambda d: D.plan_slab(dims, world, D.TransformKind.C2C, d)),
                     ("pencil 1x%d" % world, lambda d: D.plan_pencil(dims, (1, world), D.TransformKind.C2C, d))):
        fwd, bwd = mk(D.Direction.Forward), mk(D.Direction.Backward)
        ctx = D.make_context(fwd)
        x = D.DistTensor.seeded(fwd.input, rank)
        y = D.DistTensor.zeros(fwd.output, rank)
        z = D.DistTensor.zeros(bwd.output, rank)
        for _ in range(3):
            D.execute(fwd, x, ctx, out=y, sync=False)
            D.execute(bwd, y, ctx, out=z, sync=False)
        torch.cuda.synchronize()
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            D.execute(fwd, x, ctx, out=y, sync=False)
            D.execute(bwd, y, ctx, out=z, sync=False)
        e1.record()
        torch.cuda.synchronize()
        t = torch.tensor([e0.elapsed_time(e1) / 10], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        err = (torch.linalg.vector_norm(z.data - x.data) / torch.linalg.vector_norm(x.data)).item()
        kinds = set()
        D.execute(fwd, x, ctx, out=y, timers=D.TimingBreakdown())
        kinds |= {o[0] for o in ctx.last_ops()}
        if rank == 0:
            print(f"{name}: {t.item():.3f} ms per fwd+inv, round trip {err:.1e}, "
                  f"{'staged' if 'copy' in kinds else 'direct'} exchange", flush=True)
        ctx.close()
        dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
