"""Time every BASELINE.json configuration on the GPUs of this launch
(python tools/bench_configs.py, or under torchrun for N > 1).  Prints one
line per config: fwd+inv ms, GFLOP/s (5 N log2 N x 2), step roofline
fraction, round-trip rel-L2.  Informational; bench.py is the contract."""
import json
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_1506_07933_b200 as D  # noqa: E402


def configs(N):
    g2 = (2, N // 2) if N > 1 else (1, 1)
    cfg = [
        ("A 64^3 C2C f64 slab", (64, 64, 64), "slab", (N,), "c2c", "f64"),
        ("B 256^3 R2C f64 slab", (256, 256, 256), "slab", (N,), "r2c", "f64"),
        ("C 512^3 C2C f64 pencil", (512, 512, 512), "pencil", g2, "c2c", "f64"),
        ("D 1024^3 C2C f64 pencil", (1024, 1024, 1024), "pencil",
         (4, 2) if N == 8 else g2, "c2c", "f64"),
        ("E 2048x512x256 R2C f32 pencil", (2048, 512, 256), "pencil", g2, "r2c", "f32"),
    ]
    if N == 1:
        cfg = [c for c in cfg]
    return cfg


def main():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    K = int(os.environ.get("STEPS", "10"))
    only = os.environ.get("ONLY")
    for name, dims, decomp, grid, kind, prec in configs(world):
        if only and not name.startswith(only):
            continue
        kf = D.TransformKind.R2C if kind == "r2c" else D.TransformKind.C2C
        kb = D.TransformKind.C2R if kind == "r2c" else D.TransformKind.C2C
        mk = D.plan_slab if decomp == "slab" else D.plan_pencil
        g = grid[0] if decomp == "slab" else grid
        fwd = mk(dims, g, kf, D.Direction.Forward, precision=prec)
        bwd = mk(dims, g, kb, D.Direction.Backward, precision=prec)
        ctx = D.make_context(fwd)
        x = D.DistTensor.seeded(fwd.input, rank, complex_field=kind == "c2c")
        y = D.DistTensor.zeros(fwd.output, rank)
        z = D.DistTensor.zeros(bwd.output, rank)

        def step():
            D.execute(fwd, x, ctx, out=y, sync=False)
            D.execute(bwd, y, ctx, out=z, sync=False)

        for _ in range(3):
            step()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(K):
            step()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / K
        num = (torch.linalg.vector_norm(z.data - x.data) ** 2).item()
        den = (torch.linalg.vector_norm(x.data) ** 2).item()
        if world > 1:
            t = torch.tensor([ms, num, den], dtype=torch.float64, device="cuda")
            dist.all_reduce(t[:1], op=dist.ReduceOp.MAX)
            dist.all_reduce(t[1:])
            ms, num, den = t.tolist()
        n = math.prod(dims)
        flops = 2 * 5 * n * math.log2(n)
        if rank == 0:
            print(json.dumps({"config": name, "gpus": world, "grid": list(grid), "ms_fwdinv": round(ms, 4),
                              "gflops": round(flops / ms / 1e6, 1),
                              "roundtrip_rel_l2": math.sqrt(num / den)}), flush=True)
        ctx.close()
        del x, y, z
        torch.cuda.empty_cache()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
