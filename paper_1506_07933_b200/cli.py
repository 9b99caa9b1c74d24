"""dfftb-bench: the reference's dfft-bench driver (tools/dfft_bench.cpp,
bench.cpp:261-362) on the B200 path, emitting the same JSON / CSV report
(schema_version 1, report_schema.golden) and honouring --input/--output DTNS
tensors.

    python -m paper_1506_07933_b200.cli --dims 64,64,64 [--grid 2,2 | --np 4]
        [--kind c2c|r2c|c2r] [--decomp slab|pencil|general] [--reps 3]
        [--warmup 1] [--seed 1] [--verify auto|on|off] [--format json|csv]
        [--out PATH] [--input IN.dtns] [--output OUT.dtns]

Multi-rank runs are one process per GPU under torchrun.  Verification is the
reference's: relative L2 against a direct multi-dimensional DFT of the
gathered input (computed on device in double by per-axis DFT matrices), auto
for N <= 2^16 (kernels.hpp:392, bench.cpp:273).  Exit codes as dfft_bench.cpp:
0 ok, 2 verification failed, 1 error.
"""
import argparse
import math
import os
import sys
import time

import numpy as np
import torch

from . import dfft as D
from . import io as IO

ORACLE_GUARD = 1 << 16


def auto_grid(ranks, axes):
    """bench.cpp:60-78: most-square factorization, non-increasing factors."""
    shape, rem = [], ranks
    for a in range(axes, 1, -1):
        root = rem ** (1.0 / a)
        best = 1
        for f in range(1, int(root + 1e-9) + 1):
            if rem % f == 0:
                best = f
        shape.append(best)
        rem //= best
    shape.append(rem)
    return sorted(shape, reverse=True)


def direct_dft(x: torch.Tensor, inverse=False) -> torch.Tensor:
    """Multi-dimensional DFT by per-axis DFT matrices, in complex128 on device."""
    y = x.to(torch.complex128)
    for a, n in enumerate(y.shape):
        k = torch.arange(n, device=y.device, dtype=torch.float64)
        sign = 1.0 if inverse else -1.0
        F = torch.polar(torch.ones(n, n, device=y.device, dtype=torch.float64),
                        sign * 2 * math.pi * torch.outer(k, k).remainder(n) / n)
        y = torch.tensordot(y, F, dims=([a], [0])).movedim(-1, a)
    return y


def main(argv=None):
    ap = argparse.ArgumentParser(prog="dfftb-bench")
    ap.add_argument("--dims", required=True)
    ap.add_argument("--grid")
    ap.add_argument("--np", type=int)
    ap.add_argument("--kind", default="c2c", choices=["c2c", "r2c", "c2r"])
    ap.add_argument("--decomp", default="pencil", choices=["slab", "pencil", "general"])
    ap.add_argument("--pipelined", default="false")
    ap.add_argument("--chunks", type=int, default=1)
    ap.add_argument("--staging-buffers", type=int, default=2)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=1)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--verify", default="auto", choices=["auto", "on", "off"])
    ap.add_argument("--format", default="json", choices=["json", "csv"])
    ap.add_argument("--precision", default="f64", choices=["f64", "f32"])
    ap.add_argument("--out")
    ap.add_argument("--input")
    ap.add_argument("--output")
    a = ap.parse_args(argv)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    comm = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        comm = dist.group.WORLD
    dims = [int(x) for x in a.dims.split(",")]
    axes = 1 if a.decomp == "slab" else (2 if a.decomp == "pencil" else len(dims) - 1)
    grid = [int(x) for x in a.grid.split(",")] if a.grid else auto_grid(a.np or world, axes)
    if int(np.prod(grid)) != world:
        raise SystemExit(f"grid {grid} needs {int(np.prod(grid))} ranks, launched {world}")
    opts = D.PlanOptions(exchange=D.ExchangePath.Pipelined if a.pipelined == "true"
                         else D.ExchangePath.Blocking, chunks_per_peer=a.chunks,
                         staging_buffers=a.staging_buffers)
    kind = {"c2c": D.TransformKind.C2C, "r2c": D.TransformKind.R2C, "c2r": D.TransformKind.C2R}[a.kind]
    direction = D.Direction.Backward if a.kind == "c2r" else D.Direction.Forward
    mk = {"slab": lambda: D.plan_slab(dims, grid[0], kind, direction, opts, a.precision),
          "pencil": lambda: D.plan_pencil(dims, grid, kind, direction, opts, a.precision),
          "general": lambda: D.plan_general(dims, grid, kind, direction, opts, a.precision)}
    plan = mk[a.decomp]()
    ctx = D.make_context(plan, comm)
    warnings = list(plan.warnings)

    # input: DTNS file, or the seeded field (C2R: spectrum of a real seeded field)
    if a.input:
        x = IO.read_tensor(plan.input, rank, a.input)
    elif a.kind == "c2r":
        fplan = (D.plan_slab(dims, grid[0], D.TransformKind.R2C, D.Direction.Forward, None, a.precision)
                 if a.decomp == "slab" else
                 D.plan_pencil(dims, grid, D.TransformKind.R2C, D.Direction.Forward, None, a.precision)
                 if a.decomp == "pencil" else
                 D.plan_general(dims, grid, D.TransformKind.R2C, D.Direction.Forward, None, a.precision))
        field = D.DistTensor.seeded(fplan.input, rank, a.seed, complex_field=False)
        x = D.execute(fplan, field, ctx)
    else:
        x = D.DistTensor.seeded(plan.input, rank, a.seed, complex_field=a.kind == "c2c")

    for _ in range(a.warmup):
        D.execute(plan, x, ctx)
    reps = []
    y = None
    for _ in range(a.reps):
        if comm is not None:
            torch.distributed.barrier(comm)
        tb = D.TimingBreakdown()
        y = D.execute(plan, x, ctx, timers=tb)
        t = torch.tensor([tb.local_fft, tb.pack, tb.unpack, tb.staging_copy, tb.wire_comm, tb.total],
                         dtype=torch.float64, device="cuda")
        if comm is not None:
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX, group=comm)
        reps.append(dict(zip(IO.TIMING_KEYS, t.tolist())))

    def gather(dt):
        blocks = [None] * world
        if comm is not None:
            torch.distributed.all_gather_object(blocks, (dt.rank, dt.data.cpu()), group=comm)
        else:
            blocks = [(dt.rank, dt.data.cpu())]
        return [D.DistTensor(dt.dist, r, d) for r, d in blocks]

    if a.output:
        ys = gather(y)
        if rank == 0:
            IO.write_tensor(a.output, ys)

    total = int(np.prod(dims))
    do_verify = a.verify == "on" or (a.verify == "auto" and total <= ORACLE_GUARD)
    rel = None
    if do_verify:
        xs, ys = gather(x), gather(y)
        if rank == 0:
            def full(blocks):
                dist = blocks[0].dist
                arr = None
                for b in blocks:
                    e = dist.extents_of(b.rank)
                    blk = b.data.numpy().reshape(tuple(n for _, n in e))
                    if arr is None:
                        arr = np.zeros(dist.dims, dtype=blk.dtype)
                    arr[tuple(slice(o, o + n) for o, n in e)] = blk
                return arr
            xin, yout = full(xs), full(ys)
            if a.kind == "c2r":
                # Hermitian-extend the half spectrum, inverse DFT, 1/N (bench.cpp:188-231)
                full_spec = np.zeros(dims, np.complex128)
                nh = dims[-1] // 2 + 1
                full_spec[..., :nh] = xin
                lead = [(-np.arange(n)) % n for n in dims[:-1]]
                mirrored = xin[np.ix_(*lead, np.arange(nh))]  # X[-i0, ..., k]
                for k in range(nh, dims[-1]):
                    full_spec[..., k] = np.conj(mirrored[..., dims[-1] - k])
                want = direct_dft(torch.from_numpy(full_spec).cuda(), inverse=True).real.cpu().numpy() / total
                got = yout
            else:
                want = direct_dft(torch.from_numpy(xin.astype(np.complex128)).cuda()).cpu().numpy()
                if a.kind == "r2c":
                    want = want[..., : dims[-1] // 2 + 1]
                got = yout
            num = float(np.sum(np.abs(got - want) ** 2))
            den = float(np.sum(np.abs(want) ** 2))
            rel = math.sqrt(num) if den == 0 else math.sqrt(num / den)
    elif a.verify == "auto":
        warnings.append("verification skipped: problem exceeds the oracle guard")

    code = 0
    if rank == 0:
        cfg = {"dims": dims, "grid": grid, "kind": a.kind, "decomp": a.decomp, "backend": "b200",
               "pipelined": a.pipelined == "true", "chunks": a.chunks,
               "staging_buffers": a.staging_buffers, "reps": a.reps, "warmup": a.warmup,
               "seed": a.seed}
        text = IO.to_json(cfg, reps, rel, warnings) if a.format == "json" else IO.to_csv(reps)
        if a.out:
            with open(a.out, "w") as f:
                f.write(text)
        else:
            sys.stdout.write(text)
        for w in warnings:
            print(f"warning: {w}", file=sys.stderr)
        if rel is not None and rel > 1e-10 and a.precision == "f64":
            print(f"verification FAILED (rel error {rel})", file=sys.stderr)
            code = 2
    ctx.close()
    if comm is not None:
        torch.distributed.destroy_process_group()
    return code


if __name__ == "__main__":
    sys.exit(main())
