"""Helpers for the GPU parity tests: scatter a global numpy array into the
per-rank device blocks of a plan layout and gather them back (the role of
scatter_global / gather_global, dist_tensor.hpp:105-175)."""
import numpy as np
import torch

import paper_1506_07933_b200 as D


def scatter(dist, global_arr, device="cuda"):
    blocks = []
    for r in range(dist.grid.size()):
        ext = dist.extents_of(r)
        sl = tuple(slice(o, o + n) for o, n in ext)
        blk = np.ascontiguousarray(global_arr[sl])
        t = torch.from_numpy(blk.reshape(-1).copy()).to(device)
        blocks.append(D.DistTensor(dist, r, t))
    return blocks


def gather(dist, tensors, dtype=None):
    arr = None
    for r, t in enumerate(tensors):
        ext = dist.extents_of(r)
        blk = t.data.cpu().numpy()
        if arr is None:
            arr = np.zeros(dist.dims, dtype=dtype or blk.dtype)
        sl = tuple(slice(o, o + n) for o, n in ext)
        arr[sl] = blk.reshape(tuple(n for _, n in ext))
    return arr


def run_world(plan, global_in, device="cuda"):
    ctxs = D.make_world_contexts(plan, device)
    xs = scatter(plan.input, global_in, device)
    ys = D.execute_world(plan, xs, ctxs)
    torch.cuda.synchronize()
    out = gather(plan.output, ys)
    for c in ctxs:
        c.close()
    return out


def make_plan(decomp, dims, grid, kind, direction, prec="f64", **opts):
    o = D.PlanOptions(**opts) if opts else None
    k = {"c2c": D.TransformKind.C2C, "r2c": D.TransformKind.R2C, "c2r": D.TransformKind.C2R}[kind]
    d = D.Direction.Forward if direction == "forward" else D.Direction.Backward
    if decomp == "slab":
        return D.plan_slab(dims, grid[0], k, d, o, prec)
    if decomp == "pencil":
        return D.plan_pencil(dims, grid, k, d, o, prec)
    return D.plan_general(dims, grid, k, d, o, prec)


def rel_l2(got, want):
    got = np.asarray(got, dtype=np.complex128).ravel()
    want = np.asarray(want, dtype=np.complex128).ravel()
    den = np.sum(np.abs(want) ** 2)
    num = np.sum(np.abs(got - want) ** 2)
    return float(np.sqrt(num) if den == 0 else np.sqrt(num / den))


def is_pow2(n):
    return n >= 1 and (n & (n - 1)) == 0
