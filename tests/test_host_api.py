"""CPU-side checks of the C ABI and the host logic (no GPU needed):
exported symbols, plan/layout/local-size answers against the oracle (the
restated reference), exchange-count symmetry, error codes, and the
multi-process host path (handle all-gather, block tiling) on a gloo world."""
import os
import re
import socket

import numpy as np
import pytest

import oracle_lib as O
import paper_1506_07933_b200 as D
from paper_1506_07933_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_exports_every_declared_symbol():
    hdr = open(os.path.join(ROOT, "include", "dfftb", "dfftb.h")).read()
    declared = set(re.findall(r"\b(dfftb_[a-z_0-9]+)\s*\(", hdr))
    L = _lib.lib()
    missing = [s for s in declared if not hasattr(L, s)]
    assert not missing, missing
    assert declared <= set(_lib.exported_symbols()) | {"dfftb_plan_options_default"}


CONFIGS = [
    ([512, 512, 512], "pencil", [2, 4], "c2c"),
    ([1024, 1024, 1024], "pencil", [4, 2], "c2c"),
    ([256, 256, 256], "slab", [8], "r2c"),
    ([2048, 512, 256], "pencil", [4, 2], "r2c"),
    ([2048, 512, 256], "pencil", [2, 2], "r2c"),
    ([5, 5, 5], "pencil", [1, 4], "c2c"),
    ([17, 4, 4], "slab", [3], "c2c"),
    ([8, 4, 6], "pencil", [2, 2], "r2c"),
    ([8, 6, 4, 4], "general", [2, 2, 2], "c2c"),
]


def _kind(k):
    return {"c2c": D.TransformKind.C2C, "r2c": D.TransformKind.R2C,
            "c2r": D.TransformKind.C2R}[k]


def _plan(dims, decomp, grid, kind, direction):
    d = D.Direction.Forward if direction == "forward" else D.Direction.Backward
    if decomp == "slab":
        return D.plan_slab(dims, grid[0], _kind(kind), d)
    if decomp == "pencil":
        return D.plan_pencil(dims, grid, _kind(kind), d)
    return D.plan_general(dims, grid, _kind(kind), d)


@pytest.mark.parametrize("dims,decomp,grid,kind", CONFIGS)
def test_local_extents_and_signatures_match_oracle(dims, decomp, grid, kind):
    P = int(np.prod(grid))
    for direction, k in (("forward", kind), ("backward", "c2r" if kind == "r2c" else "c2c")):
        plan = _plan(dims, decomp, grid, k, direction)
        x = np.zeros(1)
        for side, dist in ((0, plan.input), (1, plan.output)):
            for r in range(P):
                off, ln = O.local_extents(dims, decomp, grid, k, direction, side, r)
                assert dist.extents_of(r) == list(zip(off, ln))
        # every rank's blocks tile the global tensor exactly once
        for dist in (plan.input, plan.output):
            cover = np.zeros(dist.dims, dtype=np.int32)
            for r in range(P):
                sl = tuple(slice(o, o + n) for o, n in dist.extents_of(r))
                cover[sl] += 1
            assert np.all(cover == 1)
        del x


@pytest.mark.parametrize("dims,decomp,grid,kind", CONFIGS[:6])
def test_exchange_counts_are_symmetric(dims, decomp, grid, kind):
    plan = _plan(dims, decomp, grid, kind, "forward")
    P = plan.nranks()
    g = D.ProcessGrid(grid)
    for t in range(plan.transpose_stage_count()):
        counts = [plan.exchange_counts(r, t) for r in range(P)]
        # which grid axis does transpose t move?  members share all coords but one
        for r in range(P):
            send, _ = counts[r]
            cr = g.coords_of(r)
            for gax in range(len(grid)):
                members = []
                for q in range(grid[gax]):
                    c = list(cr)
                    c[gax] = q
                    members.append(g.rank_of(c))
                if len(members) != len(send):
                    continue
                me = members.index(r)
                ok = all(counts[m][1][me] == send[i] for i, m in enumerate(members))
                if ok:
                    break
            else:
                pytest.fail(f"no consistent group for rank {r} transpose {t}")
        tot_s = sum(sum(c[0]) for c in counts)
        tot_r = sum(sum(c[1]) for c in counts)
        assert tot_s == tot_r


def test_error_codes_and_messages():
    with pytest.raises(D.Error, match="^SlabTooManyRanks"):
        D.plan_slab((4, 6, 8), 5, D.TransformKind.C2C, D.Direction.Forward)
    with pytest.raises(D.Error, match="^ConfigInvalid"):
        D.plan_pencil((4, 4, 4), (1, 1), D.TransformKind.R2C, D.Direction.Backward)
    with pytest.raises(D.Error, match="^GridMismatch"):
        D.plan_pencil((4, 4, 4), (2,), D.TransformKind.C2C, D.Direction.Forward)
    with pytest.raises(D.Error, match="^RankTooLow"):
        D.plan_general((2, 2, 2), (2, 4), D.TransformKind.C2C, D.Direction.Forward)
    p = D.plan_pencil((5, 5, 5), (1, 4), D.TransformKind.C2C, D.Direction.Forward)
    assert p.warnings == ["some ranks own empty blocks"]
    with pytest.raises(D.Error, match="^OutOfRange"):
        D.local_index(p.output, (5, 0, 0))


def test_local_index_spot():
    # test_plan.cpp:192-209
    p = D.plan_pencil((8, 4, 6), (2, 2), D.TransformKind.R2C, D.Direction.Forward)
    assert D.local_index(p.output, (5, 1, 2)) == (1, (5 * 2 + 1) * 2 + 0)
    assert p.output.dims == (8, 4, 4)
    assert D.hat_dims((256, 512, 1024), D.TransformKind.R2C) == (256, 512, 513)


# ------------------------------------------------------ gloo world (N > 1)

def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _gloo_worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1506_07933_b200.dfft import _all_gather_bytes
        # the context-handle exchange make_context performs (128-byte blobs)
        blob = bytes([rank]) * _lib.lib().dfftb_ctx_handle_size()
        got = _all_gather_bytes(blob, dist.group.WORLD)
        assert [b[0] for b in got] == list(range(world))
        # each rank computes its own block of the seeded field from its
        # extents; the gathered blocks reproduce the global field
        dims = [16, 8, 32]
        plan = D.plan_pencil(dims, (2, 1), D.TransformKind.C2C, D.Direction.Forward)
        full = O.seeded(dims, True)
        ext = plan.input.extents_of(rank)
        sl = tuple(slice(o, o + n) for o, n in ext)
        blocks = [None] * world
        dist.all_gather_object(blocks, (ext, full[sl]))
        rebuilt = np.zeros(dims, np.complex128)
        for e, b in blocks:
            rebuilt[tuple(slice(o, o + n) for o, n in e)] = b
        assert np.array_equal(rebuilt, full)
        # exchange counts agree across the world: what r sends to q == what q expects
        sc, rc = plan.exchange_counts(rank, 1)
        allc = [None] * world
        dist.all_gather_object(allc, (sc, rc))
        for r in range(world):
            for qq in range(world):
                assert allc[r][0][qq] == allc[qq][1][r]
        q.put((rank, "ok"))
    except Exception as e:  # noqa: BLE001
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


def test_gloo_world_size_2_host_path():
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_gloo_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=120) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    assert res == {0: "ok", 1: "ok"}, res


def test_workspace_bytes():
    # dfftb_workspace_bytes (host-only): flag page (64 sync points x 64
    # ranks) + one exchange buffer per transpose stage and execute parity
    # (two parities with peers, one for a single rank) + the work buffer (slab
    # plans only: F2 -> F1 without a transpose), each sized for the largest
    # block of the plan family, + status words + the per-axis twiddle (and
    # Bluestein) tables (+ the half-length table of the last axis of R2C / C2R
    # plans, for the half-length real lanes)
    # With peers the flag page and the buffers are rounded to 2 MiB (NVLink
    # destinations on 2 MiB boundaries); a single rank rounds to 256 bytes.
    flags = 64 * 64 * 8
    MiB2 = 2 << 20
    p = D.plan_pencil((512, 512, 512), (2, 4), D.TransformKind.C2C, D.Direction.Forward)
    blk = 512 ** 3 * 16 // 8
    # + staging images for the copy-engine exchange: one per other member of
    # the largest group (3 for the 2x4 grid)
    assert D.workspace_bytes(p, 0) == MiB2 + 2 * 2 * blk + 3 * blk + 64 + 512 * 16
    one = D.plan_pencil((512, 512, 512), (1, 1), D.TransformKind.C2C, D.Direction.Forward)
    assert D.workspace_bytes(one, 0) == flags + 2 * 512 ** 3 * 16 + 64 + 512 * 16  # 2 slots, 1 parity
    sl = D.plan_slab((64, 64, 64), 4, D.TransformKind.C2C, D.Direction.Forward)
    blk = MiB2  # 64^3 * 16 / 4 = 1 MiB, rounded
    assert D.workspace_bytes(sl, 0) == MiB2 + 2 * 2 * blk + blk + 3 * blk + 64 + 64 * 16  # slab: + work buffer
    q = D.plan_pencil((1024, 64, 64), (2, 4), D.TransformKind.C2C, D.Direction.Forward)
    blk = 1024 * 64 * 64 * 16 // 8
    assert D.workspace_bytes(q, 0) == MiB2 + 2 * 2 * blk + 3 * blk + 64 + (1024 + 64) * 16
    # R2C: + the n/2-point table of the last axis (half-length real lanes)
    r1 = D.plan_pencil((64, 64, 256), (1, 1), D.TransformKind.R2C, D.Direction.Forward)
    c1 = D.plan_pencil((64, 64, 256), (1, 1), D.TransformKind.C2C, D.Direction.Forward)
    assert D.workspace_bytes(r1, 0) - D.workspace_bytes(c1, 0) == 128 * 16
    g = D.plan_general((8, 8, 16, 16), (1, 1, 1), D.TransformKind.C2C, D.Direction.Forward)
    blk = 8 * 8 * 16 * 16 * 16
    assert D.workspace_bytes(g, 0) == flags + 3 * blk + 64 + (8 + 16) * 16  # three transposes, 1 rank
    # Bluestein length 17: chirp (17) + kernel spectrum (m = 64), fp32 complex
    b = D.plan_pencil((17, 4, 4), (1, 1), D.TransformKind.C2C, D.Direction.Forward, precision="f32")
    blk = (17 * 4 * 4 * 8 + 255) // 256 * 256
    assert D.workspace_bytes(b, 0) == flags + 2 * blk + 64 + (17 + 64) * 8 + 4 * 8
    with pytest.raises(D.Error, match="InvalidRank"):
        D.workspace_bytes(p, 8)
