"""Python mirror of the reference's plan / execute / local-size API.

Same names, argument meaning and error behaviour as the C++20 templates in
/root/reference/proj/include/dfft/ (cited per function), executed on B200 by
libdfftb.so through the C ABI.  Buffers are CUDA torch tensors (plumbing);
multi-rank worlds are one process per GPU over torch.distributed (only used
to exchange 128-byte context handles; the data path is the fused FFT +
NVLink peer-store kernel inside libdfftb).

    plan = plan_pencil((512, 512, 512), ProcessGrid(2, 4), TransformKind.C2C,
                       Direction.Forward)
    ctx = make_context(plan, comm)            # comm: torch.distributed group
    x = DistTensor.zeros(plan.input, rank)
    y = execute(plan, x, ctx)
"""
from __future__ import annotations

import ctypes
import enum
from dataclasses import dataclass, field
from typing import List, Optional, Sequence, Tuple

import torch

from . import _lib

# ----------------------------------------------------------------- errors

ERROR_NAMES = {
    1: "ZeroLength", 2: "OutOfBounds", 3: "TooLarge", 4: "LengthMismatch", 5: "NonHermitian",
    6: "SlabTooManyRanks", 7: "OutOfRange", 8: "InvalidRank", 9: "TagMismatchTimeout",
    10: "Deadlock", 11: "WorkerPanic", 12: "CountMismatch", 13: "IncompatibleLayouts",
    14: "ArenaExhausted", 15: "GridMismatch", 16: "RankTooLow", 17: "LayoutMismatch",
    18: "NotFrequencyLayout", 19: "NonZeroMean", 20: "BadMagic", 21: "DimMismatch",
    22: "TruncatedFile", 23: "ConfigInvalid", 100: "CudaError", 101: "Unsupported",
}


class Error(RuntimeError):
    """dfft::Error (errors.hpp:48-58): what() is prefixed with the code name."""

    def __init__(self, code: int, what: str):
        self.code = code
        self.code_name = ERROR_NAMES.get(code, "UnknownError")
        super().__init__(what if what.startswith(self.code_name) else f"{self.code_name}: {what}")


def _check(status: int):
    if status != 0:
        msg = _lib.lib().dfftb_last_error_message().decode()
        raise Error(status, msg)


# ------------------------------------------------------------------ enums


class TransformKind(enum.IntEnum):  # layout.hpp:289
    C2C = 0
    R2C = 1
    C2R = 2


class Direction(enum.IntEnum):  # kernels.hpp:26
    Forward = 0
    Backward = 1


class ExchangePath(enum.IntEnum):  # exchange.hpp:425
    Blocking = 0
    Staged = 1
    Pipelined = 2


class ElementKind(enum.IntEnum):  # layout.hpp:110
    Real = 0
    Complex = 1


@dataclass
class PlanOptions:  # plan.hpp:48-54
    exchange: ExchangePath = ExchangePath.Blocking
    normalize: bool = True
    chunks_per_peer: int = 1
    staging_buffers: int = 2
    validate_finite: bool = False

    def _c(self):
        return _lib.PlanOptionsC(int(self.exchange), int(bool(self.normalize)),
                                 int(self.chunks_per_peer), int(self.staging_buffers),
                                 int(bool(self.validate_finite)))


@dataclass
class TimingBreakdown:  # timing.hpp:16-37
    local_fft: float = 0.0
    pack: float = 0.0
    unpack: float = 0.0
    staging_copy: float = 0.0
    wire_comm: float = 0.0
    total: float = 0.0

    def component_sum(self):
        return self.local_fft + self.pack + self.unpack + self.staging_copy + self.wire_comm

    def max_with(self, o: "TimingBreakdown"):
        for k in ("local_fft", "pack", "unpack", "staging_copy", "wire_comm", "total"):
            setattr(self, k, max(getattr(self, k), getattr(o, k)))


class ProcessGrid(tuple):
    """Ranks on a Cartesian grid, row-major (layout.hpp:38-66)."""

    def __new__(cls, *shape):
        if len(shape) == 1 and isinstance(shape[0], (list, tuple)):
            shape = tuple(shape[0])
        return super().__new__(cls, tuple(int(s) for s in shape))

    @property
    def shape(self):
        return tuple(self)

    def ndim(self):
        return len(self)

    def size(self):
        n = 1
        for s in self:
            n *= s
        return n

    def coords_of(self, rank):
        c = [0] * len(self)
        for g in range(len(self) - 1, -1, -1):
            c[g] = rank % self[g]
            rank //= self[g]
        return c

    def rank_of(self, coords):
        r = 0
        for g, s in enumerate(self):
            r = r * s + coords[g]
        return r


def _i64(v):
    return (ctypes.c_int64 * len(v))(*[int(x) for x in v])


def _int(v):
    return (ctypes.c_int * len(v))(*[int(x) for x in v])


def block_map(n: int, p: int) -> Tuple[List[int], List[int]]:
    """Ceil-block partition (layout.hpp:80-92): (counts, offsets)."""
    c = (ctypes.c_int64 * p)()
    o = (ctypes.c_int64 * p)()
    _check(_lib.lib().dfftb_block_map(n, p, c, o))
    return list(c), list(o)


def workspace_bytes(plan: "Plan", rank: int) -> int:
    """Device bytes make_context allocates for `plan`'s family on `rank`
    (dfftb_workspace_bytes; host-only)."""
    v = ctypes.c_uint64()
    _check(_lib.lib().dfftb_workspace_bytes(plan._h, rank, ctypes.byref(v)))
    return int(v.value)


def hat_dims(dims: Sequence[int], kind: TransformKind) -> Tuple[int, ...]:
    """layout.hpp:201-207: R2C stores floor(N_last/2)+1 bins on the last axis."""
    d = list(dims)
    if kind == TransformKind.R2C and d:
        d[-1] = d[-1] // 2 + 1
    return tuple(d)


# ------------------------------------------------------------ distribution


@dataclass(frozen=True)
class Distribution:
    """Distribution (layout.hpp:125-194) of one side of a plan."""

    dims: Tuple[int, ...]
    grid: ProcessGrid
    axis_of_grid: Tuple[int, ...]
    hatted: Tuple[bool, ...]
    element: ElementKind
    _plan: object = field(default=None, compare=False, repr=False)
    _side: int = field(default=0, compare=False, repr=False)

    def ndim(self):
        return len(self.dims)

    def extents_of(self, rank: int) -> List[Tuple[int, int]]:
        """[(offset, length)] per axis (layout.hpp:165-179)."""
        nd = len(self.dims)
        off = (ctypes.c_int64 * nd)()
        ln = (ctypes.c_int64 * nd)()
        _check(_lib.lib().dfftb_plan_local_extents(self._plan._h, rank, self._side, off, ln))
        return list(zip(off, ln))

    def local_count(self, rank: int) -> int:
        n = 1
        for _, ln in self.extents_of(rank):
            n *= ln
        return n

    def local_shape(self, rank: int) -> Tuple[int, ...]:
        return tuple(ln for _, ln in self.extents_of(rank))

    def all_hatted(self):
        return all(self.hatted)


def local_index(dist: Distribution, coord: Sequence[int]) -> Tuple[int, int]:
    """Owner rank and row-major offset of a global coordinate (layout.hpp:272-295)."""
    r = ctypes.c_int()
    o = ctypes.c_int64()
    if len(coord) != len(dist.dims):
        raise Error(7, "coordinate rank mismatch")
    _check(_lib.lib().dfftb_local_index(dist._plan._h, dist._side, _i64(coord), ctypes.byref(r),
                                        ctypes.byref(o)))
    return r.value, o.value


# ------------------------------------------------------------------ plans

_DTYPES = {8: (torch.float64, torch.complex128), 4: (torch.float32, torch.complex64)}


def _prec_code(precision) -> int:
    if precision in ("f64", "double", torch.float64, torch.complex128, 8):
        return 8
    if precision in ("f32", "float", torch.float32, torch.complex64, 4):
        return 4
    raise Error(23, f"unknown precision {precision!r}")


class Plan:
    """Plan<T> (plan.hpp:59-99): immutable, shareable across ranks."""

    def __init__(self, dims, decomp, grid, kind, direction, precision="f64", options=None):
        self.dims = tuple(int(d) for d in dims)
        self.decomp = decomp
        self.grid = ProcessGrid(grid)
        self.kind = TransformKind(kind)
        self.direction = Direction(direction)
        self.prec = _prec_code(precision)
        self.options = options or PlanOptions()
        h = ctypes.c_void_p()
        _check(_lib.lib().dfftb_plan_create(len(self.dims), _i64(self.dims), decomp,
                                            len(self.grid), _int(self.grid), int(self.kind),
                                            int(self.direction), self.prec,
                                            ctypes.byref(self.options._c()), ctypes.byref(h)))
        self._h = h
        self.input = self._layout(0)
        self.output = self._layout(1)
        L = _lib.lib()
        self.warnings = [L.dfftb_plan_warning(h, i).decode()
                         for i in range(L.dfftb_plan_warning_count(h))]

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                _lib.lib().dfftb_plan_destroy(h)
            except Exception:
                pass
            self._h = None

    def _layout(self, side):
        nd = len(self.dims)
        dims = (ctypes.c_int64 * nd)()
        el = ctypes.c_int()
        aog = (ctypes.c_int * len(self.grid))()
        hat = (ctypes.c_int * nd)()
        _check(_lib.lib().dfftb_plan_layout(self._h, side, dims, ctypes.byref(el), aog, hat))
        return Distribution(tuple(dims), self.grid, tuple(aog), tuple(bool(x) for x in hat),
                            ElementKind(el.value), self, side)

    @property
    def real_dtype(self):
        return _DTYPES[self.prec][0]

    @property
    def complex_dtype(self):
        return _DTYPES[self.prec][1]

    def dtype_of(self, dist: Distribution):
        return self.complex_dtype if dist.element == ElementKind.Complex else self.real_dtype

    def nranks(self):
        return self.grid.size()

    def signature(self) -> str:
        buf = ctypes.create_string_buffer(256)
        _check(_lib.lib().dfftb_plan_signature(self._h, buf, 256))
        return buf.value.decode()

    def fft_stage_count(self) -> int:
        return _lib.lib().dfftb_plan_fft_stage_count(self._h)

    def transpose_stage_count(self) -> int:
        return _lib.lib().dfftb_plan_transpose_stage_count(self._h)

    def exchange_counts(self, rank: int, transpose_index: int):
        """make_transpose_step send/recv counts (exchange.hpp:531-540)."""
        s = (ctypes.c_int64 * 64)()
        r = (ctypes.c_int64 * 64)()
        n = ctypes.c_int()
        _check(_lib.lib().dfftb_plan_exchange_counts(self._h, rank, transpose_index, s, r,
                                                     ctypes.byref(n)))
        return list(s[:n.value]), list(r[:n.value])


def plan_slab(dims, ranks: int, kind, direction, options=None, precision="f64") -> Plan:
    """plan_slab (plan.hpp:267-354)."""
    return Plan(dims, 0, [int(ranks)], kind, direction, precision, options)


def plan_pencil(dims, grid, kind, direction, options=None, precision="f64") -> Plan:
    """plan_pencil (plan.hpp:242-250)."""
    return Plan(dims, 1, ProcessGrid(grid), kind, direction, precision, options)


def plan_general(dims, grid, kind, direction, options=None, precision="f64") -> Plan:
    """plan_general (plan.hpp:253-262)."""
    return Plan(dims, 2, ProcessGrid(grid), kind, direction, precision, options)


# ------------------------------------------------------------ dist tensor


class DistTensor:
    """DistTensor<T> (dist_tensor.hpp:21-45): one rank's block, device-resident.

    `data` is a 1-D CUDA tensor (complex or real per dist.element) holding the
    rank's block row-major, last axis fastest."""

    def __init__(self, dist: Distribution, rank: int, data: torch.Tensor):
        self.dist = dist
        self.rank = rank
        self.data = data

    @staticmethod
    def zeros(dist: Distribution, rank: int, device=None) -> "DistTensor":
        plan = dist._plan
        dev = device if device is not None else torch.device("cuda", torch.cuda.current_device())
        n = dist.local_count(rank)
        return DistTensor(dist, rank, torch.zeros(n, dtype=plan.dtype_of(dist), device=dev))

    @staticmethod
    def seeded(dist: Distribution, rank: int, seed: int = 1, complex_field: bool = True,
               device=None) -> "DistTensor":
        """fill_from_global with the bench's seeded field (bench.cpp:132-136), on device."""
        t = DistTensor.zeros(dist, rank, device)
        stream = torch.cuda.current_stream(t.data.device).cuda_stream
        with torch.cuda.device(t.data.device):
            _check(_lib.lib().dfftb_fill_seeded(dist._plan._h, rank, dist._side, seed,
                                                int(bool(complex_field)), t.data.data_ptr(),
                                                stream))
        return t

    @property
    def real(self):
        return self.data if self.dist.element == ElementKind.Real else None

    @property
    def cplx(self):
        return self.data if self.dist.element == ElementKind.Complex else None

    def extents(self):
        return self.dist.extents_of(self.rank)

    def local_size(self) -> int:
        return self.data.numel()

    def block(self) -> torch.Tensor:
        """The local block viewed with its local shape."""
        return self.data.view(self.dist.local_shape(self.rank))


# --------------------------------------------------------------- contexts


class ExecContext:
    """ExecContext (plan.hpp:359-363): this rank's exchange buffers, mapped
    peer buffers and barrier flags."""

    def __init__(self, handle, rank, device, nranks, world=None):
        self._h = handle
        self.rank = rank
        self.device = device
        self.nranks = nranks
        self._world = world  # for emulated worlds: keep siblings alive

    def close(self):
        if self._h is not None and self._h.value:
            torch.cuda.synchronize(self.device)
            _lib.lib().dfftb_ctx_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def check(self, stream=None):
        """Surface deferred errors (NonHermitian, peer timeouts)."""
        s = stream if stream is not None else torch.cuda.current_stream(self.device).cuda_stream
        _check(_lib.lib().dfftb_ctx_check(self._h, s))

    def last_ops(self):
        """Per-op device times of the last execute given `timers`: a list of
        (kind, stream, length, share, start_ms, ms) with kind "local" (FFT
        pass), "exchange" (FFT pass storing into other ranks' buffers or
        their staging images), "sync" or "copy" (a copy-engine DMA of the
        staged exchange); stream 1 is the overlapped pass on the context's
        side stream, 2 its copy streams; share = the fraction of the pass's
        lanes a chunked pass launch covers; start_ms from the execute's
        start."""
        L = _lib.lib()
        n = L.dfftb_ctx_last_ops(self._h, None, None, None, None, None, None, 0)
        m = max(n, 1)
        k, st, ln = (ctypes.c_int * m)(), (ctypes.c_int * m)(), (ctypes.c_int * m)()
        sh, t0, ms = (ctypes.c_double * m)(), (ctypes.c_double * m)(), (ctypes.c_double * m)()
        L.dfftb_ctx_last_ops(self._h, k, st, ln, sh, t0, ms, n)
        names = ("local", "exchange", "sync", "copy")
        return [(names[k[i]], st[i], ln[i], sh[i], t0[i], ms[i]) for i in range(n)]


def _resolve_device(device) -> torch.device:
    dev = torch.device(device) if device is not None else torch.device("cuda")
    if dev.type != "cuda":
        raise Error(23, "dfftb executes on CUDA devices only")
    if dev.index is None:
        dev = torch.device("cuda", torch.cuda.current_device())
    return dev


def _all_gather_bytes(blob: bytes, comm) -> List[bytes]:
    import torch.distributed as dist
    out = [None] * dist.get_world_size(comm)
    dist.all_gather_object(out, blob, group=comm)
    return out


def make_context(plan: Plan, comm=None, rank: Optional[int] = None, device=None) -> ExecContext:
    """make_context (plan.hpp:365-390).  Collective over `comm`.

    comm: a torch.distributed process group (default: the world, when
    initialized), or None for a single-rank plan.  The grid's row-major ranks
    are the group ranks; one GPU per rank."""
    import torch.distributed as tdist
    if comm is None and tdist.is_available() and tdist.is_initialized():
        comm = tdist.group.WORLD
    if comm is not None:
        size = tdist.get_world_size(comm)
        my = tdist.get_rank(comm)
    else:
        size, my = 1, 0
    if rank is not None:
        my = rank
    if size != plan.nranks():
        raise Error(15, "communicator size must match the grid")
    dev = _resolve_device(device)
    L = _lib.lib()
    h = ctypes.c_void_p()
    with torch.cuda.device(dev):
        _check(L.dfftb_ctx_create(plan._h, my, dev.index, ctypes.byref(h)))
        if size > 1:
            hs = L.dfftb_ctx_handle_size()
            buf = ctypes.create_string_buffer(hs)
            _check(L.dfftb_ctx_export_handle(h, buf))
            blobs = _all_gather_bytes(buf.raw, comm)
            allb = ctypes.create_string_buffer(b"".join(blobs), hs * size)
            _check(L.dfftb_ctx_connect(h, allb))
            tdist.barrier(group=comm)
    return ExecContext(h, my, dev, size)


def make_world_contexts(plan: Plan, device=None, devices=None) -> List[ExecContext]:
    """All P ranks of the plan emulated in THIS process (test harness for the
    exchange logic when fewer processes or GPUs than ranks exist); use
    execute_world.  `devices`: rank r lives on devices[r % len(devices)]
    (exchange stores cross NVLink); default: every rank on `device`."""
    P = plan.nranks()
    if devices is None:
        devs = [_resolve_device(device)]
    else:
        devs = [_resolve_device(d) for d in devices]
    arr = (ctypes.c_void_p * P)()
    ids = (ctypes.c_int * len(devs))(*[d.index for d in devs])
    with torch.cuda.device(devs[0]):
        _check(_lib.lib().dfftb_world_create_devices(plan._h, len(devs), ids, arr))
    ctxs = [ExecContext(ctypes.c_void_p(arr[r]), r, devs[r % len(devs)], P) for r in range(P)]
    for c in ctxs:
        c._world = ctxs
    return ctxs


# ---------------------------------------------------------------- execute


def _needs_sync(plan: Plan) -> bool:
    return plan.kind == TransformKind.C2R or plan.options.validate_finite


def execute(plan: Plan, x: DistTensor, ctx: ExecContext,
            timers: Optional[TimingBreakdown] = None, out: Optional[DistTensor] = None,
            sync: Optional[bool] = None) -> DistTensor:
    """execute (plan.hpp:463-535): collective; returns this rank's output block.

    The input is not modified.  Launches are asynchronous on the current
    stream unless timers are requested or the plan needs its deferred checks
    (C2R Hermitian check, finiteness validation) — then errors surface here
    as in the reference."""
    if x.dist is not plan.input and x.dist != plan.input:
        raise Error(17, "input layout differs from the plan's")
    dev = x.data.device
    if dev.type != "cuda":
        raise Error(23, "DistTensor data must live on a CUDA device")
    if out is None:
        out = DistTensor(plan.output, x.rank,
                         torch.empty(plan.output.local_count(x.rank),
                                     dtype=plan.dtype_of(plan.output), device=dev))
    if sync is None:
        sync = _needs_sync(plan)
    xd = x.data if x.data.is_contiguous() else x.data.contiguous()
    # the library switches to the context's device itself (and back)
    stream = torch.cuda.current_stream(dev).cuda_stream
    tc = _lib.TimingC() if timers is not None else None
    _check(_lib.lib().dfftb_execute(plan._h, ctx._h, xd.data_ptr(), out.data.data_ptr(),
                                    stream, 1 if sync else 0,
                                    ctypes.byref(tc) if tc is not None else None))
    if timers is not None:
        for k in ("local_fft", "pack", "unpack", "staging_copy", "wire_comm", "total"):
            setattr(timers, k, getattr(timers, k) + getattr(tc, k))
    return out


def execute_r2c_c2r_roundtrip(forward: Plan, backward: Plan, x: DistTensor, ctx: ExecContext,
                              timers: Optional[TimingBreakdown] = None) -> DistTensor:
    """plan.hpp:539-552."""
    if (forward.kind != TransformKind.R2C or backward.kind != TransformKind.C2R
            or forward.dims != backward.dims or forward.grid != backward.grid):
        raise Error(15, "round trip needs matching R2C/C2R plans")
    return execute(backward, execute(forward, x, ctx, timers), ctx, timers)


def execute_world(plan: Plan, xs: Sequence[DistTensor], ctxs: Sequence[ExecContext],
                  sync: Optional[bool] = None) -> List[DistTensor]:
    """Lockstep execution of all ranks of an emulated world (rank r's input
    and output on its context's device); enqueued on the current stream of
    rank 0's device."""
    P = plan.nranks()
    if len(xs) != P or len(ctxs) != P:
        raise Error(15, "need one input and one context per rank")
    outs = []
    for r, x in enumerate(xs):
        if x.dist != plan.input or x.rank != r:
            raise Error(17, "input layout differs from the plan's")
        outs.append(DistTensor(plan.output, r, torch.empty(
            plan.output.local_count(r), dtype=plan.dtype_of(plan.output), device=ctxs[r].device)))
    if sync is None:
        sync = _needs_sync(plan)
    ins = (ctypes.c_void_p * P)(*[x.data.data_ptr() for x in xs])
    os_ = (ctypes.c_void_p * P)(*[o.data.data_ptr() for o in outs])
    hs = (ctypes.c_void_p * P)(*[c._h.value for c in ctxs])
    dev = ctxs[0].device
    with torch.cuda.device(dev):
        _check(_lib.lib().dfftb_execute_world(plan._h, hs, ins, os_,
                                              torch.cuda.current_stream(dev).cuda_stream,
                                              1 if sync else 0))
    return outs


def kernel_launch_count() -> int:
    return int(_lib.lib().dfftb_kernel_launch_count())
