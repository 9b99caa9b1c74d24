"""Spectral operators over the distributed FFT (spectral.hpp:1-311).

Mirror of the reference's SpectralContext / derivative / gradient /
divergence / laplacian / inverse_laplacian.  The forward and backward
transforms are the B200 execute path; the i*k and -|k|^2 multipliers run as
one device kernel over this rank's frequency block (dfftb_spectral_apply),
or — the default for the operators below — inside the store epilogue of the
forward transform's last pass (dfftb_execute_spectral: one pass over the
spectrum less, bit-identical values).
"""
from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import torch

from . import _lib
from .dfft import (Direction, DistTensor, Distribution, ElementKind, Error, ExecContext, Plan,
                   TransformKind, _check, make_context, plan_general, plan_pencil, plan_slab)

DERIV, LAPLACIAN, INV_LAPLACIAN = 0, 1, 2


@dataclass
class WavenumberMap:  # spectral.hpp:17-20
    axis_k: List[List[float]] = field(default_factory=list)
    axis_k_deriv: List[List[float]] = field(default_factory=list)


def _lengths(domain_lengths, nd):
    if domain_lengths is None:
        return None
    if len(domain_lengths) != nd:
        raise Error(18, "one domain length per axis")
    return (ctypes.c_double * nd)(*[float(x) for x in domain_lengths])


def wavenumbers(plan: Plan, rank: int, domain_lengths: Optional[Sequence[float]] = None) -> WavenumberMap:
    """spectral.hpp:24-56 for this rank's block of a forward plan's output."""
    if plan.direction != Direction.Forward:
        raise Error(18, "wavenumbers need a fully transformed complex layout")
    nd = len(plan.dims)
    lens = _lengths(domain_lengths, nd)
    m = WavenumberMap()
    for a, (off, ln) in enumerate(plan.output.extents_of(rank)):
        for deriv, dst in ((0, m.axis_k), (1, m.axis_k_deriv)):
            buf = (ctypes.c_double * max(1, ln))()
            _check(_lib.lib().dfftb_wavenumbers(plan._h, rank, a, deriv, lens, buf))
            dst.append(list(buf[:ln]))
    return m


class SpectralContext:
    """spectral.hpp:61-98: plans for complex (C2C) and real (R2C/C2R)
    fields on one (dims, grid, comm), their wavenumber tables and one
    execution context shared by all four plans."""

    def __init__(self, dims, grid, domain_lengths=None, precision="f64", comm=None, rank=None,
                 decomp="pencil"):
        self.dims = tuple(int(d) for d in dims)
        self.grid = tuple(grid)
        self.domain_lengths = list(domain_lengths) if domain_lengths else [2 * math.pi] * len(self.dims)
        mk = {"pencil": plan_pencil, "general": plan_general}.get(decomp)
        if decomp == "slab":
            def mk(d, g, k, dr, precision):  # noqa: E306
                return plan_slab(d, g[0], k, dr, precision=precision)
        self.fwd_c2c = mk(self.dims, self.grid, TransformKind.C2C, Direction.Forward, precision=precision)
        self.bwd_c2c = mk(self.dims, self.grid, TransformKind.C2C, Direction.Backward, precision=precision)
        self.fwd_r2c = mk(self.dims, self.grid, TransformKind.R2C, Direction.Forward, precision=precision)
        self.bwd_c2r = mk(self.dims, self.grid, TransformKind.C2R, Direction.Backward, precision=precision)
        self.exec = make_context(self.fwd_c2c, comm, rank=rank)
        self.rank = self.exec.rank
        self.k_c2c = wavenumbers(self.fwd_c2c, self.rank, self.domain_lengths)
        self.k_r2c = wavenumbers(self.fwd_r2c, self.rank, self.domain_lengths)

    def _plans(self, x: DistTensor):
        real = x.dist.element == ElementKind.Real
        return (self.fwd_r2c, self.bwd_c2r) if real else (self.fwd_c2c, self.bwd_c2c)

    def _apply(self, fwd: Plan, op, axis, src: DistTensor, dst: DistTensor, accumulate=False):
        nd = len(self.dims)
        lens = _lengths(self.domain_lengths, nd)
        stream = torch.cuda.current_stream(src.data.device).cuda_stream
        with torch.cuda.device(src.data.device):
            _check(_lib.lib().dfftb_spectral_apply(fwd._h, src.rank, op, axis, lens,
                                                   src.data.data_ptr(), dst.data.data_ptr(),
                                                   1 if accumulate else 0, stream))


    def _forward_op(self, fwd: Plan, op, axis, x: DistTensor, out: Optional[DistTensor] = None,
                    accumulate=False) -> DistTensor:
        """out (+)= op(forward(x)) with the multiplier fused into the forward's
        last pass (dfftb_execute_spectral)."""
        if x.dist != fwd.input:
            raise Error(17, "input layout differs from the plan's")
        if out is None:
            out = DistTensor(fwd.output, x.rank,
                             torch.empty(fwd.output.local_count(x.rank), dtype=fwd.dtype_of(fwd.output),
                                         device=x.data.device))
        nd = len(self.dims)
        lens = _lengths(self.domain_lengths, nd)
        xd = x.data if x.data.is_contiguous() else x.data.contiguous()
        stream = torch.cuda.current_stream(x.data.device).cuda_stream
        with torch.cuda.device(x.data.device):
            _check(_lib.lib().dfftb_execute_spectral(fwd._h, self.exec._h, xd.data_ptr(), out.data.data_ptr(),
                                                     op, axis, lens, 1 if accumulate else 0, stream, 0))
        return out


def world_forward_op(fwd: Plan, ctxs: Sequence[ExecContext], xs: Sequence[DistTensor], op: int, axis: int = 0,
                     domain_lengths=None, outs: Optional[Sequence[DistTensor]] = None,
                     accumulate: bool = False) -> List[DistTensor]:
    """dfftb_execute_world_spectral: outs[r] (+)= op(forward(x))[r] for every
    rank of an emulated world (make_world_contexts), the multiplier fused
    into the forward's last pass.  Test harness for multi-rank spectral
    operators on fewer GPUs than ranks."""
    P = fwd.nranks()
    nd = len(fwd.dims)
    lens = _lengths(domain_lengths, nd)
    if outs is None:
        outs = [DistTensor(fwd.output, r, torch.empty(fwd.output.local_count(r), dtype=fwd.dtype_of(fwd.output),
                                                      device=ctxs[r].device)) for r in range(P)]
    ins = (ctypes.c_void_p * P)(*[x.data.data_ptr() for x in xs])
    os_ = (ctypes.c_void_p * P)(*[o.data.data_ptr() for o in outs])
    hs = (ctypes.c_void_p * P)(*[c._h.value for c in ctxs])
    dev = ctxs[0].device
    with torch.cuda.device(dev):
        _check(_lib.lib().dfftb_execute_world_spectral(fwd._h, hs, ins, os_, op, axis, lens,
                                                       1 if accumulate else 0,
                                                       torch.cuda.current_stream(dev).cuda_stream, 1))
    return list(outs)


def make_spectral_context(dims, grid, domain_lengths=None, precision="f64", comm=None, rank=None,
                          decomp="pencil") -> SpectralContext:
    return SpectralContext(dims, grid, domain_lengths, precision, comm, rank, decomp)


def derivative(ctx: SpectralContext, x: DistTensor, axis: int) -> DistTensor:
    """backward(i k_axis (.) forward(x)), normalized (spectral.hpp:131-164)."""
    from .dfft import execute
    fwd, bwd = ctx._plans(x)
    spec = ctx._forward_op(fwd, DERIV, axis, x)
    return execute(bwd, spec, ctx.exec)


def gradient(ctx: SpectralContext, x: DistTensor) -> List[DistTensor]:
    """spectral.hpp:167-176."""
    return [derivative(ctx, x, a) for a in range(len(ctx.dims))]


def divergence(ctx: SpectralContext, components: Sequence[DistTensor]) -> DistTensor:
    """sum_j i k_j (.) forward(c_j), one inverse transform (spectral.hpp:180-216)."""
    from .dfft import execute
    if len(components) != len(ctx.dims):
        raise Error(15, "one component per axis required")
    fwd, bwd = ctx._plans(components[0])
    acc = None
    for a, c in enumerate(components):
        acc = ctx._forward_op(fwd, DERIV, a, c, out=acc, accumulate=acc is not None)
    return execute(bwd, acc, ctx.exec)


def laplacian(ctx: SpectralContext, x: DistTensor) -> DistTensor:
    """backward(-|k|^2 (.) forward(x)), normalized (spectral.hpp:219-249)."""
    from .dfft import execute
    fwd, bwd = ctx._plans(x)
    spec = ctx._forward_op(fwd, LAPLACIAN, 0, x)
    return execute(bwd, spec, ctx.exec)


def inverse_laplacian(ctx: SpectralContext, x: DistTensor) -> DistTensor:
    """Divides by -|k|^2 with k = 0 pinned to zero; NonZeroMean unless the
    field has zero mean (spectral.hpp:251-309)."""
    from .dfft import execute
    fwd, bwd = ctx._plans(x)
    spec = ctx._forward_op(fwd, INV_LAPLACIAN, 0, x)
    return execute(bwd, spec, ctx.exec)
