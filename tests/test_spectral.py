"""Spectral operators (spectral.hpp) on the B200 path, modelled on the
reference's test_spectral.cpp.  Wavenumber conventions are host-side (CPU);
the operators run on one GPU (single rank) and are checked against analytic
fields and against numpy FFT multipliers."""
import math

import numpy as np
import pytest
import torch

import paper_1506_07933_b200 as D
from paper_1506_07933_b200 import spectral as S

TWO_PI = 2 * math.pi


def _fwd_plan(dims, grid, kind):
    k = D.TransformKind.R2C if kind == "r2c" else D.TransformKind.C2C
    if len(grid) == 1:
        return D.plan_slab(dims, grid[0], k, D.Direction.Forward)
    return D.plan_pencil(dims, grid, k, D.Direction.Forward)


def test_wavenumber_conventions():
    # test_spectral.cpp:33-75
    m = S.wavenumbers(_fwd_plan((4, 4, 4), (1, 1), "c2c"), 0)
    assert m.axis_k[0] == [0, 1, -2, -1]
    assert m.axis_k_deriv[0] == [0, 1, 0, -1]
    m = S.wavenumbers(_fwd_plan((4, 4, 8), (1, 1), "r2c"), 0)
    assert m.axis_k[2] == [0, 1, 2, 3, 4]
    assert m.axis_k_deriv[2] == [0, 1, 2, 3, 0]
    m = S.wavenumbers(_fwd_plan((8, 8, 8), (2, 2), "c2c"), 0)
    assert m.axis_k[0][0] == 0 and m.axis_k[1][0] == 0 and m.axis_k[2][0] == 0
    m = S.wavenumbers(_fwd_plan((4, 4, 4), (1, 1), "c2c"), 0, [1.0, TWO_PI, TWO_PI])
    assert m.axis_k[0][1] == pytest.approx(TWO_PI)
    bwd = D.plan_pencil((4, 4, 4), (1, 1), D.TransformKind.C2C, D.Direction.Backward)
    with pytest.raises(D.Error, match="NotFrequencyLayout"):
        S.wavenumbers(bwd, 0)


gpu = pytest.mark.gpu


def _field(dims, fn, kind):
    z, y, x = np.meshgrid(*[np.arange(n) * TWO_PI / n for n in dims], indexing="ij")
    v = fn(z, y, x)
    return v.astype(np.float64 if kind == "r2c" else np.complex128)


def _tensor(plan, arr):
    return D.DistTensor(plan.input, 0, torch.from_numpy(np.ascontiguousarray(arr).reshape(-1)).cuda())


@gpu
@pytest.mark.parametrize("kind", ["r2c", "c2c"])
def test_gradient_of_sine_mode(kind):
    # test_spectral.cpp:79-100: d/dz sin(2 z) = 2 cos(2 z), other components 0
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    dims = (8, 8, 8)
    ctx = S.make_spectral_context(dims, (1, 1))
    plan = ctx.fwd_r2c if kind == "r2c" else ctx.fwd_c2c
    x = _tensor(plan, _field(dims, lambda z, y, x_: np.sin(2 * x_), kind))
    g = S.gradient(ctx, x)
    want = _field(dims, lambda z, y, x_: 2 * np.cos(2 * x_), kind).reshape(-1)
    assert np.max(np.abs(g[2].data.cpu().numpy() - want)) < 1e-10
    assert np.max(np.abs(g[0].data.cpu().numpy())) < 1e-10
    assert np.max(np.abs(g[1].data.cpu().numpy())) < 1e-10


@gpu
def test_operators_match_numpy_multipliers():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    dims = (16, 8, 32)
    L = [1.0, 2.0, TWO_PI]
    ctx = S.make_spectral_context(dims, (1, 1), L)
    rng = np.random.default_rng(3)
    f = rng.standard_normal(dims)
    f -= f.mean()  # zero mean for the inverse Laplacian
    kk = np.meshgrid(*[TWO_PI / L[a] * np.fft.fftfreq(dims[a], 1.0 / dims[a]) for a in range(3)],
                     indexing="ij")
    F = np.fft.fftn(f)
    x = _tensor(ctx.fwd_r2c, f)
    for a in range(3):
        kd = kk[a].copy()
        kd[np.abs(kd) * L[a] / TWO_PI == dims[a] // 2] = 0  # Nyquist zeroed for derivatives
        want = np.fft.ifftn(1j * kd * F).real
        got = S.derivative(ctx, x, a).data.cpu().numpy().reshape(dims)
        assert np.max(np.abs(got - want)) < 1e-9 * np.max(np.abs(want) + 1)
    k2 = kk[0] ** 2 + kk[1] ** 2 + kk[2] ** 2
    lap = np.fft.ifftn(-k2 * F).real
    got = S.laplacian(ctx, x).data.cpu().numpy().reshape(dims)
    assert np.max(np.abs(got - lap)) < 1e-9 * np.max(np.abs(lap))
    k2i = np.where(k2 == 0, np.inf, k2)
    inv = np.fft.ifftn(F / -k2i).real
    got = S.inverse_laplacian(ctx, x).data.cpu().numpy().reshape(dims)
    assert np.max(np.abs(got - inv)) < 1e-9 * np.max(np.abs(inv))
    # div(grad f) == lap f (test_spectral.cpp:274-292, Nyquist-free field)
    fs = _field(dims, lambda z, y, x_: np.sin(3 * z) * np.cos(2 * y) + np.sin(5 * x_), "r2c")
    ctx2 = S.make_spectral_context(dims, (1, 1))
    xs = _tensor(ctx2.fwd_r2c, fs)
    dg = S.divergence(ctx2, S.gradient(ctx2, xs)).data.cpu().numpy()
    lp = S.laplacian(ctx2, xs).data.cpu().numpy()
    assert np.max(np.abs(dg - lp)) < 1e-9 * np.max(np.abs(lp))


@gpu
def test_inverse_laplacian_needs_zero_mean():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    dims = (8, 8, 8)
    ctx = S.make_spectral_context(dims, (1, 1))
    x = _tensor(ctx.fwd_r2c, np.ones(dims))
    with pytest.raises(D.Error, match="NonZeroMean"):
        S.inverse_laplacian(ctx, x)


@gpu
def test_spectral_on_emulated_world():
    # pencil 2x2 blocks: multipliers use each rank's global frequency offsets
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    dims = (8, 16, 8)
    fwd = D.plan_pencil(dims, (2, 2), D.TransformKind.C2C, D.Direction.Forward)
    bwd = D.plan_pencil(dims, (2, 2), D.TransformKind.C2C, D.Direction.Backward)
    ctxs = D.make_world_contexts(fwd)
    f = _field(dims, lambda z, y, x_: np.exp(1j * (2 * z - 3 * y + x_)), "c2c")
    from gpu_util import gather, scatter
    xs = scatter(fwd.input, f)
    ys = D.execute_world(fwd, xs, ctxs)
    import ctypes
    for r, y in enumerate(ys):
        with torch.cuda.device(y.data.device):
            D.dfft._check(D._lib.lib().dfftb_spectral_apply(fwd._h, r, S.DERIV, 1, None,
                                                            y.data.data_ptr(), y.data.data_ptr(), 0,
                                                            torch.cuda.current_stream().cuda_stream))
    zs = D.execute_world(bwd, ys, ctxs)
    got = gather(bwd.output, zs)
    assert np.max(np.abs(got - (-3j) * f)) < 1e-10


def _spectral_pair(plan, ctx, x, op, axis, lens=None, accumulate_into=None):
    """(fused, unfused) spectra of op(forward(x)) for one rank."""
    import ctypes
    lib = D._lib.lib()
    nd = len(plan.dims)
    cl = (ctypes.c_double * nd)(*lens) if lens else None
    stream = torch.cuda.current_stream().cuda_stream
    n = plan.output.local_count(0)
    fused = torch.zeros(n, dtype=plan.dtype_of(plan.output), device="cuda")
    if accumulate_into is not None:
        fused.copy_(accumulate_into)
    D.dfft._check(lib.dfftb_execute_spectral(plan._h, ctx._h, x.data.data_ptr(), fused.data_ptr(), op, axis,
                                             cl, 1 if accumulate_into is not None else 0, stream, 1))
    spec = D.execute(plan, x, ctx)
    unf = torch.zeros_like(fused)
    if accumulate_into is not None:
        unf.copy_(accumulate_into)
    D.dfft._check(lib.dfftb_spectral_apply(plan._h, 0, op, axis, cl, spec.data.data_ptr(), unf.data_ptr(),
                                           1 if accumulate_into is not None else 0, stream))
    torch.cuda.synchronize()
    return fused.cpu(), unf.cpu()


FUSED_CASES = [
    ("pencil", (32, 16, 64), (1, 1), "c2c", "f64"),
    ("pencil", (32, 16, 64), (1, 1), "r2c", "f64"),
    ("slab", (64, 32, 16), (1,), "c2c", "f32"),
    ("pencil", (16, 32, 32), (1, 1), "r2c", "f32"),
    ("pencil", (24, 20, 16), (1, 1), "c2c", "f64"),   # non-pow2: two-step fallback
    ("slab", (64, 32), (1,), "c2c", "f64"),           # 2-D
    ("general", (8, 8, 16, 16), (1, 1, 1), "c2c", "f64"),  # 4-D
]


@gpu
@pytest.mark.parametrize("decomp,dims,grid,kind,prec", FUSED_CASES)
def test_fused_spectral_epilogue_matches_two_step(decomp, dims, grid, kind, prec):
    """dfftb_execute_spectral (multiplier in the last forward pass's store)
    is bit-identical to execute + dfftb_spectral_apply."""
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    k = D.TransformKind.R2C if kind == "r2c" else D.TransformKind.C2C
    mk = {"pencil": D.plan_pencil, "general": D.plan_general}.get(decomp)
    if decomp == "slab":
        plan = D.plan_slab(dims, grid[0], k, D.Direction.Forward, precision=prec)
    else:
        plan = mk(dims, grid, k, D.Direction.Forward, precision=prec)
    ctx = D.make_context(plan)
    x = D.DistTensor.seeded(plan.input, 0, complex_field=kind == "c2c")
    lens = [1.0 + a for a in range(len(dims))]
    for op, axis in [(S.DERIV, a) for a in range(len(dims))] + [(S.LAPLACIAN, 0)]:
        f, u = _spectral_pair(plan, ctx, x, op, axis, lens)
        assert torch.equal(f, u), (op, axis)
    # accumulate (divergence) into an existing spectrum
    base = D.execute(plan, x, ctx).data.clone()
    f, u = _spectral_pair(plan, ctx, x, S.DERIV, len(dims) - 1, lens, accumulate_into=base)
    assert torch.equal(f, u)
    if prec == "f32":
        return  # a float32 field cannot be made zero-mean to 1e-12 N
    # inverse Laplacian of a zero-mean field
    xm = D.DistTensor(plan.input, 0, x.data - x.data.mean())
    f, u = _spectral_pair(plan, ctx, xm, S.INV_LAPLACIAN, 0, lens)
    assert torch.equal(f, u)


@gpu
def test_fused_inverse_laplacian_nonzero_mean():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    plan = D.plan_pencil((16, 16, 16), (1, 1), D.TransformKind.C2C, D.Direction.Forward)
    ctx = D.make_context(plan)
    x = D.DistTensor(plan.input, 0, torch.ones(16 ** 3, dtype=torch.complex128, device="cuda"))
    out = torch.empty_like(x.data)
    import ctypes
    st = D._lib.lib().dfftb_execute_spectral(plan._h, ctx._h, x.data.data_ptr(), out.data_ptr(),
                                             S.INV_LAPLACIAN, 0, None, 0,
                                             torch.cuda.current_stream().cuda_stream, 1)
    assert D._lib.lib().dfftb_error_name(st).decode() == "NonZeroMean"
