"""Spectral operators pinned to the reference's own outputs.

tests/golden/spec_*.bin were produced by the UNMODIFIED reference
(oracle/_ref/dfft_ref --spectral, tests/golden/make_golden.py): derivative
along every axis, laplacian, inverse_laplacian(laplacian(x)) (fp64 only) and
divergence(gradient(x)) of the seeded field, through make_spectral_context
(spectral.hpp:131-309) on pencil and 4-D general grids.

CPU: the goldens agree with numpy FFT multipliers (what the fixtures mean).
GPU: the B200 path reproduces them at rel-L2 <= 1e-12 (fp64) / 1e-5 (fp32)
  * fused: the multiplier in the forward's last-pass store epilogue
    (dfftb_execute_spectral / dfftb_execute_world_spectral),
  * two-step: execute, then the multiply kernel (dfftb_spectral_apply),
for every rank of the grid (emulated world over the visible GPUs).
"""
import json
import math
import os

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
GOLDEN = os.path.join(HERE, "golden")
TOL = {"f64": 1e-12, "f32": 1e-5}


def _cases():
    with open(os.path.join(GOLDEN, "golden.json")) as f:
        return json.load(f).get("spectral", [])


CASES = _cases()


def _load(case, what):
    real = case["kind"] == "r2c"
    if case["prec"] == "f64":
        dt = np.float64 if real else np.complex128
    else:
        dt = np.float32 if real else np.complex64
    return np.fromfile(os.path.join(GOLDEN, f"{case['name']}.{what}.bin"), dtype=dt).reshape(case["dims"])


def _rel(got, want):
    got = np.asarray(got, dtype=np.complex128).ravel()
    want = np.asarray(want, dtype=np.complex128).ravel()
    return float(np.sqrt(np.sum(np.abs(got - want) ** 2) / np.sum(np.abs(want) ** 2)))


def _numpy_ops(x):
    """derivatives, laplacian of a periodic field on [0, 2 pi)^d (numpy, double)."""
    dims = x.shape
    X = np.fft.fftn(x.astype(np.complex128))
    ks = []
    for n in dims:
        k = np.fft.fftfreq(n, 1.0 / n)
        ks.append(k)
    out = {}
    div = 0
    for a, n in enumerate(dims):
        kd = ks[a].copy()
        if n % 2 == 0:
            kd[n // 2] = 0.0  # Nyquist mode zeroed for first derivatives
        shape = [1] * len(dims)
        shape[a] = n
        out[f"d{a}"] = np.fft.ifftn(1j * kd.reshape(shape) * X)
        div = div - (kd * kd).reshape(shape) * X
    k2 = sum(np.meshgrid(*[k * k for k in ks], indexing="ij"))
    out["lap"] = np.fft.ifftn(-k2 * X)
    out["div"] = np.fft.ifftn(div)  # div(grad): Nyquist modes drop out
    return out


@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_goldens_match_numpy(case):
    x = _load(case, "in")
    ref = _numpy_ops(x)
    tol = 1e-12 if case["prec"] == "f64" else 2e-6
    for a in range(len(case["dims"])):
        assert _rel(_load(case, f"d{a}"), ref[f"d{a}"]) <= tol
    assert _rel(_load(case, "lap"), ref["lap"]) <= tol
    assert _rel(_load(case, "div"), ref["div"]) <= tol
    if case["prec"] == "f64":
        # inverse_laplacian(laplacian(x)) = x - mean(x)
        assert _rel(_load(case, "ilap"), x - x.mean()) <= 1e-11


def _gpu_setup(case):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    import paper_1506_07933_b200 as D
    from gpu_util import make_plan, scatter
    dims, grid, prec = case["dims"], case["grid"], case["prec"]
    real = case["kind"] == "r2c"
    decomp = case["decomp"]
    fwd = make_plan(decomp, dims, grid, "r2c" if real else "c2c", "forward", prec)
    bwd = make_plan(decomp, dims, grid, "c2r" if real else "c2c", "backward", prec)
    ndev = torch.cuda.device_count()
    devices = list(range(min(ndev, fwd.nranks())))
    ctxs = D.make_world_contexts(fwd, devices=devices)
    return D, fwd, bwd, ctxs, devices


def _scatter_world(D, plan, arr, ctxs):
    import torch
    out = []
    for r in range(plan.nranks()):
        ext = plan.input.extents_of(r)
        sl = tuple(slice(o, o + n) for o, n in ext)
        blk = np.ascontiguousarray(arr[sl]).reshape(-1)
        out.append(D.DistTensor(plan.input, r, torch.from_numpy(blk.copy()).to(ctxs[r].device)))
    return out


def _gather_world(plan, tensors, dtype):
    arr = np.zeros(plan.output.dims, dtype=dtype)
    for r, t in enumerate(tensors):
        ext = plan.output.extents_of(r)
        sl = tuple(slice(o, o + n) for o, n in ext)
        arr[sl] = t.data.cpu().numpy().reshape(tuple(n for _, n in ext))
    return arr


@pytest.mark.gpu
@pytest.mark.parametrize("path", ["fused", "two_step"])
@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_gpu_spectral_vs_reference(case, path):
    import torch
    D, fwd, bwd, ctxs, _ = _gpu_setup(case)
    from paper_1506_07933_b200 import spectral as S
    x = _load(case, "in")
    xs = _scatter_world(D, fwd, x, ctxs)
    nd = len(case["dims"])
    P = fwd.nranks()
    lib = D._lib.lib()

    def forward_op(op, axis, inputs):
        if path == "fused":
            return S.world_forward_op(fwd, ctxs, inputs, op, axis)
        spec = D.execute_world(fwd, inputs, ctxs)
        for r in range(P):
            with torch.cuda.device(ctxs[r].device):
                D.dfft._check(lib.dfftb_spectral_apply(fwd._h, r, op, axis, None, spec[r].data.data_ptr(),
                                                       spec[r].data.data_ptr(), 0,
                                                       torch.cuda.current_stream(ctxs[r].device).cuda_stream))
        return spec

    def backward(spec):
        out = D.execute_world(bwd, spec, ctxs)
        torch.cuda.synchronize()
        return _gather_world(bwd, out, x.dtype)

    tol = TOL[case["prec"]]
    errs = {}
    grads = []
    for a in range(nd):
        spec = forward_op(S.DERIV, a, xs)
        got = backward(spec)
        grads.append(got)
        errs[f"d{a}"] = _rel(got, _load(case, f"d{a}"))
    lap = backward(forward_op(S.LAPLACIAN, 0, xs))
    errs["lap"] = _rel(lap, _load(case, "lap"))
    if case["prec"] == "f64":
        # inverse_laplacian of the REFERENCE's laplacian (same input as the golden)
        lap_ref = _scatter_world(D, fwd, _load(case, "lap"), ctxs)
        errs["ilap"] = _rel(backward(forward_op(S.INV_LAPLACIAN, 0, lap_ref)), _load(case, "ilap"))
    # divergence of the reference's gradient: accumulate i k_a (.) F(g_a)
    if path == "fused":
        gs = [_scatter_world(D, fwd, _load(case, f"d{a}"), ctxs) for a in range(nd)]
        acc = None
        for a in range(nd):
            acc = S.world_forward_op(fwd, ctxs, gs[a], S.DERIV, a, outs=acc, accumulate=acc is not None)
        errs["div"] = _rel(backward(acc), _load(case, "div"))
    for c in ctxs:
        c.close()
    print(case["name"], path, {k: f"{v:.2e}" for k, v in errs.items()})
    assert all(v <= tol for v in errs.values()), errs


@pytest.mark.gpu
def test_gpu_fused_equals_two_step_bitwise():
    """The fused epilogue and the separate multiply kernel give identical
    bits on a multi-rank grid (pencil 2x2)."""
    import torch
    case = next(c for c in CASES if c["name"] == "spec_c2c_16x8x16_pencil2x2_f64")
    D, fwd, bwd, ctxs, _ = _gpu_setup(case)
    from paper_1506_07933_b200 import spectral as S
    xs = _scatter_world(D, fwd, _load(case, "in"), ctxs)
    lib = D._lib.lib()
    for op, axis in ((S.DERIV, 0), (S.DERIV, 2), (S.LAPLACIAN, 0)):
        fused = S.world_forward_op(fwd, ctxs, xs, op, axis)
        spec = D.execute_world(fwd, xs, ctxs)
        for r in range(fwd.nranks()):
            with torch.cuda.device(ctxs[r].device):
                D.dfft._check(lib.dfftb_spectral_apply(fwd._h, r, op, axis, None, spec[r].data.data_ptr(),
                                                       spec[r].data.data_ptr(), 0,
                                                       torch.cuda.current_stream(ctxs[r].device).cuda_stream))
        torch.cuda.synchronize()
        for r in range(fwd.nranks()):
            assert torch.equal(fused[r].data.cpu(), spec[r].data.cpu()), (op, axis, r)
    for c in ctxs:
        c.close()
