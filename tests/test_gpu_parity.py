"""GPU parity: the B200 path (libdfftb.so, through the C ABI) against the
reference's own outputs (tests/golden/, produced by the unmodified reference)
and against the C restatement (oracle/) on identical seeded inputs.

Tolerances (BASELINE.json north_star): rel-L2 <= 1e-12 fp64, <= 1e-5 fp32.
Multi-rank grids run as an emulated world on one GPU (every rank's fused
FFT + exchange kernels, lockstep on one stream); the real multi-process
NVLink path is covered by tests/test_multigpu.py.
"""
import numpy as np
import pytest
import torch

import oracle_lib as O
import paper_1506_07933_b200 as D
from gpu_util import gather, is_pow2, make_plan, rel_l2, run_world, scatter

pytestmark = pytest.mark.gpu

TOL = {"f64": 1e-12, "f32": 1e-5}
POW2_CASES = O.golden_cases()  # all reference goldens, incl. non-power-of-two lengths


@pytest.fixture(autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")


@pytest.mark.parametrize("case", POW2_CASES, ids=[c["name"] for c in POW2_CASES])
def test_against_reference_goldens(case):
    x, y_ref, z_ref = O.load_golden(case)
    dims, kind, prec, grid = case["dims"], case["kind"], case["prec"], case["grid"]
    fwd = make_plan(case["decomp"], dims, grid, kind, "forward", prec)
    y = run_world(fwd, x)
    assert rel_l2(y, y_ref) <= TOL[prec]
    bk = "c2r" if kind == "r2c" else "c2c"
    bwd = make_plan(case["decomp"], dims, grid, bk, "backward", prec)
    z = run_world(bwd, y_ref)
    assert rel_l2(z, z_ref) <= TOL[prec]


ORACLE_CASES = [
    # config A: 64^3 C2C fp64 single-rank slab
    ("slab", [64, 64, 64], [1], "c2c", "f64"),
    ("pencil", [64, 32, 128], [2, 2], "c2c", "f64"),
    ("pencil", [32, 64, 64], [2, 4], "c2c", "f64"),
    ("pencil", [64, 64, 32], [4, 2], "c2c", "f64"),
    ("slab", [64, 32, 32], [8], "r2c", "f64"),
    ("pencil", [128, 64, 32], [2, 2], "r2c", "f32"),
    ("pencil", [64, 32, 256], [4, 2], "r2c", "f32"),   # 129 bins over 2: 65/64 blocks
    ("slab", [32, 1024, 16], [4], "c2c", "f64"),
    ("pencil", [2048, 16, 8], [2, 2], "c2c", "f32"),
    ("slab", [16, 16, 4096], [1], "c2c", "f64"),
    ("pencil", [8, 8, 8], [8, 1], "c2c", "f64"),
    ("pencil", [8, 8, 8], [1, 8], "c2c", "f64"),
    ("pencil", [4, 4, 4], [4, 2], "r2c", "f64"),      # empty tail blocks
    ("slab", [4, 2, 2], [3], "c2c", "f64"),           # ragged slab, empty-ish tails
    # single rank, long strided axes: pair-interleaved buffers (narrow tiles)
    ("pencil", [1024, 16, 8], [1, 1], "c2c", "f64"),
    ("pencil", [16, 1024, 8], [1, 1], "c2c", "f64"),
    ("pencil", [2048, 8, 32], [1, 1], "r2c", "f32"),
    ("pencil", [8, 2048, 16], [1, 1], "c2c", "f32"),
]


@pytest.mark.parametrize("decomp,dims,grid,kind,prec", ORACLE_CASES,
                         ids=["-".join(map(str, [c[0], "x".join(map(str, c[1])),
                                                 "x".join(map(str, c[2])), c[3], c[4]]))
                              for c in ORACLE_CASES])
def test_against_oracle(decomp, dims, grid, kind, prec):
    x = O.seeded(dims, kind == "c2c", prec)
    y_ref, sig = O.execute(x, dims, decomp, grid, kind, "forward", prec)
    fwd = make_plan(decomp, dims, grid, kind, "forward", prec)
    assert fwd.signature() == sig
    y = run_world(fwd, x)
    assert rel_l2(y, y_ref) <= TOL[prec]
    bk = "c2r" if kind == "r2c" else "c2c"
    z_ref, sig_b = O.execute(y_ref, dims, decomp, grid, bk, "backward", prec)
    bwd = make_plan(decomp, dims, grid, bk, "backward", prec)
    assert bwd.signature() == sig_b
    z = run_world(bwd, y_ref)
    assert rel_l2(z, z_ref) <= TOL[prec]
    assert rel_l2(z, x) <= (1e-13 if prec == "f64" else 1e-5)  # round trip


def test_seeded_fill_matches_reference_field():
    dims = [16, 8, 32]
    for kind, cf in (("c2c", True), ("r2c", False)):
        plan = make_plan("pencil", dims, [2, 2], kind, "forward")
        xs = [D.DistTensor.seeded(plan.input, r, seed=1, complex_field=cf) for r in range(4)]
        got = gather(plan.input, xs)
        assert np.array_equal(got, O.seeded(dims, cf))


def test_single_rank_context_and_execute():
    dims = [32, 16, 64]
    plan = make_plan("pencil", dims, [1, 1], "c2c", "forward")
    ctx = D.make_context(plan)
    x = D.DistTensor.seeded(plan.input, 0)
    y = D.execute(plan, x, ctx)
    want = np.fft.fftn(O.seeded(dims, True))
    assert rel_l2(y.data.cpu().numpy().reshape(dims), want) < 1e-12
    tb = D.TimingBreakdown()
    D.execute(plan, x, ctx, timers=tb)
    assert tb.total > 0 and tb.local_fft > 0


def test_unnormalized_round_trip_scales_by_n():
    # test_plan.cpp:116-133
    dims = [16, 16, 16]
    x = O.seeded(dims, True)
    fwd = make_plan("slab", dims, [4], "c2c", "forward", normalize=False)
    bwd = make_plan("slab", dims, [4], "c2c", "backward", normalize=False)
    back = run_world(bwd, run_world(fwd, x))
    assert np.max(np.abs(back - 4096 * x)) < 1e-10


def test_delta_transforms_to_ones():
    dims = [8, 8, 8]
    x = np.zeros(dims, np.complex128)
    x[0, 0, 0] = 1
    y = run_world(make_plan("pencil", dims, [2, 2], "c2c", "forward"), x)
    assert np.max(np.abs(y - 1)) < 1e-12


def test_zero_stays_zero():
    for kind in ("c2c", "r2c"):
        dims = [4, 4, 4]
        x = np.zeros(dims, np.complex128 if kind == "c2c" else np.float64)
        y = run_world(make_plan("pencil", dims, [2, 2], kind, "forward"), x)
        assert np.all(y == 0)


def test_layout_mismatch():
    plan = make_plan("pencil", [4, 4, 4], [1, 1], "c2c", "forward")
    ctx = D.make_context(plan)
    x = D.DistTensor.zeros(plan.output, 0)
    wrong = D.DistTensor(D.Distribution((4, 4, 4), plan.grid, (1, 2), (True,) * 3,
                                        D.ElementKind.Complex, plan, 1), 0, x.data)
    with pytest.raises(D.Error, match="LayoutMismatch"):
        D.execute(plan, wrong, ctx)


def test_non_hermitian_rejected():
    # test_plan.cpp:392-408
    plan = make_plan("pencil", [4, 4, 4], [1, 1], "c2r", "backward")
    ctx = D.make_context(plan)
    spec = D.DistTensor.zeros(plan.input, 0)
    spec.data[0] = 1.0 + 0.7j
    with pytest.raises(D.Error, match="NonHermitian"):
        D.execute(plan, spec, ctx)


def test_validate_finite_is_opt_in():
    plan = make_plan("pencil", [2, 2, 2], [1, 1], "c2c", "forward", validate_finite=True)
    ctx = D.make_context(plan)
    x = D.DistTensor.zeros(plan.input, 0)
    x.data[3] = complex(float("nan"), 0)
    with pytest.raises(D.Error, match="non-finite"):
        D.execute(plan, x, ctx)
    plan2 = make_plan("pencil", [2, 2, 2], [1, 1], "c2c", "forward")
    D.execute(plan2, x, D.make_context(plan2))  # no error without the option


def test_unsupported_length_fails_loudly():
    # prime 2053: Bluestein would need a 8192-point fp64 convolution per lane
    plan = make_plan("pencil", [2053, 2, 2], [1, 1], "c2c", "forward")
    with pytest.raises(D.Error, match="Unsupported"):
        D.make_context(plan)
    plan = make_plan("pencil", [8192, 2, 2], [1, 1], "c2c", "forward")
    with pytest.raises(D.Error, match="Unsupported"):
        D.make_context(plan)


GENERIC_CASES = [
    # non-power-of-two lengths: mixed radix (13-smooth) and Bluestein (kernels.hpp:143-293)
    ("pencil", [6, 6, 6], [3, 2], "c2c", "f64"),        # test_plan.cpp:276-281
    ("pencil", [5, 5, 5], [1, 4], "c2c", "f64"),        # empty tails
    ("slab", [17, 4, 4], [3], "c2c", "f64"),            # prime -> Bluestein
    ("slab", [12, 10, 12], [4], "c2c", "f64"),
    ("pencil", [8, 8, 7], [2, 2], "r2c", "f64"),        # odd last axis
    ("pencil", [8, 4, 6], [2, 2], "r2c", "f64"),
    ("pencil", [30, 18, 20], [2, 3], "r2c", "f32"),
    ("slab", [96, 120, 64], [4], "c2c", "f64"),
    ("pencil", [2, 3, 1000], [1, 1], "r2c", "f64"),     # 1000 = 8*125
    ("pencil", [4, 2, 1021], [1, 1], "c2c", "f64"),     # prime 1021 -> Bluestein m=2048
    ("pencil", [3, 2, 509], [1, 1], "r2c", "f32"),      # prime R2C/C2R fp32
    ("slab", [11, 13, 6], [2], "c2c", "f32"),
]


@pytest.mark.parametrize("decomp,dims,grid,kind,prec", GENERIC_CASES,
                         ids=["-".join(map(str, [c[0], "x".join(map(str, c[1])),
                                                 "x".join(map(str, c[2])), c[3], c[4]]))
                              for c in GENERIC_CASES])
def test_generic_lengths_against_oracle(decomp, dims, grid, kind, prec):
    test_against_oracle(decomp, dims, grid, kind, prec)


def test_context_reused_for_forward_and_backward():
    dims = [32, 32, 32]
    fwd = make_plan("slab", dims, [1], "r2c", "forward")
    bwd = make_plan("slab", dims, [1], "c2r", "backward")
    ctx = D.make_context(fwd)
    x = D.DistTensor.seeded(fwd.input, 0, complex_field=False)
    z = D.execute_r2c_c2r_roundtrip(fwd, bwd, x, ctx)
    assert rel_l2(z.data.cpu().numpy(), x.data.cpu().numpy()) < 1e-14


def test_512_cubed_single_gpu_properties():
    # BASELINE-size checks through size-independent properties: round trip,
    # Parseval, and direct-DFT spot bins of the seeded field.
    dims = [512, 512, 512]
    fwd = make_plan("slab", dims, [1], "c2c", "forward")
    bwd = make_plan("slab", dims, [1], "c2c", "backward")
    ctx = D.make_context(fwd)
    x = D.DistTensor.seeded(fwd.input, 0)
    y = D.execute(fwd, x, ctx)
    z = D.execute(bwd, y, ctx)
    xd = x.data
    rt = (torch.linalg.vector_norm(z.data - xd) / torch.linalg.vector_norm(xd)).item()
    assert rt < 1e-14
    n = xd.numel()
    space = torch.sum(torch.abs(xd) ** 2).item()
    freq = torch.sum(torch.abs(y.data) ** 2).item()
    assert abs(n * space - freq) <= 1e-12 * freq
    # spot bins against a direct sum in double over the whole volume
    xg = xd.view(dims)
    yb = y.data.view(dims)
    for k in [(0, 0, 0), (1, 2, 3), (511, 17, 256), (100, 300, 7)]:
        ph = [torch.exp(-2j * np.pi * torch.arange(512, device=xd.device, dtype=torch.float64) *
                        k[a] / 512) for a in range(3)]
        val = torch.einsum("ijk,i,j,k->", xg, ph[0], ph[1], ph[2]).item()
        assert abs(yb[k].item() - val) <= 1e-10 * np.sqrt(freq / n)


def _spot_bins(xg, yb, dims, bins, half_last=False):
    """Largest |y[k] - direct double DFT sum| over the given bins, and the
    RMS spectrum magnitude for scale."""
    dev = xg.device
    worst = 0.0
    for k in bins:
        ph = [torch.exp(-2j * np.pi * torch.arange(dims[a], device=dev, dtype=torch.float64) * k[a] / dims[a])
              for a in range(3)]
        val = torch.einsum("ijk,i,j,k->", xg.to(torch.complex128), ph[0], ph[1], ph[2]).item()
        worst = max(worst, abs(complex(yb[k].item()) - val))
    return worst


def test_config_D_1024_cubed_properties():
    # BASELINE config D (1024^3 C2C fp64) at full size on one GPU: round trip,
    # Parseval and direct-DFT spot bins (the oracle would need ~92 GB of RAM)
    dims = [1024, 1024, 1024]
    fwd = make_plan("pencil", dims, [1, 1], "c2c", "forward")
    bwd = make_plan("pencil", dims, [1, 1], "c2c", "backward")
    ctx = D.make_context(fwd)
    x = D.DistTensor.seeded(fwd.input, 0)
    y = D.execute(fwd, x, ctx)
    z = D.execute(bwd, y, ctx)
    xd = x.data
    assert (torch.linalg.vector_norm(z.data - xd) / torch.linalg.vector_norm(xd)).item() < 1e-14
    del z
    n = xd.numel()
    space = torch.sum(torch.abs(xd) ** 2).item()
    freq = torch.sum(torch.abs(y.data) ** 2).item()
    assert abs(n * space - freq) <= 1e-12 * freq
    err = _spot_bins(xd.view(dims), y.data.view(dims), dims, [(0, 0, 0), (1023, 5, 512), (300, 700, 9)])
    assert err <= 1e-10 * np.sqrt(freq / n)
    ctx.close()


def test_config_E_r2c_f32_properties():
    # BASELINE config E (2048x512x256 R2C -> C2R fp32) at full size: round trip
    # within the fp32 tolerance and spot bins against a double direct sum
    dims = [2048, 512, 256]
    fwd = make_plan("pencil", dims, [1, 1], "r2c", "forward", "f32")
    bwd = make_plan("pencil", dims, [1, 1], "c2r", "backward", "f32")
    ctx = D.make_context(fwd)
    x = D.DistTensor.seeded(fwd.input, 0, complex_field=False)
    y = D.execute(fwd, x, ctx)
    z = D.execute(bwd, y, ctx)
    xd = x.data
    assert (torch.linalg.vector_norm(z.data - xd) / torch.linalg.vector_norm(xd)).item() < 1e-5
    hd = [2048, 512, 129]
    yb = y.data.view(hd)
    n = xd.numel()
    rms = np.sqrt(n * torch.sum(xd.double() ** 2).item())  # |X| scale (Parseval)
    err = _spot_bins(xd.view(dims), yb, dims, [(0, 0, 0), (2047, 3, 128), (1000, 255, 77)])
    assert err <= 1e-5 * rms / np.sqrt(n) * 10
    ctx.close()


def test_config_B_256_r2c_against_oracle():
    # BASELINE config B (256^3 R2C f64, slab P=1) against the C oracle at full size
    dims = [256, 256, 256]
    xg = O.seeded(dims, False, "f64")
    y_ref, _ = O.execute(xg, dims, "slab", [1], "r2c", "forward", "f64")
    fwd = make_plan("slab", dims, [1], "r2c", "forward")
    y = run_world(fwd, xg)
    assert rel_l2(y, y_ref) <= 1e-12


def test_general_4d_repeated_executes_stay_exact():
    # a 4-D general plan has three transposes -> three exchange slots per
    # execute parity; repeated executes (both parities) must agree bitwise
    # with the first and with the oracle (regression: the third slot once
    # ran past the shared region on odd executes)
    dims = [8, 8, 16, 16]
    fwd = make_plan("general", dims, [1, 1, 1], "c2c", "forward")
    bwd = make_plan("general", dims, [1, 1, 1], "c2c", "backward")
    ctx = D.make_context(fwd)
    x = D.DistTensor.seeded(fwd.input, 0)
    y0 = D.execute(fwd, x, ctx).data.clone()
    for _ in range(4):
        y = D.execute(fwd, x, ctx)
        z = D.execute(bwd, y, ctx)
        ctx.check()
        assert torch.equal(y.data, y0)
        assert rel_l2(z.data.cpu().numpy(), x.data.cpu().numpy()) < 1e-14
    xg = O.seeded(dims, True, "f64")
    y_ref, _ = O.execute(xg, dims, "general", [1, 1, 1], "c2c", "forward", "f64")
    assert rel_l2(y0.cpu().numpy().reshape(dims), y_ref) <= 1e-12
