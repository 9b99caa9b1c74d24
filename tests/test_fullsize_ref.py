"""Full-size parity against the UNMODIFIED reference at the BASELINE grids.

The reference (oracle/_ref/dfft_ref: the reference's own sources compiled by
oracle/Makefile, driven through its public plan/execute API by
oracle/ref_driver.cpp) runs on the host cores with one rank thread per grid
rank and dumps the global input, forward spectrum and round trip
(bench.cpp:132-136 seeded field).  The B200 path runs the same plans as an
emulated world of the same rank count over the visible GPUs (exchange
stores cross NVLink when there are several), and is compared at rel-L2
<= 1e-12 (fp64) / 1e-5 (fp32) (BASELINE.json north_star):
  * input bit-identical to the reference's (device-generated seeded field),
  * forward spectrum vs the reference's forward spectrum,
  * backward(reference spectrum) vs the reference's round trip,
  * our own round trip vs the input.

Configurations: C 512^3 C2C fp64 pencil 2x4, E 2048x512x256
R2C fp32 pencil 4x2, B 256^3 R2C fp64 slab 8.  D (1024^3 C2C fp64 pencil
4x2, ~92 GiB of host RAM for the reference) runs with DFFTB_TEST_HUGE=1.
"""
import json
import os
import shutil
import subprocess
import tempfile
import time

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
REF = os.path.join(ROOT, "oracle", "_ref", "dfft_ref")
TOL = {"f64": 1e-12, "f32": 1e-5}

pytestmark = pytest.mark.gpu

CASES = [
    ("B_256c_r2c_f64_slab8", [256, 256, 256], "slab", [8], "r2c", "f64"),
    ("C_512c_c2c_f64_pencil2x4", [512, 512, 512], "pencil", [2, 4], "c2c", "f64"),
    ("E_2048x512x256_r2c_f32_pencil4x2", [2048, 512, 256], "pencil", [4, 2], "r2c", "f32"),
]
HUGE = [("D_1024c_c2c_f64_pencil4x2", [1024, 1024, 1024], "pencil", [4, 2], "c2c", "f64")]


def _chunked_rel(got, want, chunk=1 << 24):
    """sqrt(sum |got - want|^2 / sum |want|^2) in double, without full-size temporaries."""
    g = got.reshape(-1)
    w = want.reshape(-1)
    num = den = 0.0
    for i in range(0, g.size, chunk):
        a = g[i:i + chunk].astype(np.complex128)
        b = w[i:i + chunk].astype(np.complex128)
        num += float(np.sum(np.abs(a - b) ** 2))
        den += float(np.sum(np.abs(b) ** 2))
    return float(np.sqrt(num / den))


def _run(case, tmp):
    import torch
    import paper_1506_07933_b200 as D
    from gpu_util import make_plan

    name, dims, decomp, grid, kind, prec = case
    if not os.path.exists(REF):
        pytest.skip("oracle/_ref/dfft_ref not built")
    prefix = os.path.join(tmp, name)
    t0 = time.time()
    cmd = [REF, "--dims", ",".join(map(str, dims)), "--decomp", decomp, "--grid", ",".join(map(str, grid)),
           "--kind", kind, "--prec", prec, "--seed", "1", "--warmup", "0", "--reps", "1", "--dump", prefix]
    rep = json.loads(subprocess.run(cmd, check=True, capture_output=True, text=True).stdout.strip().splitlines()[-1])
    t_ref = time.time() - t0

    real = kind == "r2c"
    dt_r = np.float64 if prec == "f64" else np.float32
    dt_c = np.complex128 if prec == "f64" else np.complex64
    fwd = make_plan(decomp, dims, grid, "r2c" if real else "c2c", "forward", prec)
    bwd = make_plan(decomp, dims, grid, "c2r" if real else "c2c", "backward", prec)
    P = fwd.nranks()
    ndev = torch.cuda.device_count()
    devices = list(range(min(ndev, P)))
    ctxs = D.make_world_contexts(fwd, devices=devices)
    xs = [D.DistTensor.seeded(fwd.input, r, seed=1, complex_field=not real, device=ctxs[r].device)
          for r in range(P)]

    def gather(plan, ts, dtype, side="output"):
        dist_ = plan.output if side == "output" else plan.input
        arr = np.empty(dist_.dims, dtype=dtype)
        for r, t in enumerate(ts):
            ext = dist_.extents_of(r)
            sl = tuple(slice(o, o + n) for o, n in ext)
            arr[sl] = t.data.cpu().numpy().reshape(tuple(n for _, n in ext))
        return arr

    def scatter(plan, arr):
        out = []
        for r in range(P):
            ext = plan.input.extents_of(r)
            sl = tuple(slice(o, o + n) for o, n in ext)
            blk = np.ascontiguousarray(arr[sl]).reshape(-1)
            out.append(D.DistTensor(plan.input, r, torch.from_numpy(blk).to(ctxs[r].device)))
        return out

    x_ref = np.fromfile(prefix + ".in.bin", dtype=dt_r if real else dt_c).reshape(dims)
    assert np.array_equal(gather(fwd, xs, x_ref.dtype, "input"), x_ref), "seeded input differs from the reference's"
    t1 = time.time()
    ys = D.execute_world(fwd, xs, ctxs)
    torch.cuda.synchronize()
    y = gather(fwd, ys, dt_c)
    del ys
    y_ref = np.fromfile(prefix + ".fwd.bin", dtype=dt_c).reshape(y.shape)
    e_fwd = _chunked_rel(y, y_ref)
    del y
    zs = D.execute_world(bwd, scatter(bwd, y_ref), ctxs)
    torch.cuda.synchronize()
    z = gather(bwd, zs, x_ref.dtype)
    del zs
    z_ref = np.fromfile(prefix + ".rt.bin", dtype=x_ref.dtype).reshape(dims)
    e_bwd = _chunked_rel(z, z_ref)
    del z, y_ref, z_ref
    # our own round trip
    zs = D.execute_world(bwd, D.execute_world(fwd, xs, ctxs), ctxs)
    torch.cuda.synchronize()
    e_rt = _chunked_rel(gather(bwd, zs, x_ref.dtype), x_ref)
    t_gpu = time.time() - t1
    for c in ctxs:
        c.close()
    line = {"case": name, "ranks": P, "gpus": len(devices), "fwd_vs_ref": e_fwd, "bwd_vs_ref_roundtrip": e_bwd,
            "roundtrip": e_rt, "ref_roundtrip": rep["roundtrip_rel_l2"], "ref_seconds": round(t_ref, 1),
            "gpu_check_seconds": round(t_gpu, 1)}
    print(json.dumps(line))
    tol = TOL[prec]
    assert e_fwd <= tol and e_bwd <= tol and e_rt <= tol, line


@pytest.fixture
def tmpdir_big():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    base = os.environ.get("DFFTB_TEST_TMP")
    d = tempfile.mkdtemp(prefix="dfftb_ref_", dir=base)
    yield d
    shutil.rmtree(d, ignore_errors=True)


@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_fullsize_vs_reference(case, tmpdir_big):
    _run(case, tmpdir_big)


@pytest.mark.parametrize("case", HUGE, ids=[c[0] for c in HUGE])
def test_fullsize_vs_reference_huge(case, tmpdir_big):
    if os.environ.get("DFFTB_TEST_HUGE") != "1":
        pytest.skip("set DFFTB_TEST_HUGE=1 (needs ~100 GiB host RAM and disk)")
    _run(case, tmpdir_big)
