"""Reference-compatible formats: DTNS tensor files (tensor_file.cpp) and the
bench report schema (report_schema.golden), plus the dfftb-bench CLI."""
import json
import os
import struct
import subprocess
import sys

import numpy as np
import pytest

import paper_1506_07933_b200 as D
from paper_1506_07933_b200 import io as IO

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN_SCHEMA = os.path.join(os.path.dirname(__file__), "golden", "report_schema.golden")


@pytest.mark.parametrize("dtype", [np.float64, np.complex128, np.float32, np.complex64])
def test_dtns_round_trip_and_header(tmp_path, dtype):
    a = (np.arange(2 * 3 * 5) * 0.5).reshape(2, 3, 5).astype(dtype)
    if np.iscomplexobj(a):
        a = a + 1j * a[::-1]
    p = tmp_path / "t.dtns"
    IO.write_tensor_file(str(p), a)
    raw = p.read_bytes()
    # tensor_file.cpp:84-92: "DTNS", u32 version, u8 kind, u32 axes, u64 dims
    assert raw[:4] == b"DTNS"
    assert struct.unpack("<IBI", raw[4:13]) == (1, int(IO.element_of(a)), 3)
    assert struct.unpack("<QQQ", raw[13:37]) == (2, 3, 5)
    assert len(raw) == 37 + a.nbytes
    b = IO.read_tensor_file(str(p))
    assert b.dtype == a.dtype and np.array_equal(np.asarray(b), a)


def test_dtns_errors(tmp_path):
    p = tmp_path / "bad.dtns"
    p.write_bytes(b"NOPE" + bytes(20))
    with pytest.raises(D.Error, match="^BadMagic"):
        IO.read_tensor_file(str(p))
    IO.write_tensor_file(str(p), np.zeros((4, 4)))
    p.write_bytes(p.read_bytes()[:-8])
    with pytest.raises(D.Error, match="^TruncatedFile"):
        IO.read_tensor_file(str(p))
    with pytest.raises(D.Error, match="^TruncatedFile"):
        IO.read_tensor_file(str(tmp_path / "missing.dtns"))


def test_complex_file_cannot_feed_real_layout(tmp_path):
    # tensor_file.hpp:63-66 (DimMismatch), as the C++ shim's read_tensor
    p = tmp_path / "c.dtns"
    IO.write_tensor_file(str(p), np.ones((4, 4, 4), dtype=np.complex128))
    plan = D.plan_pencil((4, 4, 4), (1, 1), D.TransformKind.R2C, D.Direction.Forward)
    with pytest.raises(D.Error, match="^DimMismatch: complex tensor file cannot feed a real layout"):
        IO.read_tensor(plan.input, 0, str(p))


def test_report_schema_matches_reference_golden():
    reps = [dict(zip(IO.TIMING_KEYS, [1e-3 * (i + 1)] * 6)) for i in range(3)]
    cfg = {"dims": [8, 8, 8], "grid": [2, 2], "kind": "c2c", "decomp": "pencil", "backend": "b200",
           "pipelined": False, "chunks": 1, "staging_buffers": 2, "reps": 3, "warmup": 1, "seed": 1}
    j = json.loads(IO.to_json(cfg, reps, 1e-15, ["w"]))
    ours = set(IO.schema_paths(j))
    golden = set(open(GOLDEN_SCHEMA).read().split("\n")) - {""}
    # the golden run used the cost-model backend, whose config block is extra
    golden_core = {g for g in golden if "/cost_model/" not in g}
    assert ours == golden_core
    assert j["performance"]["flops_estimate"] == 5 * 512 * 9
    assert j["verification"]["status"] == "passed"
    assert IO.flops_estimate([1024, 1024, 1024]) == 161061273600  # test_bench.cpp:38-43
    csv = IO.to_csv(reps).splitlines()
    assert csv[0] == "rep,local_fft,pack,unpack,staging_copy,wire_comm,total"
    assert csv[-2].startswith("min,1.000000000e-03")


@pytest.mark.gpu
@pytest.mark.parametrize("kind,dims", [("c2c", "8,8,8"), ("r2c", "8,8,6"), ("c2r", "8,4,8")])
def test_cli_verifies_against_direct_dft(tmp_path, kind, dims):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    out = tmp_path / "r.json"
    r = subprocess.run([sys.executable, "-m", "paper_1506_07933_b200.cli", "--dims", dims,
                        "--kind", kind, "--reps", "2", "--out", str(out)],
                       cwd=ROOT, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    j = json.loads(out.read_text())
    assert j["verification"]["status"] == "passed"
    assert j["verification"]["rel_error"] < 1e-12
    assert len(j["timings"]["reps"]) == 2


@pytest.mark.gpu
def test_cli_dtns_input_output(tmp_path):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    x = (np.random.default_rng(0).standard_normal((16, 8, 4))
         + 1j * np.random.default_rng(1).standard_normal((16, 8, 4)))
    IO.write_tensor_file(str(tmp_path / "in.dtns"), x)
    r = subprocess.run([sys.executable, "-m", "paper_1506_07933_b200.cli", "--dims", "16,8,4",
                        "--input", str(tmp_path / "in.dtns"), "--output", str(tmp_path / "out.dtns"),
                        "--reps", "1", "--format", "csv"],
                       cwd=ROOT, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    assert r.stdout.startswith("rep,local_fft")
    y = np.asarray(IO.read_tensor_file(str(tmp_path / "out.dtns")))
    assert np.max(np.abs(y - np.fft.fftn(x))) < 1e-12 * np.max(np.abs(y))
