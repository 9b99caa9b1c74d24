"""Generate golden fixtures from the UNMODIFIED reference (test infrastructure).

Runs oracle/_ref/dfft_ref (the reference dfft artifact compiled from
/root/reference/proj by oracle/Makefile, driven through its public
plan/execute API by oracle/ref_driver.cpp) on small seeded configurations and
stores the global input, forward spectrum and backward(forward(x)) round trip
as raw little-endian arrays next to this script, indexed by golden.json.

Spectral goldens (SPECTRAL_CASES): the reference's derivative / laplacian /
inverse_laplacian / divergence (spectral.hpp:131-309) of the seeded field
through make_spectral_context (ref_driver --spectral), stored as
<name>.{in,d0..d(n-1),lap,ilap,div}.bin.

Re-run with:  make -C oracle ref && python tests/golden/make_golden.py [--spectral-only]
"""
import json
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
REF = os.path.join(ROOT, "oracle", "_ref", "dfft_ref")

# name, dims, decomp, grid, kind, prec
CASES = [
    ("c2c_4x4x4_slab1_f64", [4, 4, 4], "slab", [1], "c2c", "f64"),
    ("c2c_8x8x8_pencil2x2_f64", [8, 8, 8], "pencil", [2, 2], "c2c", "f64"),
    ("c2c_16x8x4_slab4_f64", [16, 8, 4], "slab", [4], "c2c", "f64"),
    ("c2c_16x16x16_pencil2x4_f64", [16, 16, 16], "pencil", [2, 4], "c2c", "f64"),
    ("c2c_32x16x8_pencil4x2_f64", [32, 16, 8], "pencil", [4, 2], "c2c", "f64"),
    ("r2c_16x16x16_slab2_f64", [16, 16, 16], "slab", [2], "r2c", "f64"),
    ("r2c_32x16x8_pencil2x2_f64", [32, 16, 8], "pencil", [2, 2], "r2c", "f64"),
    ("r2c_8x8x16_slab8_f64", [8, 8, 16], "slab", [8], "r2c", "f64"),
    ("c2c_8x8x8_pencil4x2_f32", [8, 8, 8], "pencil", [4, 2], "c2c", "f32"),
    ("r2c_32x16x8_pencil2x2_f32", [32, 16, 8], "pencil", [2, 2], "r2c", "f32"),
    ("r2c_16x8x32_pencil2x1_f32", [16, 8, 32], "pencil", [2, 1], "r2c", "f32"),
    # non-power-of-two / ragged cases pin the oracle's mixed-radix, Bluestein
    # and empty-tail paths (the GPU path rejects non-pow-2 lengths for now)
    ("c2c_6x6x6_pencil3x2_f64", [6, 6, 6], "pencil", [3, 2], "c2c", "f64"),
    ("c2c_5x5x5_pencil1x4_f64", [5, 5, 5], "pencil", [1, 4], "c2c", "f64"),
    ("r2c_8x4x6_pencil2x2_f64", [8, 4, 6], "pencil", [2, 2], "r2c", "f64"),
    ("r2c_8x8x7_pencil2x2_f64", [8, 8, 7], "pencil", [2, 2], "r2c", "f64"),
    ("c2c_17x4x4_slab3_f64", [17, 4, 4], "slab", [3], "c2c", "f64"),
    ("c2c_12x10x12_slab4_f64", [12, 10, 12], "slab", [4], "c2c", "f64"),
    # general (d-1)-D decomposition of 4-D tensors (plan.hpp:253-262, test_plan.cpp:243-248)
    ("c2c_8x6x4x4_general2x2x2_f64", [8, 6, 4, 4], "general", [2, 2, 2], "c2c", "f64"),
    ("r2c_8x8x4x8_general2x2x2_f64", [8, 8, 4, 8], "general", [2, 2, 2], "r2c", "f64"),
    ("c2c_16x8x8x4_general2x1x2_f32", [16, 8, 8, 4], "general", [2, 1, 2], "c2c", "f32"),
]


# spectral operators: name, dims, grid (pencil / general by its length), kind, prec
SPECTRAL_CASES = [
    ("spec_c2c_16x8x16_pencil2x2_f64", [16, 8, 16], [2, 2], "c2c", "f64"),
    ("spec_r2c_16x8x16_pencil2x2_f64", [16, 8, 16], [2, 2], "r2c", "f64"),
    ("spec_c2c_16x16x16_pencil1x1_f64", [16, 16, 16], [1, 1], "c2c", "f64"),
    ("spec_r2c_32x16x8_pencil1x1_f32", [32, 16, 8], [1, 1], "r2c", "f32"),
    ("spec_c2c_8x4x8x8_general2x1x2_f64", [8, 4, 8, 8], [2, 1, 2], "c2c", "f64"),
    ("spec_r2c_8x8x4x8_general2x2x1_f64", [8, 8, 4, 8], [2, 2, 1], "r2c", "f64"),
]


def spectral(index_path):
    with open(index_path) as f:
        idx = json.load(f)
    out = []
    for name, dims, grid, kind, prec in SPECTRAL_CASES:
        prefix = os.path.join(HERE, name)
        cmd = [REF, "--dims", ",".join(map(str, dims)), "--grid", ",".join(map(str, grid)),
               "--kind", kind, "--prec", prec, "--seed", "1", "--spectral", "--dump", prefix]
        subprocess.run(cmd, check=True, capture_output=True, text=True)
        out.append({"name": name, "dims": dims, "grid": grid, "kind": kind, "prec": prec, "seed": 1,
                    "decomp": "pencil" if len(grid) == 2 else "general"})
        print(name)
    idx["spectral"] = out
    with open(index_path, "w") as f:
        json.dump(idx, f, indent=1)


def main():
    if not os.path.exists(REF):
        sys.exit("build the reference first: make -C oracle ref")
    if "--spectral-only" in sys.argv:
        spectral(os.path.join(HERE, "golden.json"))
        return
    index = []
    for name, dims, decomp, grid, kind, prec in CASES:
        prefix = os.path.join(HERE, name)
        cmd = [REF, "--dims", ",".join(map(str, dims)), "--decomp", decomp,
               "--grid", ",".join(map(str, grid)), "--kind", kind, "--prec", prec,
               "--seed", "1", "--warmup", "0", "--reps", "1", "--dump", prefix]
        out = subprocess.run(cmd, check=True, capture_output=True, text=True).stdout
        rep = json.loads(out.strip().splitlines()[-1])
        index.append({"name": name, "dims": dims, "decomp": decomp, "grid": grid,
                      "kind": kind, "prec": prec, "seed": 1,
                      "ref_roundtrip_rel_l2": rep["roundtrip_rel_l2"]})
        print(name, rep["roundtrip_rel_l2"])
    with open(os.path.join(HERE, "golden.json"), "w") as f:
        json.dump({"generator": "tests/golden/make_golden.py via oracle/_ref/dfft_ref",
                   "cases": index}, f, indent=1)
    spectral(os.path.join(HERE, "golden.json"))


if __name__ == "__main__":
    main()
