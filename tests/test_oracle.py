"""Pins the C restatement (oracle/) against the unmodified reference.

The golden fixtures in tests/golden/ were produced by the reference itself
(oracle/_ref/dfft_ref, see tests/golden/make_golden.py).  CPU-only.
"""
import numpy as np
import pytest

import oracle_lib as O

CASES = O.golden_cases()


@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_oracle_reproduces_reference_goldens(case):
    x, y_ref, z_ref = O.load_golden(case)
    dims, kind, prec = case["dims"], case["kind"], case["prec"]
    # the reference's seeded input (bench.cpp:132-136) is reproduced bit-exactly
    xs = O.seeded(dims, kind == "c2c", prec)
    assert np.array_equal(xs, x)
    y, sig = O.execute(x, dims, case["decomp"], case["grid"], kind, "forward", prec)
    tol = 1e-13 if prec == "f64" else 1e-6
    assert O.rel_l2(y, y_ref) <= tol
    bk = "c2r" if kind == "r2c" else "c2c"
    z, _ = O.execute(y_ref, dims, case["decomp"], case["grid"], bk, "backward", prec)
    assert O.rel_l2(z, z_ref) <= tol


def test_oracle_bit_exact_on_pow2_f64():
    # same operation order, -ffp-contract=off: the restatement is bit-identical
    case = [c for c in CASES if c["name"] == "c2c_16x16x16_pencil2x4_f64"][0]
    x, y_ref, _ = O.load_golden(case)
    y, _ = O.execute(x, case["dims"], "pencil", [2, 4], "c2c", "forward")
    assert np.array_equal(y, y_ref)


def test_signatures():
    # test_plan.cpp:148, plan.hpp:82-98
    x = np.zeros((4, 4, 4), np.complex128)
    _, sig = O.execute(x, [4, 4, 4], "slab", [2], "c2c", "forward")
    assert sig == "F2;F1;T0x;L;F0;"
    _, sig = O.execute(x, [4, 4, 4], "pencil", [2, 2], "c2c", "forward")
    assert sig == "F2;T1;F1;T0x;L;F0;"
    _, sig = O.execute(x, [4, 4, 4], "pencil", [2, 2], "c2c", "backward")
    assert sig == "F0;T0;F1;T1;F2;N;"


def test_frozen_1d_values():
    # test_kernels.cpp:44-62
    v = np.array([1, 2, 3, 4], np.complex128)
    O.lib().oracle_fft_1d(v.ctypes.data, 4, 0)
    assert np.allclose(v, [10, -2 + 2j, -2, -2 - 2j], atol=1e-15)


def test_against_brute_force_dft():
    dims = [8, 4, 8]
    x = O.seeded(dims, True)
    y, _ = O.execute(x, dims, "pencil", [2, 2], "c2c", "forward")
    assert O.rel_l2(y, O.dft(x)) < 1e-12
    assert O.rel_l2(y, np.fft.fftn(x)) < 1e-12


def test_errors():
    x = np.zeros((4, 6, 8), np.complex128)
    with pytest.raises(O.OracleError, match="SlabTooManyRanks"):
        O.execute(x, [4, 6, 8], "slab", [5], "c2c", "forward")
    with pytest.raises(O.OracleError, match="RankTooLow"):
        O.execute(np.zeros((2, 2, 2), np.complex128), [2, 2, 2], "general", [2, 4],
                  "c2c", "forward")
    with pytest.raises(O.OracleError, match="ConfigInvalid"):
        O.execute(np.zeros((4, 4, 3), np.complex128), [4, 4, 4], "pencil", [1, 1], "r2c",
                  "backward")
    spec = np.zeros((4, 4, 3), np.complex128)
    spec[0, 0, 0] = 1.0 + 0.7j  # test_plan.cpp:392-408
    with pytest.raises(O.OracleError, match="NonHermitian"):
        O.execute(spec, [4, 4, 4], "pencil", [1, 1], "c2r", "backward")


def test_block_map_examples():
    # layout.hpp:80-92; test_layout.cpp block_map examples
    assert O.block_map(10, 4) == ([3, 3, 3, 1], [0, 3, 6, 9])
    assert O.block_map(5, 4) == ([2, 2, 1, 0], [0, 2, 4, 5])
    assert O.block_map(129, 2) == ([65, 64], [0, 65])
