"""Seeded random configurations (the reference's acceptance sweep idea,
acceptance.cpp:173-189, widened): random axis lengths (powers of two, smooth
and prime), decompositions, grids up to 8 ranks, kinds and precisions, each
through the emulated world on one GPU against the C oracle, both directions
plus the round trip.  Deterministic: the case list is drawn once from a fixed
seed."""
import random

import pytest

import oracle_lib as O
from gpu_util import make_plan, rel_l2, run_world

pytestmark = pytest.mark.gpu

TOL = {"f64": 1e-12, "f32": 1e-5}
LENGTHS = [1, 2, 3, 4, 5, 6, 7, 8, 9, 12, 13, 16, 17, 24, 31, 32, 48, 64]


def _cases(n=40, seed=20261018):
    rng = random.Random(seed)
    out = []
    while len(out) < n:
        decomp = rng.choice(["slab", "pencil", "pencil", "general"])
        nd = 4 if decomp == "general" else 3
        dims = [rng.choice(LENGTHS) for _ in range(nd)]
        kind = rng.choice(["c2c", "r2c"])
        prec = rng.choice(["f64", "f64", "f32"])
        if kind == "r2c" and dims[-1] < 2:
            continue
        if decomp == "slab":
            grid = [rng.choice([1, 2, 3, 4, 8])]
            if grid[0] > dims[0]:
                continue  # SlabTooManyRanks (covered by the error tests)
        elif decomp == "pencil":
            grid = [rng.choice([1, 2, 4]), rng.choice([1, 2])]
        else:
            grid = [rng.choice([1, 2]), rng.choice([1, 2]), 1]
        if any(g > 1 and d < 2 for g, d in zip(grid, dims)):
            continue
        out.append((decomp, dims, grid, kind, prec))
    return out


CASES = _cases()


@pytest.mark.parametrize("decomp,dims,grid,kind,prec", CASES,
                         ids=["-".join([c[0], "x".join(map(str, c[1])), "x".join(map(str, c[2])), c[3], c[4]])
                              for c in CASES])
def test_random_configuration_against_oracle(decomp, dims, grid, kind, prec):
    x = O.seeded(dims, kind == "c2c", prec)
    try:
        y_ref, sig = O.execute(x, dims, decomp, grid, kind, "forward", prec)
    except Exception as e:  # configurations the reference itself rejects
        pytest.skip(f"reference rejects: {e}")
    fwd = make_plan(decomp, dims, grid, kind, "forward", prec)
    assert fwd.signature() == sig
    y = run_world(fwd, x)
    assert rel_l2(y, y_ref) <= TOL[prec]
    bk = "c2r" if kind == "r2c" else "c2c"
    z_ref, _ = O.execute(y_ref, dims, decomp, grid, bk, "backward", prec)
    bwd = make_plan(decomp, dims, grid, bk, "backward", prec)
    z = run_world(bwd, y_ref)
    assert rel_l2(z, z_ref) <= TOL[prec]
