"""ctypes binding of oracle/liboracle.so — TEST INFRASTRUCTURE (the checker).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg import
this module.  The product package never does.
"""
import ctypes
import os
import subprocess

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_DIR = os.path.join(ROOT, "oracle")
_LIB = None

KINDS = {"c2c": 0, "r2c": 1, "c2r": 2}
DECOMPS = {"slab": 0, "pencil": 1, "general": 2}


def lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(ORACLE_DIR, "liboracle.so")
        if not os.path.exists(path):
            subprocess.run(["make", "-C", ORACLE_DIR, "liboracle.so"], check=True,
                           capture_output=True)
        L = ctypes.CDLL(path)
        i64p = ctypes.POINTER(ctypes.c_int64)
        ip = ctypes.POINTER(ctypes.c_int)
        L.oracle_execute.argtypes = [ctypes.c_int, ctypes.c_int, i64p, ctypes.c_int,
                                     ctypes.c_int, ip, ctypes.c_int, ctypes.c_int,
                                     ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p,
                                     ctypes.c_char_p]
        L.oracle_local_extents.argtypes = [ctypes.c_int, i64p, ctypes.c_int, ctypes.c_int,
                                           ip, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                           ctypes.c_int, i64p, i64p]
        L.oracle_block_map.argtypes = [ctypes.c_int64, ctypes.c_int, i64p, i64p]
        L.oracle_seeded.argtypes = [ctypes.c_uint64, ctypes.c_int64, ctypes.c_int]
        L.oracle_seeded.restype = ctypes.c_double
        L.oracle_seeded_fill.argtypes = [ctypes.c_uint64, ctypes.c_int64, ctypes.c_int,
                                         ctypes.c_int, ctypes.c_void_p]
        L.oracle_dft.argtypes = [ctypes.c_void_p, ctypes.c_int, i64p, ctypes.c_int,
                                 ctypes.c_void_p]
        L.oracle_fft_1d.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int]
        _LIB = L
    return _LIB


def _i64(v):
    return (ctypes.c_int64 * len(v))(*v)


def _int(v):
    return (ctypes.c_int * len(v))(*v)


def hat(dims, kind):
    d = list(dims)
    if kind in ("r2c", "c2r"):
        d[-1] = d[-1] // 2 + 1
    return d


def seeded(dims, complex_field, prec="f64", seed=1):
    n = int(np.prod(dims))
    dt = np.float64 if prec == "f64" else np.float32
    out = np.empty(n * (2 if complex_field else 1), dtype=dt)
    lib().oracle_seeded_fill(seed, n, 1 if complex_field else 0, 8 if prec == "f64" else 4,
                             out.ctypes.data)
    if complex_field:
        out = out.view(np.complex128 if prec == "f64" else np.complex64)
    return out.reshape(dims)


def execute(x, dims, decomp, grid, kind, direction, prec="f64", normalize=True):
    """Global in -> global out through the restated distributed plan."""
    dt_r = np.float64 if prec == "f64" else np.float32
    dt_c = np.complex128 if prec == "f64" else np.complex64
    fwd = direction == "forward"
    if kind == "r2c" or (kind == "c2r" and not fwd):
        pass
    if fwd:
        in_dt = dt_r if kind == "r2c" else dt_c
        out_shape, out_dt = hat(dims, kind), dt_c
        in_shape = dims
    else:
        in_dt = dt_c
        in_shape = hat(dims, kind)
        out_shape, out_dt = dims, (dt_r if kind == "c2r" else dt_c)
    x = np.ascontiguousarray(x, dtype=in_dt).reshape(in_shape)
    out = np.zeros(out_shape, dtype=out_dt)
    sig = ctypes.create_string_buffer(128)
    st = lib().oracle_execute(8 if prec == "f64" else 4, len(dims), _i64(dims),
                              DECOMPS[decomp], len(grid), _int(grid), KINDS[kind],
                              0 if fwd else 1, 1 if normalize else 0,
                              x.ctypes.data, out.ctypes.data, sig)
    if st != 0:
        raise OracleError(st)
    return out, sig.value.decode()


def local_extents(dims, decomp, grid, kind, direction, side, rank):
    off = (ctypes.c_int64 * len(dims))()
    ln = (ctypes.c_int64 * len(dims))()
    st = lib().oracle_local_extents(len(dims), _i64(dims), DECOMPS[decomp], len(grid),
                                    _int(grid), KINDS[kind],
                                    0 if direction == "forward" else 1, side, rank, off, ln)
    if st != 0:
        raise OracleError(st)
    return list(off), list(ln)


def block_map(n, p):
    c = (ctypes.c_int64 * p)()
    o = (ctypes.c_int64 * p)()
    lib().oracle_block_map(n, p, c, o)
    return list(c), list(o)


def dft(x, direction="forward"):
    x = np.ascontiguousarray(x, dtype=np.complex128)
    out = np.empty_like(x)
    st = lib().oracle_dft(x.ctypes.data, x.ndim, _i64(list(x.shape)),
                          0 if direction == "forward" else 1, out.ctypes.data)
    if st != 0:
        raise OracleError(st)
    return out


ERROR_NAMES = [
    "OK", "ZeroLength", "OutOfBounds", "TooLarge", "LengthMismatch", "NonHermitian",
    "SlabTooManyRanks", "OutOfRange", "InvalidRank", "TagMismatchTimeout", "Deadlock",
    "WorkerPanic", "CountMismatch", "IncompatibleLayouts", "ArenaExhausted",
    "GridMismatch", "RankTooLow", "LayoutMismatch", "NotFrequencyLayout", "NonZeroMean",
    "BadMagic", "DimMismatch", "TruncatedFile", "ConfigInvalid",
]


class OracleError(RuntimeError):
    def __init__(self, code):
        self.code = code
        super().__init__(ERROR_NAMES[code] if code < len(ERROR_NAMES) else str(code))


def rel_l2(got, want):
    got = np.asarray(got, dtype=np.complex128).ravel()
    want = np.asarray(want, dtype=np.complex128).ravel()
    num = np.sum(np.abs(got - want) ** 2)
    den = np.sum(np.abs(want) ** 2)
    return float(np.sqrt(num) if den == 0 else np.sqrt(num / den))


GOLDEN_DIR = os.path.join(ROOT, "tests", "golden")


def golden_cases():
    import json
    with open(os.path.join(GOLDEN_DIR, "golden.json")) as f:
        return json.load(f)["cases"]


def load_golden(case):
    prec = case["prec"]
    dt_r = np.float64 if prec == "f64" else np.float32
    dt_c = np.complex128 if prec == "f64" else np.complex64
    p = os.path.join(GOLDEN_DIR, case["name"])
    dims = case["dims"]
    in_dt = dt_r if case["kind"] == "r2c" else dt_c
    x = np.fromfile(p + ".in.bin", dtype=in_dt).reshape(dims)
    y = np.fromfile(p + ".fwd.bin", dtype=dt_c).reshape(hat(dims, case["kind"]))
    z = np.fromfile(p + ".rt.bin", dtype=in_dt).reshape(dims)
    return x, y, z
