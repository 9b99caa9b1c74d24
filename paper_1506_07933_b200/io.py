"""Reference-compatible formats: the DTNS tensor file (tensor_file.hpp,
tensor_file.cpp) and the bench JSON / CSV report (bench.cpp:413-472, pinned by
proj/tests/data/report_schema.golden).  Host-side plumbing around the B200
execute path."""
from __future__ import annotations

import enum
import json
import math
import struct
from typing import Dict, List, Optional, Sequence

import numpy as np
import torch

from .dfft import DistTensor, Distribution, ElementKind, Error

MAGIC = b"DTNS"
VERSION = 1


class TensorElement(enum.IntEnum):  # tensor_file.hpp:16-21
    Real64 = 0
    Complex64 = 1
    Real32 = 2
    Complex32 = 3


_NP = {TensorElement.Real64: np.float64, TensorElement.Complex64: np.complex128,
       TensorElement.Real32: np.float32, TensorElement.Complex32: np.complex64}


def element_of(arr: np.ndarray) -> TensorElement:
    for k, v in _NP.items():
        if arr.dtype == v:
            return k
    raise Error(21, f"no DTNS element kind for dtype {arr.dtype}")


def write_tensor_file(path: str, arr: np.ndarray) -> None:
    """write_tensor_file (tensor_file.cpp:75-99): header + row-major payload."""
    arr = np.ascontiguousarray(arr)
    el = element_of(arr)
    head = MAGIC + struct.pack("<IBI", VERSION, int(el), arr.ndim)
    head += b"".join(struct.pack("<Q", d) for d in arr.shape)
    with open(path, "wb") as f:
        f.write(head)
        f.write(arr.astype(arr.dtype.newbyteorder("<"), copy=False).tobytes())


def read_tensor_file(path: str, mmap: bool = True) -> np.ndarray:
    """read_tensor_file (tensor_file.cpp:27-73), with the same error codes."""
    try:
        f = open(path, "rb")
    except OSError:
        raise Error(22, f"cannot open {path}")
    with f:
        head = f.read(13)
        if len(head) < 13:
            raise Error(22, f"unexpected end of {path}")
        if head[:4] != MAGIC:
            raise Error(20, f"{path} is not a DTNS tensor")
        version, kind, axes = struct.unpack("<IBI", head[4:13])
        if version != VERSION:
            raise Error(20, "unsupported DTNS version")
        if kind > 3:
            raise Error(20, "unknown element kind")
        if axes == 0 or axes > 16:
            raise Error(20, "implausible axis count")
        raw = f.read(8 * axes)
        if len(raw) < 8 * axes:
            raise Error(22, f"unexpected end of {path}")
        dims = struct.unpack("<" + "Q" * axes, raw)
        if any(d < 1 for d in dims):
            raise Error(20, "non-positive axis length")
        dt = np.dtype(_NP[TensorElement(kind)]).newbyteorder("<")
        offset = 13 + 8 * axes
        n = int(np.prod(dims))
    size_ok = False
    import os
    size_ok = os.path.getsize(path) >= offset + n * dt.itemsize
    if not size_ok:
        raise Error(22, f"unexpected end of {path}")
    if mmap:
        return np.memmap(path, dtype=dt, mode="r", offset=offset, shape=tuple(dims))
    return np.fromfile(path, dtype=dt, count=n, offset=offset).reshape(dims)


def read_tensor(dist: Distribution, rank: int, path: str, device=None) -> DistTensor:
    """read_tensor (tensor_file.hpp:49-95): this rank's block of the file.
    Real files are promoted to complex for complex layouts, as the reference
    does (bench.cpp:141-147); every rank maps the file and slices its own
    block (no rank-0 scatter needed on one node)."""
    arr = read_tensor_file(path)
    if tuple(arr.shape) != tuple(dist.dims):
        raise Error(21, "tensor file dims do not match the layout")
    if dist.element == ElementKind.Real and np.iscomplexobj(arr):
        # tensor_file.hpp:63-66: never drop imaginary parts silently
        raise Error(21, "complex tensor file cannot feed a real layout")
    sl = tuple(slice(o, o + n) for o, n in dist.extents_of(rank))
    blk = np.ascontiguousarray(arr[sl])
    plan = dist._plan
    want = plan.dtype_of(dist)
    t = torch.from_numpy(blk.reshape(-1)).to(want)
    dev = device if device is not None else torch.device("cuda", torch.cuda.current_device())
    return DistTensor(dist, rank, t.to(dev))


def write_tensor(path: str, blocks: Sequence[DistTensor]) -> None:
    """write_tensor (tensor_file.hpp:97-141) from every rank's block (the
    caller gathers them, e.g. torch.distributed.gather_object)."""
    dist = blocks[0].dist
    full = None
    for b in blocks:
        blk = b.data.cpu().numpy()
        if full is None:
            full = np.zeros(dist.dims, dtype=blk.dtype)
        ext = dist.extents_of(b.rank)
        full[tuple(slice(o, o + n) for o, n in ext)] = blk.reshape(tuple(n for _, n in ext))
    write_tensor_file(path, full)


# ------------------------------------------------------------------ report

TIMING_KEYS = ("local_fft", "pack", "unpack", "staging_copy", "wire_comm", "total")


def flops_estimate(dims: Sequence[int]) -> float:
    """bench.cpp:32-41: 5 N log2 N, exact for powers of two."""
    n = 1
    for d in dims:
        n *= int(d)
    if n <= 1:
        return 0.0
    if n & (n - 1) == 0:
        return float(5 * n * (n.bit_length() - 1))
    return 5.0 * n * math.log2(n)


def to_json(config: Dict, reps: List[Dict[str, float]], rel_error: Optional[float],
            warnings: Sequence[str] = ()) -> str:
    """The reference's report (bench.cpp:413-451, schema_version 1): min and
    median are the reps with the min / median total."""
    order = sorted(range(len(reps)), key=lambda i: reps[i]["total"])
    best = reps[order[0]]
    median = reps[order[(len(order) - 1) // 2]]
    flops = flops_estimate(config["dims"])
    status = "skipped" if rel_error is None else ("passed" if rel_error <= 1e-10 else "failed")
    cfg = {k: config[k] for k in ("dims", "grid", "kind", "decomp", "backend", "pipelined", "chunks",
                                  "staging_buffers", "reps", "warmup", "seed")}
    j = {
        "schema_version": 1,
        "config": cfg,
        "timings": {"unit": "seconds", "reps": [{k: r[k] for k in TIMING_KEYS} for r in reps],
                    "min": {k: best[k] for k in TIMING_KEYS},
                    "median": {k: median[k] for k in TIMING_KEYS}},
        "performance": {"flops_estimate": flops,
                        "gflops": flops / best["total"] / 1e9 if best["total"] > 0 else 0.0},
        "verification": {"status": status, "rel_error": 0.0 if rel_error is None else rel_error},
        "warnings": list(warnings),
    }
    return json.dumps(j, indent=2) + "\n"


def to_csv(reps: List[Dict[str, float]]) -> str:
    """bench.cpp:453-472."""
    order = sorted(range(len(reps)), key=lambda i: reps[i]["total"])
    rows = ["rep," + ",".join(TIMING_KEYS)]
    fmt = lambda r: ",".join(f"{r[k]:.9e}" for k in TIMING_KEYS)  # noqa: E731
    rows += [f"{i},{fmt(r)}" for i, r in enumerate(reps)]
    rows.append("min," + fmt(reps[order[0]]))
    rows.append("median," + fmt(reps[order[(len(order) - 1) // 2]]))
    return "\n".join(rows) + "\n"


def schema_paths(obj, prefix="") -> List[str]:
    """Flattened 'path: type' lines in the format of report_schema.golden."""
    out = []
    if isinstance(obj, dict):
        for k, v in obj.items():
            out += schema_paths(v, f"{prefix}/{k}")
    elif isinstance(obj, list):
        out.append(f"{prefix}: array")
        if obj:
            out += schema_paths(obj[0], prefix + "[]")
    else:
        t = "boolean" if isinstance(obj, bool) else "number" if isinstance(obj, (int, float)) \
            else "string"
        out.append(f"{prefix}: {t}")
    return out
