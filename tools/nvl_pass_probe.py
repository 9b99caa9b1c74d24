"""NVLink evidence for the fused exchange pass (not a benchmark).

ONE process drives a P-rank emulated world over the visible GPUs
(make_world_contexts(devices=...)): rank r lives on GPU r % ngpu, the
exchange passes store straight into the other GPU's buffers over NVLink, and
the host orders the ranks with cross-device CUDA events -- no kernel ever
waits on another, so the run is safe to replay under ncu.  Profile the
exchange pass of rank 0 (device 0) with the NVLink byte counters:

  ncu --metrics gpu__time_duration.sum,nvltx__bytes.sum,nvlrx__bytes.sum,\\
dram__bytes_read.sum,dram__bytes_write.sum -k regex:fft_pass_tma --clock-control none \\
      python tools/nvl_pass_probe.py --grid 2,1

Without ncu it prints the per-rank exchange volume the plan implies, so the
counters can be checked against it (bytes a rank sends to other ranks).
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1506_07933_b200 as D  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--dims", default="512,512,512")
    ap.add_argument("--grid", default="2,1")
    ap.add_argument("--reps", type=int, default=2)
    a = ap.parse_args()
    dims = tuple(int(v) for v in a.dims.split(","))
    grid = tuple(int(v) for v in a.grid.split(","))
    fwd = D.plan_pencil(dims, grid, D.TransformKind.C2C, D.Direction.Forward)
    P = fwd.nranks()
    ngpu = torch.cuda.device_count()
    devices = list(range(min(ngpu, P)))
    ctxs = D.make_world_contexts(fwd, devices=devices)
    xs = [D.DistTensor.seeded(fwd.input, r, device=ctxs[r].device) for r in range(P)]
    for _ in range(a.reps):
        D.execute_world(fwd, xs, ctxs)
    for d in devices:
        torch.cuda.synchronize(d)
    # elements each rank stores into each group member's buffer, per
    # transpose stage (group order; members other than the rank itself on
    # another GPU receive them over NVLink)
    for t in range(fwd.transpose_stage_count()):
        for r in range(P):
            send, _recv = fwd.exchange_counts(r, t)
            print(f"transpose {t} rank {r} (GPU {r % len(devices)}): sends {[c * 16 for c in send]} B")
    for c in ctxs:
        c.close()


if __name__ == "__main__":
    main()
