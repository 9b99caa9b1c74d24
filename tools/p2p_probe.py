"""Calibration probe (one process, all visible GPUs): NVLink peer copy
bandwidth per direction with every GPU sending to its neighbour at once, and
the local HBM copy bandwidth.  Informational only."""
import torch

n = torch.cuda.device_count()
nbytes = 512 << 20
bufs = [torch.empty(nbytes // 8, dtype=torch.float64, device=f"cuda:{d}") for d in range(n)]
dsts = [torch.empty_like(b) for b in bufs]
for d in range(n):
    for e in range(n):
        if d != e:
            try:
                torch.cuda.set_device(d)
                torch.cuda.device(d)
            except Exception:
                pass


def timed(fn, devs, reps=5):
    for d in devs:
        torch.cuda.synchronize(d)
    fn()
    for d in devs:
        torch.cuda.synchronize(d)
    starts = [torch.cuda.Event(enable_timing=True) for _ in devs]
    ends = [torch.cuda.Event(enable_timing=True) for _ in devs]
    for i, d in enumerate(devs):
        with torch.cuda.device(d):
            starts[i].record()
    for _ in range(reps):
        fn()
    for i, d in enumerate(devs):
        with torch.cuda.device(d):
            ends[i].record()
    for d in devs:
        torch.cuda.synchronize(d)
    return max(s.elapsed_time(e) for s, e in zip(starts, ends)) / reps


ms = timed(lambda: dsts[0].copy_(bufs[0]), [0])
print(f"local HBM copy: {2 * nbytes / ms / 1e6:.0f} GB/s (read+write)")
if n >= 2:
    def ring():
        for d in range(n):
            with torch.cuda.device(d):
                dsts[(d + 1) % n].copy_(bufs[d], non_blocking=True)
    ms = timed(ring, list(range(n)))
    print(f"peer copy ring, {n} GPUs concurrently: {nbytes / ms / 1e6:.0f} GB/s per GPU per direction")
