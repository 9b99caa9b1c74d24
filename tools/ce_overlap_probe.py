"""Calibration probe (not product code): can a copy-engine NVLink transfer run
at full rate while the SMs run FFT passes at full HBM rate?

On every visible GPU at once: a 512 MiB peer copy (torch copy_ between
devices = cudaMemcpyPeerAsync, a DMA engine) to the neighbour GPU on one
stream, and a 512^3-block FFT (dfftb single-rank forward, 3 passes, 2 GiB
block) on another.  Prints each alone and both together.
    python tools/ce_overlap_probe.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1506_07933_b200 as D  # noqa: E402


def main():
    n = torch.cuda.device_count()
    if n < 2:
        print("need 2+ GPUs")
        return
    devs = list(range(n))
    src = [torch.empty(512 << 20, dtype=torch.uint8, device=f"cuda:{d}") for d in devs]
    dst = [torch.empty(512 << 20, dtype=torch.uint8, device=f"cuda:{d}") for d in devs]
    plans, ctxs, xs, ys = [], [], [], []
    for d in devs:
        with torch.cuda.device(d):
            fwd = D.plan_pencil((512, 512, 512), (1, 1), D.TransformKind.C2C, D.Direction.Forward)
            ctx = D.make_context(fwd, device=f"cuda:{d}")
            x = D.DistTensor.seeded(fwd.input, 0, device=f"cuda:{d}")
            y = D.DistTensor.zeros(fwd.output, 0, device=f"cuda:{d}")
            plans.append(fwd)
            ctxs.append(ctx)
            xs.append(x)
            ys.append(y)
    s_copy = [torch.cuda.Stream(device=d) for d in devs]
    s_fft = [torch.cuda.Stream(device=d) for d in devs]

    def run(copy, fft, reps=5):
        best = None
        for _ in range(reps):
            for d in devs:
                torch.cuda.synchronize(d)
            ev = {}
            for d in devs:
                with torch.cuda.device(d):
                    e0c, e1c = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0f, e1f = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    if copy:
                        with torch.cuda.stream(s_copy[d]):
                            e0c.record()
                            dst[(d + 1) % n].copy_(src[d], non_blocking=True)
                            e1c.record()
                    if fft:
                        with torch.cuda.stream(s_fft[d]):
                            e0f.record()
                            D.execute(plans[d], xs[d], ctxs[d], out=ys[d], sync=False)
                            e1f.record()
                    ev[d] = (e0c, e1c, e0f, e1f)
            for d in devs:
                torch.cuda.synchronize(d)
            tc = max(ev[d][0].elapsed_time(ev[d][1]) for d in devs) if copy else 0.0
            tf = max(ev[d][2].elapsed_time(ev[d][3]) for d in devs) if fft else 0.0
            if best is None or tc + tf < best[0] + best[1]:
                best = (tc, tf)
        return best

    run(True, True, 2)  # warm up (graphs, peer mappings)
    c, _ = run(True, False)
    _, f = run(False, True)
    cb, fb = run(True, True)
    print(f"{n} GPUs at once: copy alone {c:.3f} ms ({(512 << 20) / c / 1e6:.0f} GB/s), "
          f"FFT fwd alone {f:.3f} ms; together: copy {cb:.3f} ms ({(512 << 20) / cb / 1e6:.0f} GB/s), "
          f"FFT {fb:.3f} ms")


if __name__ == "__main__":
    main()
