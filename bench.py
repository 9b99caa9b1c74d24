"""Benchmark: 3-D FFT GFLOP/s (5 N log2 N convention) and fwd+inv time,
512^3 C2C fp64, on 1/2/4/8 B200 (BASELINE.json).

One step = forward + inverse (normalized) 3-D FFT of the whole 512^3 volume
through libdfftb (plan / execute), pencil decomposition on a 2 x N/2 grid
(N=1: single rank).  Strong scaling: the volume is fixed as N grows.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]

For N>1 launch under torchrun (one process per GPU); rank 0 prints ONE JSON
line.  `--impl reference` times the unmodified reference CPU implementation
(oracle/_ref/dfft_ref, compiled from /root/reference) on the host cores.
"""
import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

DIMS = (512, 512, 512)
METRIC = "3D FFT GFLOP/s (5NlogN) & fwd+inv time, 512^3 C2C fp64, 1/2/4/8 B200"
UNIT = "GFLOP/s"
FLOP_FWDINV = 2 * 5 * (512 ** 3) * 27  # bench.cpp:32-41, x2 for fwd+inv
REF_BIN = os.path.join(ROOT, "oracle", "_ref", "dfft_ref")
NVL_NOMINAL_GBS = 900.0   # NVLink 5, per direction per GPU
NVL_MEASURED_GBS = 703.0  # SM peer stores, all GPUs at once (tools/p2p_store_probe.cu)


def grid_for(n):
    if n == 1:
        return (1, 1)
    return (2, n // 2)


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


# ------------------------------------------------------------ clocks sampler

class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled DURING the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index, interval_ms=10):
        self.index = index
        self.interval_ms = interval_ms
        self.rows = []  # (host time, fields)
        self.window = None
        self._proc = None
        self._t = None

    def _read(self):
        for line in self._proc.stdout:
            line = line.strip()
            if line:
                self.rows.append((time.time(), [c.strip() for c in line.split(",")]))

    def start(self):
        """Continuous `nvidia-smi -lms` stream; returns once it is producing."""
        try:
            self._proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", f"-lms={self.interval_ms}"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            return
        self._t = threading.Thread(target=self._read, daemon=True)
        self._t.start()
        t0 = time.time()
        while not self.rows and time.time() - t0 < 5:
            time.sleep(0.01)

    def stop(self):
        time.sleep(2 * self.interval_ms / 1000.0)
        if self._proc:
            self._proc.terminate()
            try:
                self._proc.wait(timeout=5)
            except Exception:
                self._proc.kill()
        if self._t:
            self._t.join(timeout=5)

    def summary(self):
        sm = []
        mx = None
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        rows = [r for t, r in self.rows
                if self.window is None or self.window[0] <= t <= self.window[1]]
        in_window = len(rows)
        if not rows and self.rows and self.window:
            # region shorter than the sampling period: nearest samples around it
            mid = 0.5 * (self.window[0] + self.window[1])
            rows = [r for _, r in sorted(self.rows, key=lambda tr: abs(tr[0] - mid))[:2]]
        for r in rows:
            try:
                sm.append(float(r[1]))
                mx = float(r[2])
                for k, name in enumerate(names):
                    if r[4 + k].lower().startswith("active"):
                        reasons.add(name)
            except Exception:
                pass
        sm.sort()
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm),
                "samples_in_timed_region": in_window}


# --------------------------------------------------------- reference (CPU)

def cpu_threads():
    """The reference has one thread per rank and no intra-rank threading
    (transport.cpp:92-119): use the largest power-of-two rank count the host
    cores allow (capped at 64)."""
    n = min(os.cpu_count() or 1, 64)
    p = 1
    while p * 2 <= n:
        p *= 2
    return p


def cpu_grid(p):
    a = 1
    while a * a < p:
        a *= 2
    a = a if a * a == p else a // 2
    return f"{a},{p // a}"


def run_reference(warmup, reps, dims=DIMS):
    """The unmodified reference (plan/execute through its public API) on host
    cores: P rank threads, pencil grid, one fwd+inv per rep."""
    if not os.path.exists(REF_BIN):
        raise RuntimeError("oracle/_ref/dfft_ref not built (make -C oracle ref)")
    p = cpu_threads()
    grid = cpu_grid(p)
    cmd = [REF_BIN, "--dims", ",".join(map(str, dims)), "--decomp", "pencil", "--grid", grid,
           "--kind", "c2c", "--prec", "f64", "--seed", "1", "--warmup", str(warmup),
           "--reps", str(reps)]
    out = subprocess.run(cmd, check=True, capture_output=True, text=True).stdout
    rep = json.loads(out.strip().splitlines()[-1])
    return rep, p, grid


def reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    warm = min(args.warmup, 1)
    reps = max(1, min(args.steps, 3))
    rep, p, grid = run_reference(warm, reps)
    t = rep["fwdinv_median_s"]
    value = FLOP_FWDINV / t / 1e9
    sample = (f"512^3 C2C fp64 fwd+inv, pencil {grid.replace(',', 'x')}, {p} rank threads, "
              f"median of {reps} reps after {warm} warmup (reference bench protocol)")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": args.gpus, "steps": reps, "warmup": warm, "ms_per_step": t * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (bench.cpp seeded_value, seed 1)",
        "config": {"workload": "512^3 C2C fp64 forward+inverse", "dims": list(DIMS),
                   "grid": [int(x) for x in grid.split(",")], "decomp": "pencil",
                   "host_threads": p},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": p, "kind": "reference",
                         "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "roundtrip_rel_l2": rep["roundtrip_rel_l2"],
        "fwd_s": rep["fwd_median_s"], "inv_s": rep["inv_median_s"],
    }
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------ B200 arm

def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="dfftb")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        return reference_arm(args)

    import torch
    import torch.distributed as dist

    import paper_1506_07933_b200 as D
    from paper_1506_07933_b200.telemetry import NvlinkCounters

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    N = world
    if N != args.gpus and rank == 0:
        print(f"warning: --gpus {args.gpus} but WORLD_SIZE {world}; using {world}", file=sys.stderr)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    W = max(3, args.warmup)
    K = max(1, args.steps)

    grid = grid_for(N)
    fwd = D.plan_pencil(DIMS, grid, D.TransformKind.C2C, D.Direction.Forward)
    bwd = D.plan_pencil(DIMS, grid, D.TransformKind.C2C, D.Direction.Backward)
    ctx = D.make_context(fwd)
    x = D.DistTensor.seeded(fwd.input, rank, seed=1)
    y = D.DistTensor.zeros(fwd.output, rank)
    z = D.DistTensor.zeros(bwd.output, rank)
    stream = torch.cuda.current_stream()

    def step():
        D.execute(fwd, x, ctx, out=y, sync=False)
        D.execute(bwd, y, ctx, out=z, sync=False)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(v):
        if world == 1:
            return v
        t = torch.tensor([v], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return t.item()

    launches0 = D.kernel_launch_count()
    for _ in range(W):
        step()
    barrier()
    ctx.check()

    sampler = ClockSampler(local) if rank == 0 else None
    if sampler:
        sampler.start()
    nvl = NvlinkCounters(local) if world > 1 else None
    barrier()
    nvl0 = nvl.read() if nvl and nvl.available else None
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    l_before = D.kernel_launch_count()
    t_host0 = time.time()
    e0.record(stream)
    for _ in range(K):
        step()
    e1.record(stream)
    barrier()
    t_host1 = time.time()
    nvl1 = nvl.read() if nvl0 else None
    l_timed = D.kernel_launch_count() - l_before
    if sampler:
        sampler.stop()
        sampler.window = (t_host0, t_host1)
    ms = max_over_ranks(e0.elapsed_time(e1)) / K
    ctx.check()
    nvl_meas = None
    if world > 1:
        # driver NVLink data counters around the timed region (NVML), per GPU
        ok = 1.0 if nvl1 else 0.0
        tx = (nvl1[0] - nvl0[0]) / K if nvl1 else 0.0
        rx = (nvl1[1] - nvl0[1]) / K if nvl1 else 0.0
        t = torch.tensor([ok, tx, rx, tx, rx], dtype=torch.float64, device=dev)
        tmin = t.clone()
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.all_reduce(tmin, op=dist.ReduceOp.MIN)
        if tmin[0].item() == 1.0:
            n_loc_max = max(fwd.input.local_count(r) for r in range(world))
            p0_, p1_ = grid
            expect = 2 * 16 * n_loc_max * ((p1_ - 1) / p1_ + (p0_ - 1) / p0_)
            nvl_meas = {"source": "NVML NVLINK_THROUGHPUT_DATA_TX/RX (driver counters, all links)",
                        "tx_bytes_per_step_per_gpu_max": t[1].item(),
                        "rx_bytes_per_step_per_gpu_max": t[2].item(),
                        "tx_bytes_per_step_per_gpu_min": tmin[3].item(),
                        "algorithmic_bytes_per_step_per_gpu": expect,
                        "tx_GBs_over_step": t[1].item() / (ms * 1e-3) / 1e9}
        else:
            nvl_meas = {"unavailable": nvl.why if nvl and not nvl.available else "counter read failed"}

    # parity of what was timed: round trip of the last step
    rt = (torch.linalg.vector_norm(z.data - x.data) ** 2).item()
    den = (torch.linalg.vector_norm(x.data) ** 2).item()
    if world > 1:
        t = torch.tensor([rt, den], dtype=torch.float64, device=dev)
        dist.all_reduce(t)
        rt, den = t[0].item(), t[1].item()
    rt_err = math.sqrt(rt / den)

    # the reference bench's protocol (bench.cpp:300-339): each
    # rep times fwd and inv separately with CUDA events after a barrier, max
    # over ranks, then min and median over the reps
    reps = []
    for _ in range(10):
        barrier()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        ev[0].record(stream)
        D.execute(fwd, x, ctx, out=y, sync=False)
        ev[1].record(stream)
        D.execute(bwd, y, ctx, out=z, sync=False)
        ev[2].record(stream)
        torch.cuda.synchronize()
        reps.append((max_over_ranks(ev[0].elapsed_time(ev[1])), max_over_ranks(ev[1].elapsed_time(ev[2]))))

    def minmed(v):
        v = sorted(v)
        return {"min": v[0], "median": v[(len(v) - 1) // 2]}

    ref_protocol = {"reps": len(reps), "fwd_ms": minmed([a for a, _ in reps]),
                    "inv_ms": minmed([b for _, b in reps]), "fwdinv_ms": minmed([a + b for a, b in reps])}

    # per-pass device times: CUDA events around every pass / sync point of 3
    # more steps (op by op, no graph), TimingBreakdown + ExecContext.last_ops
    tb_f, tb_b = D.TimingBreakdown(), D.TimingBreakdown()
    ops = []  # (dir, execute index, kind, stream, n, share, start_ms, ms)
    for i in range(3):
        D.execute(fwd, x, ctx, out=y, timers=tb_f)
        ops += [("fwd", 2 * i) + o for o in ctx.last_ops()]
        D.execute(bwd, y, ctx, out=z, timers=tb_b)
        ops += [("bwd", 2 * i + 1) + o for o in ctx.last_ops()]
    KIND, SHARE, START, MS = 2, 5, 6, 7
    pass_ms = sum(o[MS] for o in ops if o[KIND] in ("local", "exchange")) / 3  # per step, SM passes
    local_ms = sum(o[MS] for o in ops if o[KIND] == "local") / 3
    local_share = sum(o[SHARE] for o in ops if o[KIND] == "local") / 3  # full passes (chunks count part)
    exch_ms = sum(o[MS] for o in ops if o[KIND] == "exchange") / 3
    sync_ms = sum(o[MS] for o in ops if o[KIND] == "sync") / 3
    copy_ms = sum(o[MS] for o in ops if o[KIND] == "copy") / 3
    n_local = int(round(local_share))
    local_elems = fwd.input.local_count(rank)
    alg_bytes = 2 * 16 * local_elems  # one read + one write of the local block per pass
    peak, peak_kind = peaks()
    # HBM roofline of the dominant HBM-bound kernel: the local passes (all 6
    # passes at N=1; per full pass when the staged exchange chunks them; the
    # exchange traffic is NVLink-bound and reported below)
    avg_pass_ms = max_over_ranks(local_ms / max(1e-9, local_share))
    achieved = alg_bytes / (avg_pass_ms * 1e-3) / 1e9
    # NVLink: payload each rank stores into OTHER ranks per step (the plans'
    # exchange counts, make_transpose_step) over the exchange passes' time
    # pencil transposes (plan.hpp:149-236): forward T1 (grid axis 1) then T0
    # (axis 0), backward T0 then T1; a rank's own section is its coordinate
    coords = (rank // grid[1], rank % grid[1])
    remote = 0
    for plan, axes in ((fwd, (1, 0)), (bwd, (0, 1))):
        for t in range(plan.transpose_stage_count()):
            send, _ = plan.exchange_counts(rank, t)
            if len(send) > 1:
                remote += 16 * (sum(send) - send[coords[axes[t]]])
    # NVLink-active time per step: the union of the intervals of the ops that
    # move peer bytes -- exchange passes with direct peer stores (full
    # passes) and copy-engine DMAs of the staged exchange
    def nvl_active(ex):
        iv = sorted((o[START], o[START] + o[MS]) for o in ops if o[1] == ex and
                    (o[KIND] == "copy" or (o[KIND] == "exchange" and o[SHARE] >= 1.0)))
        tot, cur = 0.0, None
        for a, b in iv:
            if cur is None or a > cur[1]:
                if cur:
                    tot += cur[1] - cur[0]
                cur = [a, b]
            else:
                cur[1] = max(cur[1], b)
        return tot + (cur[1] - cur[0] if cur else 0.0)
    nvl_ms = max_over_ranks(sum(nvl_active(e) for e in range(6)) / 3)
    staged = any(o[KIND] == "copy" for o in ops)
    nvl_achieved = remote / (nvl_ms * 1e-3) / 1e9 if nvl_ms > 0 else None
    op_list = [{"dir": o[0], "kind": o[KIND], "stream": o[3], "n": o[4], "share": round(o[SHARE], 4),
                "start_ms": round(o[START], 4), "ms": round(o[MS], 4)}
               for o in ops if o[1] < 2]

    # end-to-end through the public API with host buffers: every step copies
    # its input from pinned host memory, runs fwd+inv and reads the result
    # back.  Copies run on their own streams, double-buffered, so step s+1's
    # upload overlaps step s's compute and download (PCIe is full duplex).
    e2e = None
    if not args.no_e2e:
        hx = torch.empty(local_elems, dtype=torch.complex128, pin_memory=True)
        hx.copy_(x.data.cpu())
        hz = [torch.empty(local_elems, dtype=torch.complex128, pin_memory=True) for _ in range(2)]
        xin = [D.DistTensor(fwd.input, rank, torch.empty_like(x.data)) for _ in range(2)]
        zout = [D.DistTensor(bwd.output, rank, torch.empty_like(z.data)) for _ in range(2)]
        s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()
        s_cmp = torch.cuda.current_stream()
        ev = {}

        def e2e_step(i):
            b = i % 2
            with torch.cuda.stream(s_in):
                if ("cmp", i - 2) in ev:
                    s_in.wait_event(ev[("cmp", i - 2)])   # buffer b no longer read
                xin[b].data.copy_(hx, non_blocking=True)
                ev[("in", i)] = torch.cuda.Event()
                ev[("in", i)].record(s_in)
            s_cmp.wait_event(ev[("in", i)])
            if ("out", i - 2) in ev:
                s_cmp.wait_event(ev[("out", i - 2)])      # zout[b] downloaded
            D.execute(fwd, xin[b], ctx, out=y, sync=False)
            D.execute(bwd, y, ctx, out=zout[b], sync=False)
            ev[("cmp", i)] = torch.cuda.Event()
            ev[("cmp", i)].record(s_cmp)
            with torch.cuda.stream(s_out):
                s_out.wait_event(ev[("cmp", i)])
                hz[b].copy_(zout[b].data, non_blocking=True)
                ev[("out", i)] = torch.cuda.Event()
                ev[("out", i)].record(s_out)

        for i in range(2):
            e2e_step(i)
        barrier()
        ev.clear()
        Ke = max(16, min(K, 32))  # amortise the pipeline fill (first upload, last download)
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record(s_in)
        for i in range(Ke):
            e2e_step(i)
        t1.record(s_out)
        barrier()
        ems = max_over_ranks(t0.elapsed_time(t1)) / Ke
        ok_e2e = bool(torch.equal(hz[(Ke - 1) % 2], z.data.cpu()))
        e2e = {"value": FLOP_FWDINV / (ems * 1e-3) / 1e9, "unit": UNIT,
               "ms_per_step": ems, "h2d_bytes_per_step": hx.numel() * 16,
               "d2h_bytes_per_step": hz[0].numel() * 16,
               "api": "paper_1506_07933_b200.execute (plan/execute through the C ABI)",
               "steps": Ke,
               # concurrent pinned up+down copies: 49.4 GB/s per direction
               # on one B200 (tools/pcie_probe.py)
               "pcie_floor_ms": hx.numel() * 16 / 49.4e9 * 1e3,
               "result_matches_device_run": ok_e2e}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline and os.path.exists(REF_BIN):
        try:
            rep, p, g = run_reference(1, 3)
            cpu = {"value": FLOP_FWDINV / rep["fwdinv_median_s"] / 1e9, "unit": UNIT, "cores": p,
                   "kind": "reference",
                   "sample": f"512^3 C2C fp64 fwd+inv, pencil {g.replace(',', 'x')}, {p} rank threads, "
                             f"median of 3 reps after 1 warm-up (BASELINE.md protocol): "
                             f"{rep['fwdinv_median_s']:.2f} s per fwd+inv"}
        except Exception as ex:  # reported, not fatal
            cpu = {"error": str(ex)}

    if rank == 0:
        value = FLOP_FWDINV / (ms * 1e-3) / 1e9
        # roofline of the whole step: slower of HBM (6 passes) and NVLink terms
        n_loc = local_elems
        t_hbm = 2 * 6 * 16 * n_loc / (peak * 1e9)
        p0, p1 = grid
        nvl = 2 * 16 * n_loc * ((p1 - 1) / p1 + (p0 - 1) / p0)
        # measured NVLink figure: SM-issued peer stores, all GPUs at once
        # (tools/p2p_store_probe.cu, profiles/r2_p2p_probe.txt); nominal below
        t_nvl = nvl / (NVL_MEASURED_GBS * 1e9)
        # SURVEY §8(d) convention: nominal 8 TB/s HBM and 900 GB/s NVLink
        t_nominal = max(2 * 6 * 16 * n_loc / 8.0e12, nvl / 900e9)
        traffic, traffic_src = None, None
        if world == 1:
            for src in ("profiles/r2/traffic.json", "profiles/r1_traffic.json"):
                try:
                    with open(os.path.join(ROOT, src)) as f:
                        traffic = json.load(f)["512^3_c2c_f64_grid1x1"]["dram_bytes_per_pass_avg"]
                    traffic_src = src + " (ncu --set full of the bench's passes, per pass)"
                    break
                except Exception:
                    traffic = None
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K,
            "warmup": W, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (reference bench seeded field, generated on device)",
            "config": {"workload": "512^3 C2C fp64 forward+inverse (normalized)",
                       "dims": list(DIMS), "decomp": "pencil", "grid": list(grid),
                       "parallelism": f"pencil{p0}x{p1}", "l2": "inputs larger than L2",
                       "exchange": ("staged: the FFT pass stores peer parts into staging images, "
                                    "copy-engine DMAs move them over NVLink in chunks overlapped with the "
                                    "next local pass; direct NVLink peer stores from the FFT pass for an "
                                    "exchange that feeds another exchange") if staged
                                   else "fused FFT + NVLink peer stores"},
            "gpu_launches": l_timed,
            "roundtrip_rel_l2": rt_err,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "traffic_source": traffic_src,
                         "algorithmic_bytes_per_pass": alg_bytes,
                         "kernel": "fft_pass_tma_kernel, local passes (average over the %d local passes "
                                   "per fwd+inv; CUDA events around each pass, 3 steps after the timed "
                                   "region)" % n_local,
                         "nvlink": None if nvl_achieved is None else {
                             "kernel": "exchange passes with direct peer stores (fft_pass_tma_kernel) and "
                                       "copy-engine DMAs of the staged exchange",
                             "payload_bytes_per_step": remote, "nvlink_active_ms_per_step": nvl_ms,
                             "achieved": nvl_achieved, "unit": "GB/s",
                             "peak_measured": NVL_MEASURED_GBS, "frac_measured": nvl_achieved / NVL_MEASURED_GBS,
                             "peak_nominal": NVL_NOMINAL_GBS, "frac_nominal": nvl_achieved / NVL_NOMINAL_GBS,
                             "counters": "profiles/r2/ncu_nvlink_exchange_pass_summary.txt (ncu nvltx bytes)"},
                         "peak_source": peak_kind,
                         "step_bound": "nvlink" if t_nvl > t_hbm else "hbm",
                         "step_roofline_ms": 1e3 * max(t_hbm, t_nvl),
                         "step_frac": 1e3 * max(t_hbm, t_nvl) / ms,
                         "nvlink_peak_measured_GBs": NVL_MEASURED_GBS,
                         "nvlink_peak_nominal_GBs": NVL_NOMINAL_GBS,
                         "step_roofline_ms_nominal_8TBs_900GBs": 1e3 * t_nominal,
                         "step_frac_nominal": 1e3 * t_nominal / ms},
            "clocks": sampler.summary() if sampler else None,
            "nvlink_counters": nvl_meas,
            "e2e": e2e,
            "cpu_baseline": cpu,
            # TimingBreakdown (timing.hpp:16-37) of the forward: local_fft =
            # local passes; wire_comm = exchange passes (FFT + NVLink stores)
            # + sync points; pack / unpack / staging_copy are fused (0)
            "fwd_breakdown_ms": {"local_fft": tb_f.local_fft / 3 * 1e3, "wire_comm": tb_f.wire_comm / 3 * 1e3,
                                 "pack": 0.0, "unpack": 0.0, "staging_copy": 0.0,
                                 "total": tb_f.total / 3 * 1e3},
            "step_ops_ms": {"passes": pass_ms, "exchange_passes": exch_ms, "sync_points": sync_ms,
                            "dma_copies": copy_ms},
            "ops_one_step": op_list,
            "reference_protocol": ref_protocol,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
