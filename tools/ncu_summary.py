"""Summarise an ncu report (raw page) into a short table: per kernel the
duration, DRAM bytes/throughput, issue utilisation, registers, top stalls."""
import csv
import subprocess
import sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[0]


def g(r, k):
    try:
        return r[hdr.index(k)]
    except ValueError:
        return "n/a"


for r in rows[2:]:
    name = g(r, "Kernel Name")
    dur = float(g(r, "gpu__time_duration.sum"))
    rd = float(g(r, "dram__bytes_read.sum"))
    wr = float(g(r, "dram__bytes_write.sum"))
    stalls = []
    for i, h in enumerate(hdr):
        if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio"):
            try:
                stalls.append((float(r[i]), h[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
            except ValueError:
                pass
    stalls.sort(reverse=True)
    print(f"{name[:75]}")
    print(f"   duration {dur:.3f} (ncu units: {hdr and 'see csv'}), dram read {rd:.3f} write {wr:.3f}, "
          f"dram% {g(r, 'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed')}, "
          f"issue% {g(r, 'sm__inst_issued.avg.pct_of_peak_sustained_active')}, "
          f"regs {g(r, 'launch__registers_per_thread')}, warps/SM {g(r, 'sm__warps_active.avg.per_cycle_active')}")
    print("   top stalls: " + ", ".join(f"{n} {v:.2f}" for v, n in stalls[:5]))
