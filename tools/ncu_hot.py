"""Summarise an ncu source page (SASS): top instructions by warp-stall
samples, grouped with their stall-reason columns.  Usage:
  python tools/ncu_hot.py REPORT.ncu-rep KERNEL_REGEX [N]"""
import csv
import io
import subprocess
import sys

rep, kre = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                      "-k", "regex:" + kre], capture_output=True, text=True).stdout
lines = out.splitlines()
# first kernel block only
start = next(i for i, l in enumerate(lines) if l.startswith('"Address"'))
end = next((i for i in range(start + 1, len(lines)) if lines[i].startswith('"Kernel Name"')), len(lines))
rows = list(csv.reader(io.StringIO("\n".join(lines[start:end]))))
h = rows[0]
ia, isrc, iss = h.index("Address"), h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
stall_cols = [i for i, x in enumerate(h) if x.startswith("stall_") or "Stall" in x and i != iss]
data = []
tot = 0
for r in rows[1:]:
    try:
        s = int(r[iss])
    except ValueError:
        continue
    tot += s
    data.append((s, r))
data.sort(key=lambda t: -t[0])
print("total samples", tot)
for s, r in data[:n]:
    extra = []
    for i in stall_cols:
        try:
            v = int(r[i])
        except ValueError:
            continue
        if v > 0.2 * s and h[i] not in ("Warp Stall Sampling (Not-issued Samples)",):
            extra.append(f"{h[i]}={v}")
    print(f"{s:6d} {100*s/tot:5.1f}%  {r[ia][-5:]}  {r[isrc].strip()[:60]:60s} {' '.join(extra)[:120]}")
