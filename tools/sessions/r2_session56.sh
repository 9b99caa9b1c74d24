#!/bin/bash
# round-2 GPU session 56 (1 GPU): final-code launch list of the N=1 bench (ncu gpu__time_duration, after a clean run)
O=gpurun_out/s56
mkdir -p $O
timeout 300 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > $O/bench.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches.csv \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > $O/ncu.log 2>&1
echo "ncu exit $?"
python - <<'PY'
import csv, collections
rows = [r for r in csv.reader(open("gpurun_out/s56/launches.csv")) if len(r) > 10]
h = rows[0]
ik, iv, im = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Name")
agg = collections.OrderedDict()
for r in rows[1:]:
    if r[im] != "gpu__time_duration.sum":
        continue
    k = r[ik].split("(")[0][:90]
    v = float(r[iv].replace(",", ""))
    a = agg.setdefault(k, [0, 0.0])
    a[0] += 1
    a[1] += v
tot = sum(v for _, v in agg.values())
with open("gpurun_out/s56/launches_summary.txt", "w") as f:
    f.write("# round 2 session 56: ncu --metrics gpu__time_duration.sum --clock-control none -c 400 python bench.py --steps 2 --warmup 3 (final code, N=1); per kernel: launches, total, share\n")
    for k, (n, v) in agg.items():
        f.write(f"{n:5d}  {v/1e3:10.1f} us  {100*v/tot:5.1f}%  {k}\n")
print(open("gpurun_out/s56/launches_summary.txt").read())
PY
grep -c . $O/launches.csv
echo done
