#!/bin/bash
# round-2 GPU session 38 (1 GPU): why the E backward 512-point fp32 pass is 1.7x the forward one (ncu source hot spots)
O=gpurun_out/s38
mkdir -p $O
R=/tmp/ncu_reports; mkdir -p $R
P="python tools/prof_one.py --dims 2048,512,256 --kind r2c --prec f32 --warmup 1 --steps 1"
$P > $O/pE.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:fft_pass -s 6 -c 6 -o $R/prof_E $P > $O/ncu_E.log 2>&1
tail -3 $O/ncu_E.log
python tools/ncu_summary.py $R/prof_E.ncu-rep > $O/summary_E.txt 2>&1
for k in "512, 16, 16, 1, 2, 0" "512, 16, 16, 1, 2, 1" "2048, 16, 4, 1, 2, 0"; do
  echo "==== $k" >> $O/hot.txt
  python tools/ncu_hot.py $R/prof_E.ncu-rep "fft_pass_tma_kernel<float, $k" 25 >> $O/hot.txt 2>&1
done
ncu -i $R/prof_E.ncu-rep --page raw --csv > $O/raw_E.csv 2>/dev/null
python - > $O/metrics.txt <<'PY'
import csv
rows = list(csv.reader(open("gpurun_out/s38/raw_E.csv")))
h = rows[0]
want = [c for c in h if any(s in c for s in ("bank_conflicts", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "smsp__inst_executed_op_shared", "l1tex__data_pipe_lsu_wavefronts_mem_shared", "lts__t_sectors_srcunit_tex_op_write.sum",
        "sm__warps_active.avg.pct", "smsp__average_warp_latency_issue_stalled_mio_throttle", "lts__t_sectors_op_write.sum", "lts__t_sectors_op_read.sum"))]
ik = h.index("Kernel Name")
for r in rows[2:]:
    print(r[ik][:70])
    for c in want:
        print("   ", c, r[h.index(c)])
PY
rm -f $R/*.ncu-rep
ls -la $O
echo done
