#!/bin/bash
# round-2 GPU session 69 (1 GPU): ncu --set full of config E's six passes with the final code (one fwd+inv after a warm-up)
O=gpurun_out/s69
mkdir -p $O
R=/tmp/ncu_reports; mkdir -p $R
P="python tools/prof_one.py --dims 2048,512,256 --kind r2c --prec f32 --warmup 1 --steps 1"
$P > $O/p.log 2>&1 && \
ncu --set full --clock-control none -k regex:fft_pass -s 6 -c 6 -o $R/prof $P > $O/ncu.log 2>&1
tail -1 $O/ncu.log
python tools/ncu_summary.py $R/prof.ncu-rep > $O/summary.txt 2>&1
ncu -i $R/prof.ncu-rep --page raw --csv > $O/raw.csv 2>/dev/null
python - > $O/metrics.txt <<'PY'
import csv
rows = list(csv.reader(open("gpurun_out/s69/raw.csv")))
h = rows[0]
want = [c for c in h if c in ("gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum")]
ik = h.index("Kernel Name")
for r in rows[2:]:
    print(r[ik][:70])
    for c in want:
        print("   ", c, r[h.index(c)])
PY
rm -f $R/*.ncu-rep $O/raw.csv
cat $O/summary.txt
echo done
