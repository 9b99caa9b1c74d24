#!/bin/bash
# round-2 GPU session 40 (1 GPU): fp32 bank-aware lane stride (exp/libdfftb_ls4.so, DFFTB_LS_FP32=1) vs default on config E, op times x2 each; ncu of the variant
O=gpurun_out/s40
mkdir -p $O
R=/tmp/ncu_reports; mkdir -p $R
for rep in 1 2; do
  for lib in "" "exp/libdfftb_ls4.so"; do
    echo "== ${lib:-default} rep $rep" >> $O/ab.log
    timeout 200 env DFFTB_LIB_OVERRIDE=$lib python tools/op_times_config.py 2048,512,256 r2c f32 pencil >> $O/ab.log 2>&1
    timeout 200 env DFFTB_LIB_OVERRIDE=$lib ONLY=E python tools/bench_configs.py >> $O/ab.log 2>&1
  done
done
P="python tools/prof_one.py --dims 2048,512,256 --kind r2c --prec f32 --warmup 1 --steps 1"
DFFTB_LIB_OVERRIDE=exp/libdfftb_ls4.so $P > $O/pE.log 2>&1 && \
DFFTB_LIB_OVERRIDE=exp/libdfftb_ls4.so ncu --set full --clock-control none -k regex:fft_pass -s 6 -c 6 -o $R/prof_E_ls4 $P > $O/ncu_E.log 2>&1
python tools/ncu_summary.py $R/prof_E_ls4.ncu-rep > $O/summary_E_ls4.txt 2>&1
ncu -i $R/prof_E_ls4.ncu-rep --page raw --csv > $O/raw.csv 2>/dev/null
python - > $O/metrics.txt <<'PY'
import csv
rows = list(csv.reader(open("gpurun_out/s40/raw.csv")))
h = rows[0]
want = [c for c in h if c in ("gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "lts__t_sectors_srcunit_tex_op_read.sum", "lts__t_sector_hit_rate.pct")]
ik = h.index("Kernel Name")
for r in rows[2:]:
    print(r[ik][:70])
    for c in want:
        print("   ", c, r[h.index(c)])
PY
rm -f $R/*.ncu-rep $O/raw.csv
grep -E "==|total|n= 2048|ms_fwdinv" $O/ab.log
cat $O/metrics.txt
echo done
