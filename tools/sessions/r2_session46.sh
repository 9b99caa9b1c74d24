#!/bin/bash
# round-2 GPU session 46 (1 GPU): ncu source hot spots of config D's strided 1024-point pass (F1 of the profiled forward)
O=gpurun_out/s46
mkdir -p $O
R=/tmp/ncu_reports; mkdir -p $R
P="python tools/prof_one.py --dims 1024,1024,1024 --kind c2c --prec f64 --warmup 1 --steps 1"
$P > $O/pD.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:fft_pass -s 7 -c 1 -o $R/prof_D_F1 $P > $O/ncu_D.log 2>&1
tail -2 $O/ncu_D.log
python tools/ncu_summary.py $R/prof_D_F1.ncu-rep > $O/summary_D_F1.txt 2>&1
python tools/ncu_hot.py $R/prof_D_F1.ncu-rep fft_pass 40 > $O/hot_D_F1.txt 2>&1
ncu -i $R/prof_D_F1.ncu-rep --page details --csv > $O/details_D_F1.csv 2>/dev/null
rm -f $R/*.ncu-rep
head -50 $O/hot_D_F1.txt
cat $O/summary_D_F1.txt
echo done
