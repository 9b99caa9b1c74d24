#!/bin/bash
# round-2 GPU session 70 (1 GPU): ncu --set full of config D's first two forward passes (contiguous and strided 1024-point fp64) with the final code
O=gpurun_out/s70
mkdir -p $O
R=/tmp/ncu_reports; mkdir -p $R
P="python tools/prof_one.py --dims 1024,1024,1024 --kind c2c --prec f64 --warmup 1 --steps 1"
$P > $O/p.log 2>&1 && \
ncu --set full --clock-control none -k regex:fft_pass -s 6 -c 2 -o $R/prof $P > $O/ncu.log 2>&1
tail -1 $O/ncu.log
python tools/ncu_summary.py $R/prof.ncu-rep > $O/summary.txt 2>&1
rm -f $R/*.ncu-rep
cat $O/summary.txt
echo done
