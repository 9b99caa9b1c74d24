#!/bin/bash
# round-2 GPU session 20 (1 GPU): 2-CTA cluster pass A/B on the current code; ncu of the E 2048-point pass
O=gpurun_out/s20
mkdir -p $O
R=/tmp/ncu_reports; mkdir -p $R
for s in "" "DFFTB_CL2=1"; do
  echo "== ${s:-default}" >> $O/ab.log
  for c in D E; do timeout 300 env $s ONLY=$c python tools/bench_configs.py >> $O/ab.log 2>&1; done
  for c in "2048,512,256 r2c f32 pencil" "1024,1024,1024 c2c f64 pencil"; do timeout 200 env $s python tools/op_times_config.py $c >> $O/ab.log 2>&1; done
done
P="python tools/prof_one.py --dims 2048,512,256 --kind r2c --prec f32 --warmup 1 --steps 1"
$P > $O/pE.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:fft_pass -s 6 -c 6 -o $R/prof_E $P > $O/ncu_E.log 2>&1
python tools/ncu_summary.py $R/prof_E.ncu-rep > $O/summary_E.txt 2>&1
rm -f $R/*.ncu-rep
echo done
