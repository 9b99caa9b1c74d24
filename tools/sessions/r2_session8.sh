#!/bin/bash
# round-2 GPU session 8 (1 GPU): small-tile variants for config A; ncu launch list of the bench;
# ncu --set full of the 512^3, D (1024^3 fp64) and E (2048x512x256 R2C fp32) passes.
# Reports are summarised on the box (raw-page CSV + tools/ncu_summary.py) and deleted:
# gpurun brings back at most 64 MiB.
O=gpurun_out/s8
mkdir -p $O
R=/tmp/ncu_reports
mkdir -p $R
for v in "" "exp/libdfftb_w16.so" "exp/libdfftb_w8.so"; do
  echo "== lib ${v:-default}" >> $O/configs_small.log
  timeout 300 env DFFTB_LIB_OVERRIDE=$v ONLY=A python tools/bench_configs.py >> $O/configs_small.log 2>&1
  timeout 300 env DFFTB_LIB_OVERRIDE=$v ONLY=B python tools/bench_configs.py >> $O/configs_small.log 2>&1
done
B="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
$B > $O/bench_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_bench.csv $B > $O/ncu_launch.log 2>&1
for cfg in "512:--dims 512,512,512:6" "D:--dims 1024,1024,1024:3" "E:--dims 2048,512,256 --kind r2c --prec f32:6"; do
  name=${cfg%%:*}; rest=${cfg#*:}; args=${rest%:*}; cnt=${rest##*:}
  P="python tools/prof_one.py $args --warmup 1 --steps 1"
  $P > $O/p_$name.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:fft_pass -s 6 -c $cnt -o $R/prof_$name $P > $O/ncu_$name.log 2>&1
  ncu -i $R/prof_$name.ncu-rep --page raw --csv > $O/raw_$name.csv 2>&1
  python tools/ncu_summary.py $R/prof_$name.ncu-rep > $O/summary_$name.txt 2>&1
  python tools/ncu_hot.py $R/prof_$name.ncu-rep fft_pass 30 > $O/hot_$name.txt 2>&1
  rm -f $R/prof_$name.ncu-rep
done
du -sh $O
echo done
