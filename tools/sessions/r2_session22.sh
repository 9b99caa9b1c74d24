#!/bin/bash
# round-2 GPU session 22 (1 GPU): final-code ncu: bench launch list; --set full of the 512^3, B and D passes
O=gpurun_out/s22
mkdir -p $O
R=/tmp/ncu_reports; mkdir -p $R
B="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
$B > $O/bench_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file $O/launches_bench.csv $B > $O/ncu_launch.log 2>&1
for cfg in "512:--dims 512,512,512:6" "B:--dims 256,256,256 --kind r2c:6" "D:--dims 1024,1024,1024:3"; do
  name=${cfg%%:*}; rest=${cfg#*:}; args=${rest%:*}; cnt=${rest##*:}
  P="python tools/prof_one.py $args --warmup 1 --steps 1"
  $P > $O/p_$name.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:fft_pass -s 6 -c $cnt -o $R/prof_$name $P > $O/ncu_$name.log 2>&1
  ncu -i $R/prof_$name.ncu-rep --page raw --csv > $O/raw_$name.csv 2>&1
  python tools/ncu_summary.py $R/prof_$name.ncu-rep > $O/summary_$name.txt 2>&1
  python tools/ncu_hot.py $R/prof_$name.ncu-rep fft_pass 25 > $O/hot_$name.txt 2>&1
  rm -f $R/prof_$name.ncu-rep
done
du -sh $O
echo done
