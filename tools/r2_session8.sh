#!/bin/bash
# round-2 GPU session 8 (1 GPU): small-tile variants for config A; ncu launch list of the bench;
# ncu --set full of the 512^3, D (1024^3 fp64) and E (2048x512x256 R2C fp32) passes
O=gpurun_out/s8
mkdir -p $O
for v in "" "exp/libdfftb_w16.so" "exp/libdfftb_w8.so"; do
  echo "== lib ${v:-default}" >> $O/configs_small.log
  timeout 300 env DFFTB_LIB_OVERRIDE=$v python tools/bench_configs.py >> $O/configs_small.log 2>&1
done
B="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
$B > $O/bench_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_bench.csv $B > $O/ncu_launch.log 2>&1
P1="python tools/prof_one.py --warmup 1 --steps 1"
$P1 > $O/p512.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:fft_pass -s 6 -c 6 -o $O/prof_512 $P1 > $O/ncu_512.log 2>&1
PD="python tools/prof_one.py --dims 1024,1024,1024 --warmup 1 --steps 1"
$PD > $O/pD.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:fft_pass -s 6 -c 3 -o $O/prof_D $PD > $O/ncu_D.log 2>&1
PE="python tools/prof_one.py --dims 2048,512,256 --kind r2c --prec f32 --warmup 1 --steps 1"
$PE > $O/pE.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:fft_pass -s 6 -c 6 -o $O/prof_E $PE > $O/ncu_E.log 2>&1
echo done
