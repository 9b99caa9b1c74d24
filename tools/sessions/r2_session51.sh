#!/bin/bash
# round-2 GPU session 51 (1 GPU): lane stride TPL mod 16 for rows tiles of few threads per lane (exp/libdfftb_lsrows.so) vs default, config E
O=gpurun_out/s51
mkdir -p $O
for rep in 1 2; do
for lib in "" exp/libdfftb_lsrows.so; do
  echo "== ${lib:-default} rep $rep" >> $O/ab.log
  timeout 300 env DFFTB_LIB_OVERRIDE=$lib ONLY=E python tools/bench_configs.py >> $O/ab.log 2>&1
  [ $rep = 1 ] && timeout 200 env DFFTB_LIB_OVERRIDE=$lib python tools/op_times_config.py 2048,512,256 r2c f32 pencil >> $O/ab.log 2>&1
done
done
grep -E "==|total|ms_fwdinv|local" $O/ab.log | sed 's/"gflops.*//'
echo done
