#!/bin/bash
# round-2 GPU session 43 (1 GPU): radix-16 stages for 1024-point fp64 lanes (exp/libdfftb_e16a: 512 threads W=8; e16b: 256 threads W=4) vs default on config D
O=gpurun_out/s43
mkdir -p $O
for rep in 1 2; do
for lib in "" exp/libdfftb_e16a.so exp/libdfftb_e16b.so; do
  echo "== ${lib:-default} rep $rep" >> $O/ab.log
  timeout 300 env DFFTB_LIB_OVERRIDE=$lib ONLY=D python tools/bench_configs.py >> $O/ab.log 2>&1
  [ $rep = 1 ] && timeout 200 env DFFTB_LIB_OVERRIDE=$lib python tools/op_times_config.py 1024,1024,1024 c2c f64 pencil >> $O/ab.log 2>&1
done
done
grep -E "==|total|ms_fwdinv|local" $O/ab.log | sed 's/"gflops.*//'
echo done
