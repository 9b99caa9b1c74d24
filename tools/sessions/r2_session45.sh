#!/bin/bash
# round-2 GPU session 45 (1 GPU): same-box A/B, radix-16 1024-point fp64 (default lib) vs the old radix-8 (exp/libdfftb_e8.so), config D x3
O=gpurun_out/s45
mkdir -p $O
for rep in 1 2 3; do
for lib in "" exp/libdfftb_e8.so; do
  echo "== ${lib:-default} rep $rep" >> $O/ab.log
  timeout 300 env DFFTB_LIB_OVERRIDE=$lib ONLY=D python tools/bench_configs.py >> $O/ab.log 2>&1
done
done
timeout 200 python tools/op_times_config.py 1024,1024,1024 c2c f64 pencil >> $O/ab.log 2>&1
grep -E "==|total|ms_fwdinv|local" $O/ab.log | sed 's/"gflops.*//'
echo done
