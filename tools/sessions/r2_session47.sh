#!/bin/bash
# round-2 GPU session 47 (1 GPU): single-rank R2C forward as F2, F0, F1 (DFFTB_R2C_ORDER) and the fp32 bank-aware lane stride (exp/libdfftb_ls4.so) on config E
O=gpurun_out/s47
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "exit $?" >> $O/pytest_gpu.log
tail -3 $O/pytest_gpu.log
for rep in 1 2; do
for v in "X=1" "DFFTB_R2C_ORDER=0" "DFFTB_LIB_OVERRIDE=exp/libdfftb_ls4.so" "DFFTB_LIB_OVERRIDE=exp/libdfftb_ls4.so DFFTB_R2C_ORDER=0"; do
  echo "== $v rep $rep" >> $O/ab.log
  timeout 300 env $v ONLY=E python tools/bench_configs.py >> $O/ab.log 2>&1
  [ $rep = 1 ] && timeout 200 env $v python tools/op_times_config.py 2048,512,256 r2c f32 pencil >> $O/ab.log 2>&1
done
done
grep -E "==|total|ms_fwdinv|local" $O/ab.log | sed 's/"gflops.*//'
echo done
