#!/bin/bash
# round-2 GPU session 21 (1 GPU): fp32 lane-stride residue (exp/libdfftb_ls4.so) vs default, PDL off
O=gpurun_out/s21
mkdir -p $O
for v in "" "exp/libdfftb_ls4.so" "" "exp/libdfftb_ls4.so"; do
  echo "== lib ${v:-default}" >> $O/ab.log
  timeout 300 env DFFTB_LIB_OVERRIDE=$v ONLY=E python tools/bench_configs.py >> $O/ab.log 2>&1
  timeout 200 env DFFTB_LIB_OVERRIDE=$v python tools/op_times_config.py 2048,512,256 r2c f32 pencil >> $O/ab.log 2>&1
done
timeout 600 env DFFTB_LIB_OVERRIDE=exp/libdfftb_ls4.so python -m pytest tests/test_gpu_parity.py -m gpu -x -q > $O/pytest_ls4.log 2>&1; echo "exit $?" >> $O/pytest_ls4.log
echo done
