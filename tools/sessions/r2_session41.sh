#!/bin/bash
# round-2 GPU session 41 (1 GPU): lane-blocked buffers for narrow strided passes + single-rank forward in the fixed order
O=gpurun_out/s41
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "exit $?" >> $O/pytest_gpu.log
tail -4 $O/pytest_gpu.log
for s in "X=1" "DFFTB_BLOCKED=0" "DFFTB_BLOCKED=0 DFFTB_SINGLE_FWD=0"; do
  echo "== $s" >> $O/ab.log
  for c in C D E; do timeout 300 env $s ONLY=$c python tools/bench_configs.py >> $O/ab.log 2>&1; done
  timeout 200 env $s python tools/op_times_config.py 2048,512,256 r2c f32 pencil >> $O/ab.log 2>&1
  timeout 200 env $s python tools/op_times_config.py 1024,1024,1024 c2c f64 pencil >> $O/ab.log 2>&1
done
grep -E "==|total|ms_fwdinv|local" $O/ab.log | sed 's/"gflops.*//'
timeout 300 python bench.py > $O/bench_n1.log 2>&1
grep -o '"ms_per_step": [0-9.]*' $O/bench_n1.log
echo done
