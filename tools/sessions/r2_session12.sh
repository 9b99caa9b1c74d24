#!/bin/bash
# round-2 GPU session 12 (1 GPU): bank-aware lane strides for narrow strided tiles (W < 8 fp64 / 16 fp32)
O=gpurun_out/s12
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "exit $?" >> $O/pytest_gpu.log
timeout 300 python tools/bench_configs.py > $O/configs_n1.log 2>&1
for c in "2048,512,256 r2c f32 pencil" "1024,1024,1024 c2c f64 pencil"; do
  echo "== $c" >> $O/optimes.log
  timeout 200 python tools/op_times_config.py $c >> $O/optimes.log 2>&1
done
timeout 200 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > $O/bench_n1.log 2>&1
echo done
