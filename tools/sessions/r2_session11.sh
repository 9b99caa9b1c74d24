#!/bin/bash
# round-2 GPU session 11 (1 GPU): TMA row pairs for odd-length fp32 rows (C2R user blocks)
O=gpurun_out/s11
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "exit $?" >> $O/pytest_gpu.log
for v in 1 0; do
  echo "== DFFTB_PAIRS=$v" >> $O/pairs.log
  timeout 300 env DFFTB_PAIRS=$v ONLY=E python tools/bench_configs.py >> $O/pairs.log 2>&1
  timeout 300 env DFFTB_PAIRS=$v ONLY=B python tools/bench_configs.py >> $O/pairs.log 2>&1
  timeout 200 env DFFTB_PAIRS=$v python tools/op_times_config.py 2048,512,256 r2c f32 pencil >> $O/pairs.log 2>&1
done
echo done
