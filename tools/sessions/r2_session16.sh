#!/bin/bash
# round-2 GPU session 16 (1 GPU): internal row alignment (16 / 32 / 64 bytes) for odd-length rows
O=gpurun_out/s16
mkdir -p $O
for a in 16 32 64; do
  echo "== DFFTB_ROW_ALIGN=$a" >> $O/align.log
  for c in B E C D; do timeout 300 env DFFTB_ROW_ALIGN=$a ONLY=$c python tools/bench_configs.py >> $O/align.log 2>&1; done
  timeout 200 env DFFTB_ROW_ALIGN=$a python tools/op_times_config.py 2048,512,256 r2c f32 pencil >> $O/align.log 2>&1
done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "exit $?" >> $O/pytest_gpu.log
echo done
