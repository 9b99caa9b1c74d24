#!/bin/bash
# round-2 GPU session 17 (1 GPU): half-length R2C/C2R fix (stride units), row alignment A/B
O=gpurun_out/s17
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_spectral_golden.py tests/test_fullsize_ref.py -m gpu -x -q -s > $O/pytest_gpu.log 2>&1; echo "exit $?" >> $O/pytest_gpu.log
for s in "" "DFFTB_RHALF=0" "DFFTB_ROW_ALIGN=16" "DFFTB_ROW_ALIGN=64"; do
  echo "== ${s:-default}" >> $O/ab.log
  for c in B E; do timeout 300 env $s ONLY=$c python tools/bench_configs.py >> $O/ab.log 2>&1; done
  timeout 200 env $s python tools/op_times_config.py 2048,512,256 r2c f32 pencil >> $O/ab.log 2>&1
done
echo done
