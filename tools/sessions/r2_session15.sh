#!/bin/bash
# round-2 GPU session 15 (4 GPUs): half-length R2C / C2R lanes; rank-independent overlap chunking; full test suite
O=gpurun_out/s15
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q -s > $O/pytest_gpu.log 2>&1; echo "exit $?" >> $O/pytest_gpu.log
for v in 1 0; do
  echo "== DFFTB_RHALF=$v" >> $O/rhalf.log
  for c in B E; do timeout 300 env DFFTB_RHALF=$v ONLY=$c python tools/bench_configs.py >> $O/rhalf.log 2>&1; done
  timeout 200 env DFFTB_RHALF=$v python tools/op_times_config.py 2048,512,256 r2c f32 pencil >> $O/rhalf.log 2>&1
  timeout 200 env DFFTB_RHALF=$v python tools/op_times_config.py 256,256,256 r2c f64 slab >> $O/rhalf.log 2>&1
done
echo done
