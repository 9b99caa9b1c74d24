#!/bin/bash
# round-2 GPU session 13 (1 GPU): graph replay vs op-by-op for D / E (PDL, graphs on/off)
O=gpurun_out/s13
mkdir -p $O
for s in "" "DFFTB_PDL=0" "DFFTB_GRAPHS=0" "DFFTB_PDL=0 DFFTB_GRAPHS=0"; do
  echo "== ${s:-default}" >> $O/ab.log
  for c in D E C A; do timeout 300 env $s ONLY=$c python tools/bench_configs.py >> $O/ab.log 2>&1; done
done
timeout 900 python -m pytest tests/test_gpu_fuzz.py tests/test_gpu_parity.py -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "exit $?" >> $O/pytest_gpu.log
echo done
