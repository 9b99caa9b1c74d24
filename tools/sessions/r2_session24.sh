#!/bin/bash
# round-2 GPU session 24 (1 GPU): PDL on short passes (configs A, B; E at N=1 for reference)
O=gpurun_out/s24
mkdir -p $O
for r in 1 2; do
for s in "DFFTB_PDL=0" "DFFTB_PDL=1"; do
  echo "== $s" >> $O/ab.log
  for c in A B E; do timeout 300 env $s ONLY=$c python tools/bench_configs.py >> $O/ab.log 2>&1; done
done
done
echo done
