#!/bin/bash
# round-2 GPU session 57 (4 GPUs): staged exchange chunk-count sweep (6/8/12) at N=2 and N=4, bench ms_per_step x2
O=gpurun_out/s57
mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for n in 2 4; do
for c in 8 6 12 8; do
  timeout 200 env DFFTB_DMA_CHUNKS=$c $TR --nproc-per-node $n --master-port $((29600 + RANDOM % 300)) bench.py --gpus $n --no-e2e > $O/b_n${n}_c$c.log 2>&1
  echo "N=$n C=$c: $(grep -o '"ms_per_step": [0-9.]*' $O/b_n${n}_c$c.log | head -1)"
done
done
echo done
