#!/bin/bash
# round-2 GPU session 63 (4 GPUs): staged chunk passes leave k SMs free for the signal kernels (DFFTB_DMA_SPARE=k) at N=2/4
O=gpurun_out/s63
mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for n in 2 4; do
for k in 0 1 2 0 1; do
  timeout 200 env DFFTB_DMA_SPARE=$k $TR --nproc-per-node $n --master-port $((29600 + RANDOM % 300)) bench.py --gpus $n --no-e2e > $O/b.log 2>&1
  echo "N=$n spare=$k: $(grep -o '"ms_per_step": [0-9.]*' $O/b.log | head -1) rt $(grep -o '"roundtrip_rel_l2": [0-9.e-]*' $O/b.log | head -1)"
done
done
echo done
