#!/bin/bash
# round-2 GPU session 30 (2 GPUs): staged exchange op times at 1 and 2 chunks (copy-engine rate in the library)
O=gpurun_out/s30
mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for c in 1 2; do
timeout 200 env DFFTB_DMA=1 DFFTB_OVERLAP_CHUNKS=$c DFFTB_OP_TIMES=1 $TR --nproc-per-node 2 --master-port 2969$c bench.py --gpus 2 --steps 3 --warmup 3 > $O/optimes_dma_c$c.log 2>&1
echo "== C=$c"; grep "rank 0" $O/optimes_dma_c$c.log | head -16
done
echo done
