#!/bin/bash
# round-2 GPU session 61 (4 GPUs): config E at N=2/4 with the [x1][x0][x2] axis-0 buffer kept (DFFTB_DMA_FLAT=0; E's exchanges are not staged) vs default
O=gpurun_out/s61
mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for n in 2 4; do
for v in "X=1" "DFFTB_DMA_FLAT=0" "X=1" "DFFTB_DMA_FLAT=0"; do
  echo "N=$n $v: $(timeout 300 env $v ONLY=E $TR --nproc-per-node $n --master-port $((29600 + RANDOM % 300)) tools/bench_configs.py 2>&1 | grep config | sed 's/"gflops.*//')"
done
done
echo done
