#!/bin/bash
# round-2 GPU session 55 (4 GPUs): config E at N=2/4 with the staged exchange allowed on 512-byte rows (DFFTB_DMA_MIN_ROW=512) and 4 chunks
O=gpurun_out/s55
mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for n in 2 4; do
for v in "X=1" "DFFTB_DMA_MIN_ROW=512" "DFFTB_DMA_MIN_ROW=512 DFFTB_DMA_CHUNKS=4" "DFFTB_DMA_MIN_ROW=256 DFFTB_DMA_CHUNKS=4"; do
  echo "== N=$n $v" >> $O/ab.log
  timeout 300 env $v ONLY=E $TR --nproc-per-node $n --master-port $((29700 + RANDOM % 200)) tools/bench_configs.py 2>&1 | grep config >> $O/ab.log
done
done
cat $O/ab.log | sed 's/"gflops.*//'
echo done
