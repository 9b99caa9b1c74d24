#!/bin/bash
# round-2 GPU session 60 (4 GPUs): staged exchange with the last k of 8 chunks stored to the peers directly (DFFTB_DMA_DIRECT=k) at N=2 / N=4; parity at 4 GPUs
O=gpurun_out/s60
mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 300 env DFFTB_DMA_DIRECT=3 DFFTB_DMA_MIN_MB=0 DFFTB_DMA_MIN_ROW=0 $TR --nproc-per-node 4 --master-port 29681 tests/mgpu_check.py > $O/mgpu4.log 2>&1; echo "exit $?" >> $O/mgpu4.log
grep -c "^ok" $O/mgpu4.log; grep FAIL $O/mgpu4.log; tail -1 $O/mgpu4.log
for n in 2 4; do
for k in 0 2 3 4 0; do
  timeout 200 env DFFTB_DMA_DIRECT=$k $TR --nproc-per-node $n --master-port $((29600 + RANDOM % 300)) bench.py --gpus $n --no-e2e > $O/b.log 2>&1
  echo "N=$n k=$k: $(grep -o '"ms_per_step": [0-9.]*' $O/b.log | head -1)"
done
done
echo done
