#!/bin/bash
# round-2 GPU session 58 (4 GPUs): DFFTB_DMA_CHAIN=1 (stage the first exchange of a direction too; its consumer exchange pass runs in chunks with direct peer stores) at N=4 / N=2; parity at 4 GPUs
O=gpurun_out/s58
mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 300 env DFFTB_DMA_CHAIN=1 DFFTB_DMA_MIN_MB=0 DFFTB_DMA_MIN_ROW=0 $TR --nproc-per-node 4 --master-port 29681 tests/mgpu_check.py > $O/mgpu4_chain.log 2>&1; echo "exit $?" >> $O/mgpu4_chain.log
grep -c "^ok" $O/mgpu4_chain.log; grep FAIL $O/mgpu4_chain.log; tail -1 $O/mgpu4_chain.log
for n in 4 2; do
for v in "X=1" "DFFTB_DMA_CHAIN=1" "X=1" "DFFTB_DMA_CHAIN=1"; do
  timeout 200 env $v $TR --nproc-per-node $n --master-port $((29600 + RANDOM % 300)) bench.py --gpus $n --no-e2e > $O/b.log 2>&1
  echo "N=$n $v: $(grep -o '"ms_per_step": [0-9.]*' $O/b.log | head -1)"
done
timeout 400 env DFFTB_DMA_CHAIN=1 ONLY=D $TR --nproc-per-node $n --master-port $((29600 + RANDOM % 300)) tools/bench_configs.py 2>&1 | grep config | sed 's/"gflops.*//'
done
echo done
