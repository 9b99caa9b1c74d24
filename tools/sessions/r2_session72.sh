#!/bin/bash
# round-2 GPU session 72 (4 GPUs): staged-exchange signal kernels on their own streams (DFFTB_DMA_SIGSTREAM=1) -- parity (staging forced) at 2/4 GPUs, bench A/B at N=2/4
O=gpurun_out/s72
mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for n in 2 4; do
timeout 300 env DFFTB_DMA_SIGSTREAM=1 DFFTB_DMA_MIN_MB=0 DFFTB_DMA_MIN_ROW=0 DFFTB_EXPECT_STAGED=1 $TR --nproc-per-node $n --master-port $((29500 + n)) tests/mgpu_check.py > $O/mgpu$n.log 2>&1; echo "exit $?" >> $O/mgpu$n.log
echo "mgpu $n: $(grep -c '^ok' $O/mgpu$n.log) ok, $(grep -c FAIL $O/mgpu$n.log) FAIL, $(tail -1 $O/mgpu$n.log)"
done
for n in 2 4; do
for v in "X=1" "DFFTB_DMA_SIGSTREAM=1" "X=1" "DFFTB_DMA_SIGSTREAM=1"; do
  timeout 200 env $v $TR --nproc-per-node $n --master-port $((29600 + RANDOM % 300)) bench.py --gpus $n --no-e2e > $O/b.log 2>&1
  echo "N=$n $v: $(grep -o '"ms_per_step": [0-9.]*' $O/b.log | head -1) rt $(grep -o '"roundtrip_rel_l2": [0-9.e-]*' $O/b.log | head -1)"
done
done
for n in 2 4; do echo "D N=$n sigstream: $(timeout 400 env DFFTB_DMA_SIGSTREAM=1 ONLY=D $TR --nproc-per-node $n --master-port $((29600 + RANDOM % 300)) tools/bench_configs.py 2>&1 | grep config | sed 's/"gflops.*//')"; done
echo done
