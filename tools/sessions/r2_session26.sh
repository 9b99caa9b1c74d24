#!/bin/bash
# round-2 GPU session 26 (2 GPUs): staged (copy-engine) exchange -- parity and A/B at N=2
O=gpurun_out/s26
mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 300 $TR --nproc-per-node 2 --master-port 29681 tests/mgpu_check.py > $O/mgpu2.log 2>&1; echo "exit $?" >> $O/mgpu2.log
tail -3 $O/mgpu2.log
timeout 200 $TR --nproc-per-node 2 --master-port 29682 bench.py --gpus 2 > $O/bench_n2_default.log 2>&1
for c in 4 2 8; do
  timeout 200 env DFFTB_DMA=1 DFFTB_OVERLAP_CHUNKS=$c $TR --nproc-per-node 2 --master-port 2968$c bench.py --gpus 2 > $O/bench_n2_dma_c$c.log 2>&1
done
timeout 200 env DFFTB_DMA=1 DFFTB_OP_TIMES=1 $TR --nproc-per-node 2 --master-port 29689 bench.py --gpus 2 --steps 3 --warmup 3 > $O/optimes_dma.log 2>&1
timeout 200 env DFFTB_OP_TIMES=1 $TR --nproc-per-node 2 --master-port 29690 bench.py --gpus 2 --steps 3 --warmup 3 > $O/optimes_default.log 2>&1
for f in $O/bench_n2_*.log; do echo "$f: $(grep -o '"ms_per_step": [0-9.]*' $f)"; done
echo done
