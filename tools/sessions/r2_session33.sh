#!/bin/bash
# round-2 GPU session 33 (4 GPUs): staged exchange parity and A/B at N=4
O=gpurun_out/s33
mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 300 env DFFTB_DMA=1 $TR --nproc-per-node 4 --master-port 29681 tests/mgpu_check.py > $O/mgpu4_dma.log 2>&1; echo "exit $?" >> $O/mgpu4_dma.log
grep -c "^ok" $O/mgpu4_dma.log; grep FAIL $O/mgpu4_dma.log; tail -1 $O/mgpu4_dma.log
timeout 200 $TR --nproc-per-node 4 --master-port 29682 bench.py --gpus 4 > $O/bench_n4_default.log 2>&1
for c in 4 8 16; do
  timeout 200 env DFFTB_DMA=1 DFFTB_OVERLAP_CHUNKS=$c $TR --nproc-per-node 4 --master-port 2969$((c % 10)) bench.py --gpus 4 > $O/bench_n4_dma_c$c.log 2>&1
done
timeout 200 env DFFTB_DMA=1 DFFTB_OVERLAP_CHUNKS=16 $TR --nproc-per-node 2 --master-port 29688 bench.py --gpus 2 > $O/bench_n2_dma_c16.log 2>&1
timeout 200 env DFFTB_DMA=1 DFFTB_OVERLAP_CHUNKS=8 DFFTB_OP_TIMES=1 $TR --nproc-per-node 4 --master-port 29689 bench.py --gpus 4 --steps 3 --warmup 3 > $O/optimes_n4_dma.log 2>&1
for f in $O/bench_n*.log; do echo "$f: $(grep -o '"ms_per_step": [0-9.]*' $f | head -1)"; done
grep "rank 0" $O/optimes_n4_dma.log | head -60
echo done
