#!/bin/bash
# round-2 GPU session 34 (2 GPUs): staged exchange, 1 vs 2 copy streams, repeat A/B at N=2
O=gpurun_out/s34
mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 300 env DFFTB_DMA=1 DFFTB_DMA_STREAMS=2 $TR --nproc-per-node 2 --master-port 29681 tests/mgpu_check.py > $O/mgpu2_dma2.log 2>&1; echo "exit $?" >> $O/mgpu2_dma2.log
tail -1 $O/mgpu2_dma2.log
for rep in 1 2; do
timeout 200 $TR --nproc-per-node 2 --master-port 29682 bench.py --gpus 2 > $O/bench_n2_default_$rep.log 2>&1
for c in 4 8; do
  for ns in 1 2; do
  timeout 200 env DFFTB_DMA=1 DFFTB_DMA_STREAMS=$ns DFFTB_OVERLAP_CHUNKS=$c $TR --nproc-per-node 2 --master-port 2968$c bench.py --gpus 2 > $O/bench_n2_dma_c${c}_s${ns}_$rep.log 2>&1
  done
done
done
timeout 200 env DFFTB_DMA=1 DFFTB_DMA_STREAMS=2 DFFTB_OVERLAP_CHUNKS=8 DFFTB_OP_TIMES=1 $TR --nproc-per-node 2 --master-port 29689 bench.py --gpus 2 --steps 3 --warmup 3 > $O/optimes_dma2.log 2>&1
for f in $O/bench_n2_*.log; do echo "$f: $(grep -o '"ms_per_step": [0-9.]*' $f | head -1)"; done
grep "rank 0" $O/optimes_dma2.log | head -40
echo done
