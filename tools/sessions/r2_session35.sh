#!/bin/bash
# round-2 GPU session 35 (4 GPUs): staged exchange copy-stream count and chunk sweep at N=2 and N=4
O=gpurun_out/s35
mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
run() {  # name gpus env...
  local name=$1 g=$2; shift 2
  timeout 200 env "$@" $TR --nproc-per-node $g --master-port $((29600 + RANDOM % 300)) bench.py --gpus $g > $O/$name.log 2>&1
  echo "$name: $(grep -o '"ms_per_step": [0-9.]*' $O/$name.log | head -1)"
}
run n2_default 2 X=1
for ns in 2 3 4; do for c in 8 16; do run n2_c${c}_s$ns 2 DFFTB_DMA=1 DFFTB_DMA_STREAMS=$ns DFFTB_OVERLAP_CHUNKS=$c; done; done
run n4_default 4 X=1
for ns in 1 2 4; do for c in 4 8 16; do run n4_c${c}_s$ns 4 DFFTB_DMA=1 DFFTB_DMA_STREAMS=$ns DFFTB_OVERLAP_CHUNKS=$c; done; done
echo done
