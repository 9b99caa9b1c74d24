#!/bin/bash
# round-2 GPU session 9 (2 GPUs): co-resident overlapped exchange/local pass pairs
O=gpurun_out/s9
mkdir -p $O
B="--steps 10 --warmup 3 --no-e2e --no-cpu-baseline"
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
timeout 600 python -m pytest tests/test_multigpu.py -x -q -s > $O/pytest_mgpu.log 2>&1; echo "exit $?" >> $O/pytest_mgpu.log
for s in "DFFTB_OVERLAP=0" "DFFTB_OVERLAP=1" "DFFTB_OVERLAP=1 DFFTB_OVERLAP_CHUNKS=2" "DFFTB_OVERLAP=1 DFFTB_OVERLAP_CHUNKS=8" "DFFTB_OVERLAP=1 DFFTB_OVERLAP_CORES=0"; do
  echo "== $s" >> $O/bench.log
  timeout 200 env $s $TR --master-port 29641 bench.py --gpus 2 $B >> $O/bench.log 2>&1
done
echo done
