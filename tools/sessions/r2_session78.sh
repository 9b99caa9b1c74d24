#!/bin/bash
# round-2 GPU session 78 (4 GPUs): staged exchange with one copy stream per remote member (DFFTB_DMA_PERMEMBER=1) for groups of 4 -- correctness and group probe
O=gpurun_out/s78
mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 300 env DFFTB_DMA_PERMEMBER=1 DFFTB_DMA_MAX_GROUP=64 DFFTB_DMA_MIN_MB=0 DFFTB_DMA_MIN_ROW=0 DFFTB_EXPECT_STAGED=1 $TR --nproc-per-node 4 --master-port 29504 tests/mgpu_check.py > $O/mgpu4.log 2>&1; echo "exit $?" >> $O/mgpu4.log
echo "mgpu 4: $(grep -c '^ok' $O/mgpu4.log) ok, $(grep -c FAIL $O/mgpu4.log) FAIL, $(tail -1 $O/mgpu4.log)"
for v in X=1 "DFFTB_DMA_MAX_GROUP=4 DFFTB_DMA_PERMEMBER=1" "DFFTB_DMA_MAX_GROUP=4"; do echo "== $v"; timeout 300 env $v $TR --nproc-per-node 4 --master-port $((29600 + RANDOM % 300)) tools/group_probe.py 2>&1 | grep "ms per"; done
echo done
