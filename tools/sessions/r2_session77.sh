#!/bin/bash
# round-2 GPU session 77 (4 GPUs): staged exchange limited to groups of two (DFFTB_DMA_MAX_GROUP=2) -- group probe, multi-GPU tests, bench N=2/4
O=gpurun_out/s77
mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for v in X=1 DFFTB_DMA_MAX_GROUP=4; do echo "== $v"; timeout 300 env $v $TR --nproc-per-node 4 --master-port $((29600 + RANDOM % 300)) tools/group_probe.py 2>&1 | grep "ms per"; done
timeout 900 python -m pytest tests/test_multigpu.py -q -s > $O/pytest_mgpu.log 2>&1; echo "exit $?" >> $O/pytest_mgpu.log
grep -E "passed|failed|exit" $O/pytest_mgpu.log; grep -c "staged DMA exchange" $O/pytest_mgpu.log; grep FAIL $O/pytest_mgpu.log
for n in 2 4; do timeout 200 $TR --nproc-per-node $n --master-port $((29600 + RANDOM % 300)) bench.py --gpus $n --no-e2e > $O/b$n.log 2>&1; echo "N=$n: $(grep -o '"ms_per_step": [0-9.]*' $O/b$n.log | head -1)"; done
echo done
