#!/bin/bash
# round-2 GPU session 73 (2 GPUs): staging agreement across ranks (handle flag) -- multi-GPU tests and bench N=2
O=gpurun_out/s73
mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 900 python -m pytest tests/test_multigpu.py -q -s > $O/pytest_mgpu.log 2>&1; echo "exit $?" >> $O/pytest_mgpu.log
grep -E "passed|failed|exit|FAIL" $O/pytest_mgpu.log
timeout 200 $TR --nproc-per-node 2 --master-port 29671 bench.py --gpus 2 --no-e2e > $O/b.log 2>&1
grep -o '"ms_per_step": [0-9.]*' $O/b.log | head -1
echo done
