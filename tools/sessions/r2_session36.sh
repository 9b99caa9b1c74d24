#!/bin/bash
# round-2 GPU session 36 (4 GPUs): staged exchange as the default -- multi-GPU tests, bench lines, configs
O=gpurun_out/s36
mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 900 python -m pytest tests/test_multigpu.py -q -s > $O/pytest_mgpu.log 2>&1; echo "exit $?" >> $O/pytest_mgpu.log
grep -E "^ok|FAIL|passed|failed|exit" $O/pytest_mgpu.log | tail -30
timeout 300 python bench.py > $O/bench_n1.log 2>&1
timeout 300 $TR --nproc-per-node 2 --master-port 29671 bench.py --gpus 2 > $O/bench_n2.log 2>&1
timeout 300 $TR --nproc-per-node 4 --master-port 29672 bench.py --gpus 4 > $O/bench_n4.log 2>&1
timeout 300 env DFFTB_DMA=0 $TR --nproc-per-node 2 --master-port 29673 bench.py --gpus 2 > $O/bench_n2_direct.log 2>&1
timeout 300 env DFFTB_DMA=0 $TR --nproc-per-node 4 --master-port 29674 bench.py --gpus 4 > $O/bench_n4_direct.log 2>&1
for f in $O/bench_*.log; do echo "$f: $(grep -o '"ms_per_step": [0-9.]*' $f | head -1)"; done
timeout 400 $TR --nproc-per-node 2 --master-port 29675 tools/bench_configs.py > $O/configs_n2.log 2>&1
timeout 400 $TR --nproc-per-node 4 --master-port 29676 tools/bench_configs.py > $O/configs_n4.log 2>&1
tail -6 $O/configs_n2.log $O/configs_n4.log
echo done
