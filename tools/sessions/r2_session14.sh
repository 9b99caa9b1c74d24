#!/bin/bash
# round-2 GPU session 14 (4 GPUs): final-code evidence: full GPU test suite, bench lines at N=1/2/4
# (driver defaults: e2e + cpu_baseline at N=1), all configs at N=2/4, the reference arm
O=gpurun_out/s14
mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 1500 python -m pytest tests -m gpu -x -q -s > $O/pytest_gpu.log 2>&1; echo "exit $?" >> $O/pytest_gpu.log
timeout 300 python bench.py > $O/bench_n1.log 2>&1
timeout 300 $TR --nproc-per-node 2 --master-port 29651 bench.py --gpus 2 > $O/bench_n2.log 2>&1
timeout 300 $TR --nproc-per-node 4 --master-port 29652 bench.py --gpus 4 > $O/bench_n4.log 2>&1
timeout 400 $TR --nproc-per-node 2 --master-port 29653 tools/bench_configs.py > $O/configs_n2.log 2>&1
timeout 400 $TR --nproc-per-node 4 --master-port 29654 tools/bench_configs.py > $O/configs_n4.log 2>&1
timeout 300 python tools/bench_configs.py > $O/configs_n1.log 2>&1
timeout 300 python bench.py --impl reference > $O/bench_ref.log 2>&1
echo done
