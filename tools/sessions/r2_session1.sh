#!/bin/bash
# round-2 GPU session 1 (2 GPUs): topology, multi-GPU parity, benches, NVLink probe
set -x
O=gpurun_out/s1
mkdir -p $O
nvidia-smi topo -m > $O/topo.txt 2>&1
nvidia-smi > $O/smi.txt 2>&1
free -g > $O/free.txt; nproc > $O/nproc.txt; lscpu > $O/lscpu.txt
timeout 300 python -m pytest tests/test_multigpu.py -x -q -s > $O/pytest_mgpu.log 2>&1; echo "mgpu exit $?" >> $O/pytest_mgpu.log
timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus 2 --steps 10 --warmup 3 --no-e2e > $O/bench_n2.log 2>&1
timeout 200 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > $O/bench_n1.log 2>&1
timeout 120 tools/p2p_probe > $O/p2p_probe.txt 2>&1
timeout 120 env DFFTB_OP_TIMES=1 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29612 bench.py --gpus 2 --steps 2 --warmup 3 --no-e2e > $O/optimes_n2.log 2>&1
nvidia-smi nvlink -gt d > $O/nvlink_gt.txt 2>&1
echo done
