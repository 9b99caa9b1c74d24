#!/bin/bash
# round-2 GPU session 37 (4 GPUs): staged exchange only where it pays (global-size rule) -- configs at N=2/4
O=gpurun_out/s37
mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 400 $TR --nproc-per-node 2 --master-port 29675 tools/bench_configs.py > $O/configs_n2.log 2>&1
timeout 400 $TR --nproc-per-node 4 --master-port 29676 tools/bench_configs.py > $O/configs_n4.log 2>&1
grep config $O/configs_n2.log $O/configs_n4.log
timeout 400 env DFFTB_DMA=0 $TR --nproc-per-node 2 --master-port 29677 tools/bench_configs.py > $O/configs_n2_direct.log 2>&1
timeout 400 env DFFTB_DMA=0 $TR --nproc-per-node 4 --master-port 29678 tools/bench_configs.py > $O/configs_n4_direct.log 2>&1
grep config $O/configs_n2_direct.log $O/configs_n4_direct.log
echo done
