#!/bin/bash
# round-2 GPU session 23 (4 GPUs): full GPU test suite and final-code bench lines / configs at N=1/2/4
O=gpurun_out/s23
mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 1500 python -m pytest tests -m gpu -q -s > $O/pytest_gpu.log 2>&1; echo "exit $?" >> $O/pytest_gpu.log
timeout 300 python bench.py > $O/bench_n1.log 2>&1
timeout 300 $TR --nproc-per-node 2 --master-port 29671 bench.py --gpus 2 > $O/bench_n2.log 2>&1
timeout 300 $TR --nproc-per-node 4 --master-port 29672 bench.py --gpus 4 > $O/bench_n4.log 2>&1
timeout 300 python tools/bench_configs.py > $O/configs_n1.log 2>&1
timeout 400 $TR --nproc-per-node 2 --master-port 29673 tools/bench_configs.py > $O/configs_n2.log 2>&1
timeout 400 $TR --nproc-per-node 4 --master-port 29674 tools/bench_configs.py > $O/configs_n4.log 2>&1
for s in "DFFTB_RHALF=0"; do
  echo "== $s" >> $O/ab.log
  for c in B E; do timeout 300 env $s ONLY=$c python tools/bench_configs.py >> $O/ab.log 2>&1; done
done
timeout 200 python tools/op_times_config.py 2048,512,256 r2c f32 pencil >> $O/ab.log 2>&1
echo done
