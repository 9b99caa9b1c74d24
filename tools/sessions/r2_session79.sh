#!/bin/bash
# round-2 GPU session 79 (4 GPUs): last full check of the final code (staging limited to groups of two) -- pytest -m gpu, bench lines at N=1/2/4, reference arm
O=gpurun_out/s79
mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 1800 python -m pytest tests -m gpu -q -s > $O/pytest_gpu.log 2>&1; echo "exit $?" >> $O/pytest_gpu.log
tail -3 $O/pytest_gpu.log
timeout 300 python bench.py > $O/bench_n1.log 2>&1
timeout 300 $TR --nproc-per-node 2 --master-port 29671 bench.py --gpus 2 > $O/bench_n2.log 2>&1
timeout 300 $TR --nproc-per-node 4 --master-port 29672 bench.py --gpus 4 > $O/bench_n4.log 2>&1
timeout 300 $TR --nproc-per-node 4 --master-port 29673 bench.py --impl reference --gpus 4 --steps 2 --warmup 1 > $O/bench_ref_n4.log 2>&1
for f in $O/bench_n*.log; do echo "$f: $(grep -o '"ms_per_step": [0-9.]*' $f | head -1)"; done
grep -c '^{' $O/bench_ref_n4.log
echo done
