#!/bin/bash
# round-2 GPU session 44 (1 GPU): radix-16 / 256-thread 1024-point fp64 default -- GPU suite, configs, headline
O=gpurun_out/s44
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "exit $?" >> $O/pytest_gpu.log
tail -3 $O/pytest_gpu.log
timeout 400 python tools/bench_configs.py > $O/configs_n1.log 2>&1
grep config $O/configs_n1.log | sed 's/"gflops.*//'
timeout 300 python bench.py > $O/bench_n1.log 2>&1
grep -o '"ms_per_step": [0-9.]*' $O/bench_n1.log | head -1
echo done
