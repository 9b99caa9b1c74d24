#!/bin/bash
# round-2 GPU session 52 (1 GPU): rows lane stride as the default -- GPU suite, configs, E op times
O=gpurun_out/s52
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "exit $?" >> $O/pytest_gpu.log
tail -5 $O/pytest_gpu.log
timeout 400 python tools/bench_configs.py >> $O/configs.log 2>&1; timeout 300 python bench.py > $O/bench_n1.log 2>&1; grep -o "\"ms_per_step\": [0-9.]*" $O/bench_n1.log | head -1
grep config $O/configs.log | sed 's/"gflops.*//'
timeout 200 python tools/op_times_config.py 2048,512,256 r2c f32 pencil > $O/optimes_E.log 2>&1
cat $O/optimes_E.log
echo done
