#!/bin/bash
# round-2 GPU session 49 (1 GPU): paired 16-byte cp.async loader for 8-byte-aligned fp32 rows -- GPU suite, E op times
O=gpurun_out/s49
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "exit $?" >> $O/pytest_gpu.log
tail -5 $O/pytest_gpu.log
for rep in 1 2; do timeout 300 env ONLY=E python tools/bench_configs.py >> $O/configs.log 2>&1; done
grep config $O/configs.log | sed 's/"gflops.*//'
timeout 200 python tools/op_times_config.py 2048,512,256 r2c f32 pencil > $O/optimes_E.log 2>&1
cat $O/optimes_E.log
echo done
