#!/bin/bash
# round-2 GPU session 4 (2 GPUs): chain lowering correctness + speed, D at full size vs the reference
O=gpurun_out/s4
mkdir -p $O
timeout 600 env DFFTB_CHAIN=1 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py -m gpu -x -q > $O/pytest_chain_forced.log 2>&1; echo "exit $?" >> $O/pytest_chain_forced.log
timeout 600 python -m pytest tests -m gpu -x -q --ignore=tests/test_fullsize_ref.py > $O/pytest_gpu.log 2>&1; echo "exit $?" >> $O/pytest_gpu.log
timeout 300 python tools/bench_configs.py > $O/configs_n1.log 2>&1
timeout 200 env DFFTB_CHAIN=0 ONLY=D python tools/bench_configs.py > $O/configD_nochain.log 2>&1
timeout 200 env DFFTB_CHAIN=0 ONLY=E python tools/bench_configs.py > $O/configE_nochain.log 2>&1
timeout 200 env DFFTB_CHAIN=1 ONLY=C python tools/bench_configs.py > $O/configC_chain.log 2>&1
timeout 200 env DFFTB_CHAIN=1 ONLY=B python tools/bench_configs.py > $O/configB_chain.log 2>&1
for c in "2048,512,256 r2c f32 pencil" "1024,1024,1024 c2c f64 pencil" "256,256,256 r2c f64 slab"; do
  echo "== $c" >> $O/optimes.log
  timeout 200 python tools/op_times_config.py $c >> $O/optimes.log 2>&1
done
timeout 1500 env DFFTB_TEST_HUGE=1 python -m pytest tests/test_fullsize_ref.py -m gpu -q -s -k huge > $O/pytest_huge.log 2>&1; echo "exit $?" >> $O/pytest_huge.log
free -g >> $O/pytest_huge.log
echo done
