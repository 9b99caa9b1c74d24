#!/bin/bash
# round-2 GPU session 5 (1 GPU): gather-chain lowering, PDL
O=gpurun_out/s5
mkdir -p $O
timeout 600 env DFFTB_CHAIN=1 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py -m gpu -x -q > $O/pytest_chain_forced.log 2>&1; echo "exit $?" >> $O/pytest_chain_forced.log
timeout 600 python -m pytest tests -m gpu -x -q --ignore=tests/test_fullsize_ref.py > $O/pytest_gpu.log 2>&1; echo "exit $?" >> $O/pytest_gpu.log
timeout 300 python tools/bench_configs.py > $O/configs_n1.log 2>&1
for s in "DFFTB_CHAIN=0" "DFFTB_CHAIN=1" "DFFTB_PDL=0"; do
  echo "== $s" >> $O/configs_ab.log
  timeout 300 env $s python tools/bench_configs.py >> $O/configs_ab.log 2>&1
done
for c in "2048,512,256 r2c f32 pencil" "1024,1024,1024 c2c f64 pencil" "256,256,256 r2c f64 slab" "512,512,512 c2c f64 pencil" "64,64,64 c2c f64 slab"; do
  echo "== $c" >> $O/optimes.log
  timeout 200 python tools/op_times_config.py $c >> $O/optimes.log 2>&1
  echo "== CHAIN=0 $c" >> $O/optimes.log
  timeout 200 env DFFTB_CHAIN=0 python tools/op_times_config.py $c >> $O/optimes.log 2>&1
done
echo done
