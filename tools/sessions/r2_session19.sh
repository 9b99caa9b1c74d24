#!/bin/bash
# round-2 GPU session 19 (1 GPU): pair-interleaved single-rank buffers for narrow strided passes
O=gpurun_out/s19
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_spectral_golden.py -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "exit $?" >> $O/pytest_gpu.log
for s in "" "DFFTB_PAIR2=0"; do
  echo "== ${s:-default}" >> $O/ab.log
  for c in D E C; do timeout 300 env $s ONLY=$c python tools/bench_configs.py >> $O/ab.log 2>&1; done
  for c in "2048,512,256 r2c f32 pencil" "1024,1024,1024 c2c f64 pencil"; do timeout 200 env $s python tools/op_times_config.py $c >> $O/ab.log 2>&1; done
done
echo done
