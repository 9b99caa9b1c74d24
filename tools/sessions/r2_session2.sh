#!/bin/bash
# round-2 GPU session 2 (2 GPUs): restructured executor (program cache,
# graphs, overlapped exchange): full GPU tests, N=1 and N=2 A/B benches
O=gpurun_out/s2
mkdir -p $O
B="--steps 10 --warmup 3 --no-e2e --no-cpu-baseline"
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "exit $?" >> $O/pytest_gpu.log
timeout 200 python bench.py $B > $O/bench_n1.log 2>&1
timeout 200 env DFFTB_GRAPHS=0 python bench.py $B > $O/bench_n1_nograph.log 2>&1
timeout 300 python tools/bench_configs.py > $O/configs_n1.log 2>&1
timeout 120 env DFFTB_GRAPHS=0 ONLY=A python tools/bench_configs.py > $O/configA_nograph.log 2>&1
for s in "DFFTB_OVERLAP=1" "DFFTB_OVERLAP=0" "DFFTB_OVERLAP_CHUNKS=8" "DFFTB_OVERLAP_CHUNKS=2" "DFFTB_OVERLAP_FRAC=0.4" "DFFTB_OVERLAP_FRAC=0.6"; do
  echo "== $s" >> $O/bench_n2.log
  timeout 200 env $s $TR --master-port 29621 bench.py --gpus 2 $B >> $O/bench_n2.log 2>&1
done
timeout 200 env DFFTB_OP_TIMES=1 $TR --master-port 29622 bench.py --gpus 2 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > $O/optimes_n2.log 2>&1
timeout 300 $TR --master-port 29623 tools/bench_configs.py > $O/configs_n2.log 2>&1
echo done
