#!/bin/bash
# round-2 GPU session 6 (4 GPUs): multi-process parity at 2 and 4 GPUs, N=2/4 benches (overlap A/B),
# all configs at N=4, NVLink byte counters of the exchange passes (one-process world, ncu)
O=gpurun_out/s6
mkdir -p $O
B="--steps 10 --warmup 3 --no-e2e --no-cpu-baseline"
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
nvidia-smi topo -m > $O/topo.txt 2>&1
timeout 900 python -m pytest tests/test_multigpu.py -x -q -s > $O/pytest_mgpu.log 2>&1; echo "exit $?" >> $O/pytest_mgpu.log
for s in "DFFTB_OVERLAP=1" "DFFTB_OVERLAP=0"; do
  echo "== N=4 $s" >> $O/bench.log
  timeout 200 env $s $TR --nproc-per-node 4 --master-port 29631 bench.py --gpus 4 $B >> $O/bench.log 2>&1
  echo "== N=2 $s" >> $O/bench.log
  timeout 200 env $s $TR --nproc-per-node 2 --master-port 29632 bench.py --gpus 2 $B >> $O/bench.log 2>&1
done
timeout 400 $TR --nproc-per-node 4 --master-port 29633 tools/bench_configs.py > $O/configs_n4.log 2>&1
timeout 300 python tools/nvl_pass_probe.py --grid 2,2 --reps 1 > $O/nvl_probe.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,nvltx__bytes.sum,nvlrx__bytes.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  -k regex:fft_pass_tma --clock-control none -c 12 --csv --log-file $O/ncu_nvl.csv \
  python tools/nvl_pass_probe.py --grid 2,2 --reps 1 > $O/ncu_nvl.log 2>&1
echo done
