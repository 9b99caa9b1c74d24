#!/bin/bash
# round-2 GPU session 10 (1 GPU): L2 promotion of the strided-lane tensor maps for narrow rows (D, E); config A with the new small-tile default
O=gpurun_out/s10
mkdir -p $O
for v in 0 1 2 3; do
  echo "== DFFTB_L2PROMO=$v" >> $O/l2promo.log
  for c in D E C; do timeout 300 env DFFTB_L2PROMO=$v ONLY=$c python tools/bench_configs.py >> $O/l2promo.log 2>&1; done
done
for c in "2048,512,256 r2c f32 pencil" "1024,1024,1024 c2c f64 pencil"; do
  for v in 1 3; do
    echo "== L2PROMO=$v $c" >> $O/optimes.log
    timeout 200 env DFFTB_L2PROMO=$v python tools/op_times_config.py $c >> $O/optimes.log 2>&1
  done
done
timeout 300 python tools/bench_configs.py > $O/configs_n1.log 2>&1
echo done
