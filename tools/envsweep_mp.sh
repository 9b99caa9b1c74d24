#!/bin/bash
# A/B sweep of environment settings for the N-GPU bench (first arg: N):
#   bash tools/envsweep_mp.sh 2 "DFFTB_OVERLAP=0" "DFFTB_OVERLAP_FRAC=0.5"
n=$1; shift
for setting in "$@"; do
  env $setting timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
    --master-port 29555 bench.py --gpus $n --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null \
   | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('[$setting]', round(d['ms_per_step'],3), d['roundtrip_rel_l2'], {k: round(v,3) for k,v in d['fwd_breakdown_ms'].items()})"
done
