#!/bin/bash
# A/B sweep of environment settings (N=1 bench, compact output):
#   bash tools/envsweep.sh "" "DFFTB_GRAPHS=0" "DFFTB_L2PROMO=2"
for setting in "$@"; do
  env $setting python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null \
   | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('[$setting]', round(d['ms_per_step'],3), round(d['roofline']['frac'],3), d['roundtrip_rel_l2'], {k: round(v,3) for k,v in d['fwd_breakdown_ms'].items()})"
done
