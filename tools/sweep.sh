#!/bin/bash
# A/B sweep of experimental library builds in exp/ (N=1 bench, compact output)
for lib in "" $(ls exp/*.so 2>/dev/null); do
  name=${lib:-default}
  DFFTB_LIB_OVERRIDE=${lib:+$PWD/$lib} python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null \
   | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$name', round(d['ms_per_step'],3), round(d['roofline']['frac'],3), {k: round(v,3) for k,v in d['fwd_breakdown_ms'].items()})"
done
