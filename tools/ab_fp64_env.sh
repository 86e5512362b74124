#!/bin/bash
# FP64 A/B over one environment knob (tools/sweep.py, C2A1C0, auto tiles): tools/ab_fp64_env.sh VAR "v1 v2" [reps]
VAR=$1; VALS=$2; REPS=${3:-2}
for rep in $(seq $REPS); do for v in $VALS; do
  env $VAR=$v timeout 600 python tools/sweep.py --only ${ONLY:-config1,config3a_rank_k,config3b_inner_product,config3c_panel_panel,config2} --quick --members C2A1C0 --tiles auto 2>/dev/null \
   | python -c "import json,sys
for l in sys.stdin:
    d=json.loads(l)
    if 'tflops' in d: print('$VAR=$v', d['config'], d['shape'], round(d['pct_fp64_peak'],2))"
done; done
