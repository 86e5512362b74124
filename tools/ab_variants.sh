#!/bin/bash
# A/B of library builds in exp_libs/<name>.so over the FP64 configs (tools/sweep.py --quick, C2A1C0, auto tiles),
# REPS alternating rounds:  REPS=2 ONLY=config1,... tools/ab_variants.sh base variant ...
REPS=${REPS:-2}
for rep in $(seq $REPS); do for v in "$@"; do
  TILEMUL_B200_LIB=$PWD/exp_libs/$v.so timeout 600 python tools/sweep.py --quick --members C2A1C0 --tiles auto \
    --only ${ONLY:-config1,config3a_rank_k,config3b_inner_product,config3c_panel_panel,config2} 2>/dev/null \
   | python -c "import json,sys
for l in sys.stdin:
    d=json.loads(l)
    if 'error' in d: print('$v', d['config'], 'ERR', d['error'][:80])
    elif 'tflops' in d: print('$v', d['config'], d['shape'], d['launch'].get('staging'), d['launch'].get('launches'), round(d['pct_fp64_peak'],2))"
done; done
