#!/bin/bash
# A/B sweep of library builds in exp_libs/<name>.so (TILEMUL_B200_LIB): prints
# TFLOP/s and % of the FP64 peak per config for each variant, same process
# layout as tools/sweep.py. ONLY=<configs> narrows the sweep.
#   tools/ab_libs.sh base variant [base variant ...]
for v in "$@"; do
  echo "== $v"
  TILEMUL_B200_LIB=$PWD/exp_libs/$v.so timeout 300 python tools/sweep.py --tiles ${TILES:-auto} --staging ${STAGING:-auto} --members C2A1C0 --only ${ONLY:-config1,config3a_rank_k,config3c_panel_panel} 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l)
    if 'error' in d: print(d['config'], 'ERR', d['error'][:80]); continue
    print(d['config'], d['shape'], d['cta_tile'], d['launch'].get('staging'), round(d['tflops'],2), round(d['pct_fp64_peak'],1))"
done
