#!/bin/bash
# DRAM bytes per task-kernel launch for each library variant in exp_libs/
# (one ncu process per variant, metrics only): tools/dram_ab.sh old base
for v in "$@"; do
  TILEMUL_B200_LIB=$PWD/exp_libs/$v.so timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct \
    -k "regex:k_dmma($|<)" --csv --log-file gpurun_out/dram_$v.csv \
    python tools/sweep.py --once --tiles auto --members C2A1C0 --l2-frac ${L2FRAC:-0.25} --only ${ONLY:-config2,config3a_rank_k} > /dev/null 2>&1
  echo "== $v rc=$?"
  python - "$v" <<'PY'
import csv, sys
v = sys.argv[1]
rows = list(csv.reader(open(f"gpurun_out/dram_{v}.csv")))
i = [k for k, r in enumerate(rows) if r and r[0] == "ID"][0]
h = rows[i]
by = {}
for r in rows[i + 1:]:
    d = dict(zip(h, r))
    by.setdefault(d["ID"], {})[d["Metric Name"]] = (d["Metric Value"], d["Metric Unit"])
for k, m in by.items():
    print(k, {n: m[n] for n in sorted(m)})
PY
done
