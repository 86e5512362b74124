#!/bin/bash
# DRAM bytes + duration of the bench's task kernel (16384^3, planner plan) for
# each library variant in exp_libs/: tools/dram_bench.sh old base ...
for v in "$@"; do
  TILEMUL_B200_LIB=$PWD/exp_libs/$v.so timeout 900 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct \
    --clock-control none -k "regex:k_dmma($|<)" -s 3 -c ${COUNT:-1} --csv --log-file gpurun_out/dramb_$v.csv \
    python bench.py --steps ${STEPS:-1} --warmup 3 --no-e2e --no-cpu ${SIZE:+--size $SIZE} > /dev/null 2>&1
  echo "== $v rc=$? $(grep -E 'dram__bytes_read|gpu__time|hit_rate' gpurun_out/dramb_$v.csv | awk -F'","' '{print $(NF-2), $(NF-1), $NF}' | tr '\n' ' ')"
done
