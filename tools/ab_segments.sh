#!/bin/bash
# FP64 16384^3 bench (device arm only) across TMA segment lengths (TILEMUL_TMA_SEGMENT_SLABS), 2 rounds.
for rep in 1 2; do for v in ${SEGS:-4096 6144 8192 12288}; do
  TILEMUL_TMA_SEGMENT_SLABS=$v timeout 300 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('seg=$v', round(d['value'],3), round(d['pct_of_fp64_peak'],2), d['roofline']['launches_per_step'])"
done; done
for v in ${SEGS:-4096 6144 8192 12288}; do
  TILEMUL_TMA_SEGMENT_SLABS=$v timeout 600 ncu --clock-control none --metrics dram__bytes_read.sum -k regex:k_dmma_tma --csv \
    python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu --no-verify 2>/dev/null | grep dram__bytes_read | \
    awk -F'","' -v v=$v '{gsub(/"/,"",$NF); s+=$NF} END {print "seg=" v " dram_read_GB_first_step(sum of launches) " s/1e9}'
done
