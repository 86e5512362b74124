#!/bin/bash
# FP64 16384^3 bench (device arm) with/without programmatic dependent launch between TMA segments.
timeout 600 python -m pytest tests/test_gpu_tma.py tests/test_gpu_baseline_shapes.py -q -m gpu -x > gpurun_out/pdl_tests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/pdl_tests.log
for rep in 1 2 3; do for v in 0 1; do
  TILEMUL_TMA_PDL=$v timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('pdl=$v', round(d['value'],3), round(d['pct_of_fp64_peak'],2), d['verified']['ok'])"
done; done
for v in 0 1; do
  TILEMUL_TMA_PDL=$v timeout 600 ncu --clock-control none --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum -k regex:k_dmma_tma --csv \
    python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu --no-verify 2>/dev/null | grep -E 'dram__bytes|gpu__time' | \
    awk -F'","' -v v=$v '{gsub(/"/,"",$NF); s[$(NF-2)]+=$NF} END {for (k in s) print "pdl=" v, k, s[k]}'
done
