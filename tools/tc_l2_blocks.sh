#!/bin/bash
# Config 4 across L2-block shapes of the 256x512 raster (TC_L2_BLOCK_WIDE): CUDA-event TF/s (bench_tc) and
# ncu DRAM reads of one launch. Usage: tools/tc_l2_blocks.sh "bf16:2048x4608 tf32:1024x1024 ..."
for c in $1; do
  dt=${c%%:*}; blk=${c##*:}
  TC_L2_BLOCK_WIDE=$blk TC_CASES=$dt:256:512 TC_CUBLAS=0 timeout 240 python tools/bench_tc.py | python -c "import json,sys
for l in sys.stdin:
    d=json.loads(l); print('$dt $blk tflops', round(d['tflops'],1))"
  TC_L2_BLOCK_WIDE=$blk TC_CASES=$dt:256:512 TC_CUBLAS=0 timeout 300 ncu --clock-control none --metrics dram__bytes_read.sum,gpu__time_duration.sum -k regex:k_tc2 -s 3 -c 1 --csv python tools/bench_tc.py 2>/dev/null | grep -E 'dram__bytes_read|gpu__time' | awk -F'","' -v c="$dt $blk" '{gsub(/"/,"",$NF); print c" ncu "$(NF-2)" "$NF}'
done
