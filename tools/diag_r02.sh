#!/bin/bash
# Round-2 diagnostics: ncu --set full of the short-k FP64 launches (rank-k, 2048^3)
# and of the config-4 tcgen05 pair kernels (tf32, bf16), exported to csv on the box.
mkdir -p gpurun_out
NCU="ncu --set full --clock-control none --import-source on"
exp() { ncu -i gpurun_out/$1.ncu-rep --page raw --csv > gpurun_out/$1_raw.csv 2>/dev/null;
        ncu -i gpurun_out/$1.ncu-rep --page source --csv --print-source sass > gpurun_out/$1_src.csv 2>/dev/null; }
python tools/profile_one.py --shape 16384,16384,256 --staging tma > /dev/null 2>&1 && \
  timeout 600 $NCU -k "regex:k_dmma" -s 1 -c 1 -o gpurun_out/rankk python tools/profile_one.py --shape 16384,16384,256 --staging tma > gpurun_out/rankk.log 2>&1; exp rankk
timeout 600 $NCU -k "regex:k_dmma" -s 1 -c 1 -o gpurun_out/sq2048 python tools/profile_one.py --shape 2048,2048,2048 > gpurun_out/sq2048.log 2>&1; exp sq2048
TC_CASES=tf32:256:512 TC_CUBLAS=0 timeout 900 $NCU -k "regex:k_tc2" -s 3 -c 1 -o gpurun_out/tf32w python tools/bench_tc.py > gpurun_out/tf32w.log 2>&1; exp tf32w
TC_CASES=tf32:256:512,bf16:256:512 TC_CUBLAS=1 timeout 600 python tools/bench_tc.py > gpurun_out/tc_bench.log 2>&1
ls -la gpurun_out
