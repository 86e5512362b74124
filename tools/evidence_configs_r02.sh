#!/bin/bash
# ncu --set full of one task-kernel launch per BASELINE config (this build), exported to raw csv.
mkdir -p gpurun_out
NCU="ncu --set full --clock-control none"
cap() { tag=$1; shift; timeout 900 $NCU -k "$KREGEX" -s ${SKIP:-1} -c 1 -o gpurun_out/$tag "$@" > gpurun_out/$tag.log 2>&1; echo "$tag rc=$?";
        ncu -i gpurun_out/$tag.ncu-rep --page raw --csv > gpurun_out/${tag}_raw.csv 2>/dev/null; rm -f gpurun_out/$tag.ncu-rep; }
KREGEX="regex:k_dmma" cap c1 python tools/profile_one.py --shape 2048,2048,2048
KREGEX="regex:k_dmma" cap c3a python tools/profile_one.py --shape 16384,16384,256
KREGEX="regex:k_dmma" cap c3b python tools/profile_one.py --shape 512,512,131072
KREGEX="regex:k_dmma" cap c3c python tools/profile_one.py --shape 65536,256,1024 --family B2A1C0
KREGEX="regex:k_tc2" SKIP=3 TC_CASES=bf16:256:512 TC_CUBLAS=0 cap c4bf16 python tools/bench_tc.py
KREGEX="regex:k_tc2" SKIP=3 TC_CASES=tf32:256:512 TC_CUBLAS=0 cap c4tf32 python tools/bench_tc.py
