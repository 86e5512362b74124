#!/bin/bash
# First-contact probe on the GPU box: FP64 peaks, device properties, host cores.
mkdir -p gpurun_out
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.sw_power_cap --format=csv -lms 200 > gpurun_out/probe_clocks.csv &
SMI=$!
./tools/fp64_peak > gpurun_out/fp64_peak.jsonl 2>&1
kill $SMI
nproc > gpurun_out/host.txt; lscpu >> gpurun_out/host.txt; free -g >> gpurun_out/host.txt
nvidia-smi >> gpurun_out/host.txt
ncu --version >> gpurun_out/host.txt 2>&1
cat gpurun_out/fp64_peak.jsonl
