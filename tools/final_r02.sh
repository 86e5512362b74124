#!/bin/bash
# Round-2 closing pass on one B200: smoke, every GPU test, the headline bench line, the config-4 lines,
# then the headline kernel's launch list + --set full capture for roofline.traffic (this build's kernel id).
mkdir -p gpurun_out
python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/gputest.log 2>&1; echo "gpu tests rc=$?"; tail -2 gpurun_out/gputest.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?"
for c in 4 4tf32; do timeout 600 python bench.py --config $c --no-cpu > gpurun_out/bench_c$c.log 2>&1; echo "bench config $c rc=$?"; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r02_16384.csv \
  python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu > gpurun_out/ncu_launches.log 2>&1; echo "launch list rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_dmma_tma -c 14 -o gpurun_out/bench16k \
  python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu --no-verify > gpurun_out/ncu_full.log 2>&1; echo "full capture rc=$?"
ncu -i gpurun_out/bench16k.ncu-rep --page raw --csv > gpurun_out/bench16k_raw.csv 2>/dev/null; rm -f gpurun_out/bench16k.ncu-rep
