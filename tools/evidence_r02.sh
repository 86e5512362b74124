#!/bin/bash
# Round-2 evidence pass on one B200: the bench's own launch list and a --set full capture of one
# step's 14 task-kernel launches (bench traffic), then the model check's ncu metrics pass.
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r02_16384.csv \
  python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu > gpurun_out/ncu_launches.log 2>&1; echo "launch list rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_dmma_tma -c 14 -o gpurun_out/bench16k \
  python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu --no-verify > gpurun_out/ncu_full.log 2>&1; echo "full capture rc=$?"
ncu -i gpurun_out/bench16k.ncu-rep --page raw --csv > gpurun_out/bench16k_raw.csv 2>/dev/null; rm -f gpurun_out/bench16k.ncu-rep
timeout 2400 ncu --clock-control none --metrics dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_write.sum,gpu__time_duration.sum \
  -k regex:"k_dmma|k_reduce" --csv --log-file gpurun_out/mc.csv python tools/model_cases.py > gpurun_out/mc.jsonl 2> gpurun_out/mc.err; echo "model cases rc=$?"
ls -la gpurun_out | tail -20
