#!/bin/bash
# Generic config-4 A/B over one environment knob: tools/ab_env.sh VAR "v1 v2 ..." [reps]
#   parity tests with each non-default value, then tools/bench_tc.py per value (alternating, reps rounds),
#   then one ncu launch per value (DRAM, time, tensor-pipe activity).
VAR=$1; VALS=$2; REPS=${3:-2}
mkdir -p gpurun_out
for v in $VALS; do
  env $VAR=$v timeout 300 python -m pytest tests/test_gpu_tc.py tests/test_gpu_baseline_shapes.py -q -m gpu -x -k "tc or config4" > gpurun_out/ab_env_tests_$v.log 2>&1
  echo "tests $VAR=$v rc=$?"; tail -1 gpurun_out/ab_env_tests_$v.log
done
for rep in $(seq $REPS); do for v in $VALS; do
  env $VAR=$v TC_CASES=${TC_CASES:-bf16:256:512,tf32:256:512} TC_CUBLAS=0 timeout 240 python tools/bench_tc.py \
    | python -c "import json,sys
for l in sys.stdin:
    d=json.loads(l); print('$VAR=$v', d['dtype'], d['cta_tile'][:7], round(d['tflops'],1))"
done; done
if [ -n "$CUBLAS" ]; then TC_CASES=bf16:256:512 TC_CUBLAS=1 timeout 300 python tools/bench_tc.py | python -c "import json,sys
for l in sys.stdin:
    d=json.loads(l); print(d.get('impl','ours'), d['dtype'], round(d['tflops'],1))"; fi
for v in $VALS; do
  env $VAR=$v TC_CASES=${NCU_CASE:-bf16:256:512} TC_CUBLAS=0 timeout 400 ncu --clock-control none \
    --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_active,sm__cycles_elapsed.avg.per_second,lts__t_sectors_srcunit_tex_op_read.sum,l1tex__m_xbar2l1tex_read_bytes.sum \
    -k regex:k_tc2 -s 3 -c 1 --csv timeout 300 python tools/bench_tc.py 2>/dev/null | grep -E "\"(dram|gpu__time|sm__|lts__|l1tex__)" | awk -F'","' '{print "'$VAR'='$v' ncu "$(NF-2)" "$NF}'
done
