#!/bin/bash
# A/B of cluster-launch-control tile scheduling (TILEMUL_TC_CLC) on the tcgen05 pair kernels (config 4):
# parity tests with CLC on, then CUDA-event TF/s (tools/bench_tc.py) and one ncu launch per variant.
mkdir -p gpurun_out
TILEMUL_TC_CLC=1 timeout 300 python -m pytest tests/test_gpu_tc.py tests/test_gpu_baseline_shapes.py -q -m gpu -x -k "tc or config4" > gpurun_out/clc_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/clc_tests.log
for rep in 1 2; do for v in 0 1; do
  TILEMUL_TC_CLC=$v TC_CASES=${TC_CASES:-bf16:256:512,tf32:256:512,bf16:256:256} TC_CUBLAS=0 timeout 240 python tools/bench_tc.py \
    | python -c "import json,sys
for l in sys.stdin:
    d=json.loads(l); print('clc=$v', d['dtype'], d['cta_tile'], round(d['tflops'],1), d['clocks'].get('sm_mhz'), d['clocks'].get('power_w_median'))"
done; done
for v in 0 1; do
  TILEMUL_TC_CLC=$v TC_CASES=${NCU_CASE:-bf16:256:512} TC_CUBLAS=0 timeout 400 ncu --clock-control none \
    --metrics dram__bytes_read.sum,gpu__time_duration.sum,sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_active,lts__t_sectors_srcunit_tex_op_read.sum,lts__throughput.avg.pct_of_peak_sustained_elapsed \
    -k regex:k_tc2 -s 3 -c 1 --csv timeout 300 python tools/bench_tc.py 2>/dev/null | grep -E '"(dram|gpu__time|sm__pipe|lts)' | awk -F'","' '{print "clc='$v' "$(NF-2)" "$NF}'
done
