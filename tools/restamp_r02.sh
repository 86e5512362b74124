#!/bin/bash
# After tools/final_r02.sh + evidence_configs_r02.sh came back in gpurun_out/: regenerate the ncu summaries
# (stamped with the local build's kernel id) and copy the bench lines, GPU test log and launch list into profiles/.
python tools/ncu_summary.py --rep gpurun_out/bench16k_raw.csv --launches gpurun_out/launches_r02_16384.csv --workload "fp64 C+=A*B m=n=k=16384 column-major, family C2A1C0 fused/DMMA" --tag r02_fp64_16384_tma --staging tma --launches-per-step 14 --flops 8796093022208 --model-bytes 53929312256 --blocksizes '{"0:m": 128, "0:n": 128, "1:m": 128, "1:k": 106, "2:m": 1408, "2:n": 1408}' > /dev/null
gen() { [ -f gpurun_out/$1_raw.csv ] && python tools/ncu_summary.py --rep gpurun_out/$1_raw.csv --workload "$2" --tag r02_final_$1 --staging tma --launches-per-step 1 --flops $3 --kernel-regex "$4" > /dev/null; }
gen c1 "fp64 C+=A*B m=n=k=2048 C2A1C0 fused/DMMA (stream-K)" 17179869184 "k_dmma"
gen c3a "fp64 C+=A*B m=n=16384 k=256 (rank-k) C2A1C0 fused/DMMA" 137438953472 "k_dmma"
gen c3b "fp64 C+=A*B m=n=512 k=131072 (inner product) C2A1C0 fused/DMMA (split-k)" 68719476736 "k_dmma"
gen c3c "fp64 C+=A*B m=65536 n=256 k=1024 (panel-panel) B2A1C0 fused/DMMA" 34359738368 "k_dmma"
gen c4bf16 "config4 bf16 C(fp32)+=A*B m=n=k=16384, 256x512 SM-pair tiles, 2048x2048 raster" 8796093022208 "k_tc"
gen c4tf32 "config4 tf32 C(fp32)+=A*B m=n=k=16384, 256x512 SM-pair tiles, 2048x2048 raster" 8796093022208 "k_tc"
for f in bench.log:bench_r02_fp64_16384.json bench_c1.log:bench_c1_r02_final.json bench_c3a.log:bench_c3a_r02_final.json bench_c3b.log:bench_c3b_r02_final.json bench_c3c.log:bench_c3c_r02_final.json bench_c4.log:bench_c4_r02_final.json bench_c4tf32.log:bench_c4tf32_r02_final.json; do
  src=${f%%:*}; dst=${f##*:}; [ -f gpurun_out/$src ] && tail -1 gpurun_out/$src > profiles/$dst; done
cp gpurun_out/gputest.log profiles/gputest_r02.log; cp gpurun_out/launches_r02_16384.csv profiles/launches_r02_fp64_16384.csv
python - <<'PY'
import json, glob
for f in ['profiles/ncu_summary_r02_fp64_16384_tma.json'] + sorted(glob.glob('profiles/ncu_summary_r02_final_c*.json')):
    d = json.load(open(f)); k = d['kernels'][0]
    print(f.split('/')[-1], d['kernel_id'], round(d['tflops_under_ncu'], 2), k.get('dmma_pipe_pct_of_active'), round(d['dram_bytes_per_step'] / 1e9, 3), d.get('measured_over_model'))
PY
