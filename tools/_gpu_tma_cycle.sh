mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/gputest.log 2>&1; echo "tests rc=$?"; tail -5 gpurun_out/gputest.log
for st in tma cpasync; do
timeout 900 python tools/sweep.py --tiles auto,128x64,64x64 --staging $st > gpurun_out/sweep_$st.jsonl 2> gpurun_out/sweep_$st.err; echo "sweep $st rc=$?"
done
python - <<'PY'
import json
rows={}
for st in ("tma","cpasync"):
    for l in open(f"gpurun_out/sweep_{st}.jsonl"):
        r=json.loads(l)
        if "tflops" in r: rows.setdefault((r["config"],tuple(r["shape"]),r["family"],r["cta_tile"]),{})[st]=r["pct_fp64_peak"]
for k,v in rows.items():
    if k[2]=="C2A1C0": print(k, {s: round(x,2) for s,x in v.items()})
PY
for st in tma cpasync; do
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_dmma --launch-skip 1 -c 1 -f -o gpurun_out/rankk_$st python tools/profile_one.py --tile 128 --tile-n 64 --staging $st > gpurun_out/ncu_rankk_$st.log 2>&1; echo "ncu $st rc=$?"
done
