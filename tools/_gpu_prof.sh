mkdir -p gpurun_out
for st in tma cpasync; do
python tools/profile_one.py --tile 128 --tile-n 64 --staging $st || exit 1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_dmma --launch-skip 1 -c 1 -f -o gpurun_out/rankk_$st python tools/profile_one.py --tile 128 --tile-n 64 --staging $st > gpurun_out/ncu_rankk_$st.log 2>&1; echo "ncu $st rc=$?"
done
