#!/bin/bash
# One GPU round-trip: smoke, GPU parity tests, bench (ours), in that order.
# Usage: tools/gpu_cycle.sh [bench args...]
mkdir -p gpurun_out
python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke.log
python -m pytest tests -q -m gpu -x > gpurun_out/gputest.log 2>&1; echo "gpu tests rc=$?"; tail -15 gpurun_out/gputest.log
python bench.py "$@" > gpurun_out/bench.log 2>&1; echo "bench rc=$?"; tail -c 2500 gpurun_out/bench.log
