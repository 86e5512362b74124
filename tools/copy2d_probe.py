#!/usr/bin/env python
"""Pinned-host -> device bandwidth of strided (2-D) copies against contiguous ones: a column-major operand's
row block is `cols` runs of `rows * 8` bytes, one per column (pitch = the operand's leading dimension). The
host-buffer pipeline's upload order (csrc/host_pipe.cpp) cuts A into row blocks; this probe says what a run
length costs.   python tools/copy2d_probe.py"""
import ctypes
import json
import time

import torch

rt = ctypes.CDLL("libcudart.so.12")
rt.cudaMemcpy2DAsync.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_size_t,
                                 ctypes.c_size_t, ctypes.c_int, ctypes.c_void_p]
H2D = 1
ld = 16384  # elements: the 16384^3 operands' leading dimension
total = 1 << 30  # bytes per measurement
h = torch.empty(ld * 16384, dtype=torch.float64).pin_memory()
d = torch.empty(ld * 16384, dtype=torch.float64, device="cuda")
st = torch.cuda.current_stream().cuda_stream


def t(f, reps=3):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        f()
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    return best


def ncols(rows):
    return min(16384, total // (rows * 8))


def copy2d(rows, pieces=1):
    cols = ncols(rows)
    per = max(1, cols // pieces)
    def go():
        for p in range(0, cols, per):
            c = min(per, cols - p)
            rc = rt.cudaMemcpy2DAsync(d.data_ptr() + p * ld * 8, ld * 8, h.data_ptr() + p * ld * 8, ld * 8, rows * 8, c, H2D, st)
            assert rc == 0, rc
    return go


print(json.dumps({"contiguous_GBps": total / t(lambda: d[: total // 8].copy_(h[: total // 8], non_blocking=True)) / 1e9}), flush=True)
for rows in (16384, 8192, 4096, 2048, 1024, 512, 256):
    nb = ncols(rows) * rows * 8
    print(json.dumps({"rows": rows, "run_bytes": rows * 8, "bytes": nb, "one_call_GBps": nb / t(copy2d(rows)) / 1e9,
                      "calls_of_4096_cols_GBps": nb / t(copy2d(rows, pieces=max(1, ncols(rows) // 4096))) / 1e9}), flush=True)
