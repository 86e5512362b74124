#!/usr/bin/env python
"""Pinned PCIe bandwidth one way and both ways at once (two streams): the bound of the C-dominated
host-buffer shapes (rank-k: 2.1 GB of C up and down).   python tools/duplex_probe.py"""
import json
import time

import torch

n = (1 << 30) // 8
hu, hd = torch.empty(n, dtype=torch.float64).pin_memory(), torch.empty(n, dtype=torch.float64).pin_memory()
du, dd = torch.empty(n, dtype=torch.float64, device="cuda"), torch.empty(n, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def t(f, reps=3):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        f()
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    return best


def up():
    with torch.cuda.stream(s1):
        du.copy_(hu, non_blocking=True)


def down():
    with torch.cuda.stream(s2):
        hd.copy_(dd, non_blocking=True)


def both():
    up()
    down()


g = (1 << 30) / 1e9
print(json.dumps({"h2d_GBps": g / t(up), "d2h_GBps": g / t(down), "both_GBps_each": g / t(both)}))
