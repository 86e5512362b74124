#!/usr/bin/env python
"""One config through T.execute for an ncu capture: a warm-up launch, then
`--reps` profiled launches (capture with --launch-skip 1 -k regex:k_dmma).

  python tools/profile_one.py --shape 16384,16384,256 --tile 128 --tile-n 64 --staging tma
"""
from __future__ import annotations

import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shape", default="16384,16384,256")
    ap.add_argument("--family", default="C2A1C0")
    ap.add_argument("--tile", type=int, default=0)
    ap.add_argument("--tile-n", type=int, default=0)
    ap.add_argument("--split", type=int, default=0)
    ap.add_argument("--staging", default="auto")
    ap.add_argument("--reps", type=int, default=1)
    ap.add_argument("--ld-pad", type=int, default=0, help="leading-dimension padding (elements) of A, B and C")
    a = ap.parse_args()
    import torch
    from paper_1904_05717_b200 import planner, tilemul as T

    m, n, k = (int(x) for x in a.shape.split(","))
    _, bs, hier = planner.plan_for_gpu(a.family, (m, n, k))
    nest = T.build_plan(T.parse_name(a.family), bs, hier, T.Shape(m, n, k))
    P = a.ld_pad
    Ab = torch.empty(k * (m + P), dtype=torch.float64, device="cuda")
    Bb = torch.empty(n * (k + P), dtype=torch.float64, device="cuda")
    Cb = torch.empty(n * (m + P), dtype=torch.float64, device="cuda")
    for x, s in ((Ab, 1), (Bb, 2), (Cb, 3)):
        T.fill_uniform_device(x, s)
    A = Ab.view(k, m + P).t()[:m, :]
    B = Bb.view(n, k + P).t()[:k, :]
    C = Cb.view(n, m + P).t()[:m, :]
    opts = T.ExecOptions(numerics="dmma", split_k=a.split, tile=a.tile, tile_n=a.tile_n, staging=a.staging)
    for _ in range(1 + a.reps):
        T.execute(nest, A, B, C, opts)
    torch.cuda.synchronize()
    print(nest.last_launch())


if __name__ == "__main__":
    main()
