"""Stress: many repeated launches of the 128x128 TMA kernel, each compared bitwise with the cp.async result."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np, torch
from oracle import oracle as O
from paper_1904_05717_b200 import tilemul as T
from test_gpu_tma import fused_nest

REPS = int(os.environ.get("REPS", "200"))
SLEEP = float(os.environ.get("SLEEP", "0"))
for (m, n, k) in ((336, 608, 1118), (1200, 1100, 700), (2048, 2048, 2048), (4096, 4096, 512)):
    nest = fused_nest(m, n, k)
    a, b, c = O.fill_uniform(77, [(m, k), (k, n), (m, n)])
    A, B, C0 = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda(), torch.from_numpy(c).cuda()
    for split in (1, 0, -1, 3):
        kw = dict(split_k=split, tile=128, tile_n=128)
        ref = C0.clone()
        T.execute(nest, A, B, ref, T.ExecOptions(staging="cpasync", **kw))
        torch.cuda.synchronize()
        bad = 0
        for rep in range(REPS):
            Cd = C0.clone()
            if SLEEP: time.sleep(SLEEP)
            T.execute(nest, A, B, Cd, T.ExecOptions(staging="tma", **kw))
            torch.cuda.synchronize()
            d = torch.nonzero(Cd != ref).flatten()
            if d.numel():
                bad += 1
                if bad <= 3:
                    ii, jj = (d % m).cpu().numpy(), (d // m).cpu().numpy()
                    err = (Cd[d] - ref[d]).abs()
                    print(f"  {m}x{n}x{k} split {split} rep {rep}: {d.numel()} differ, abs max {err.max().item():.3e} min {err.min().item():.3e}; "
                          f"tiles {sorted(set(zip((ii//128).tolist(), (jj//128).tolist())))[:6]} warp tiles {sorted(set(zip((ii//32%4).tolist(), (jj//32%4).tolist())))[:16]} "
                          f"rows%32 {sorted(set((ii%32).tolist()))[:16]} n={len(set((ii%32).tolist()))} cols%32 n={len(set((jj%32).tolist()))}", flush=True)
        print(f"{m}x{n}x{k} split {split}: {bad}/{REPS} bad ({nest.last_launch()})", flush=True)
