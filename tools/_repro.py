import sys, os
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
import numpy as np, torch
from oracle import oracle as O
from paper_1904_05717_b200 import tilemul as T
import helpers as H
staging = sys.argv[1]; only = int(sys.argv[2]) if len(sys.argv) > 2 else -1
rng = np.random.default_rng(101)
for trial in range(40):
    d = H.random_descriptor(rng)
    shape = T.Shape(*[int(x) for x in rng.integers(1, 97, size=3)])
    bs = H.random_blocksizes(rng, d, shape)
    if only >= 0 and trial != only: continue
    nest = T.build_plan(d, bs, H.roomy(3), shape)
    a, b, c = O.fill_uniform(1000 + trial, [(shape.m, shape.k), (shape.k, shape.n), (shape.m, shape.n)])
    print(trial, T.format_name(d), shape, [(L.dim, L.blocksize) for L in nest.loops], flush=True)
    Cd = torch.from_numpy(c.copy()).cuda()
    T.execute(nest, torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda(), Cd, T.ExecOptions(staging=staging))
    torch.cuda.synchronize()
    print("  ok", nest.last_launch(), flush=True)
