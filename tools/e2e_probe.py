import os, sys, time, json, itertools, subprocess
sys.path.insert(0, os.getcwd())
import torch
n = 2 * 1024**3 // 8
h = torch.empty(n, dtype=torch.float64).pin_memory()
h2 = torch.empty(n, dtype=torch.float64).pin_memory()
d = torch.empty(n, dtype=torch.float64, device="cuda")
d2 = torch.empty(n, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for _ in range(2):
    d.copy_(h, non_blocking=True); torch.cuda.synchronize()
def t(f):
    torch.cuda.synchronize(); t0 = time.perf_counter(); f(); torch.cuda.synchronize(); return time.perf_counter() - t0
bw_h2d = 2 * 1024**3 / t(lambda: d.copy_(h, non_blocking=True)) / 1e9
bw_d2h = 2 * 1024**3 / t(lambda: h.copy_(d, non_blocking=True)) / 1e9
def both():
    with torch.cuda.stream(s1): d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
bw_both = 2 * 2 * 1024**3 / t(both) / 1e9
print(json.dumps({"h2d_GBps": bw_h2d, "d2h_GBps": bw_d2h, "bidir_total_GBps": bw_both}), flush=True)

# host-buffer pipeline configurations at the bench workload (16384^3, pinned)
from paper_1904_05717_b200 import tilemul as T
import bench
m = n = k = int(os.environ.get("SIZE", "16384"))
nest, bs, hier = bench.make_plan(T, m, n, k)
opts = T.ExecOptions(numerics="dmma", schedule="fused", split_k=0)
A = torch.empty(m * k, dtype=torch.float64).pin_memory().numpy(); A[:] = 0.5
B = torch.empty(k * n, dtype=torch.float64).pin_memory().numpy(); B[:] = 0.25
C = torch.empty(m * n, dtype=torch.float64).pin_memory().numpy(); C[:] = 0.0
Ad = torch.full((m * k,), 0.5, dtype=torch.float64, device="cuda")
Bd = torch.full((k * n,), 0.25, dtype=torch.float64, device="cuda")
Cd = torch.zeros(m * n, dtype=torch.float64, device="cuda")
T.execute(nest, Ad, Bd, Cd, opts); torch.cuda.synchronize()
dev = min(t(lambda: T.execute(nest, Ad, Bd, Cd, opts)) for _ in range(3))
print(json.dumps({"device_ms": dev * 1e3}), flush=True)
for wave, taper, nq, nb in itertools.product([1, 0], [0, 1], [4, 8, 16], [4, 8, 16]):
    os.environ.update(TM_PIPE_WAVE=str(wave), TM_PIPE_TAPER=str(taper), TM_PIPE_NQ=str(nq), TM_PIPE_NB=str(nb))
    T.execute(nest, A, B, C, opts)
    ts = []
    for _ in range(3):
        t0 = time.perf_counter(); T.execute(nest, A, B, C, opts); ts.append(time.perf_counter() - t0)
    print(json.dumps({"wave": wave, "taper": taper, "nq": nq, "nb": nb, "ms": min(ts) * 1e3,
                      "launches": nest.last_launch()["launches"]}), flush=True)
