import sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_1904_05717_b200 import tilemul as T
import bench
size = int(sys.argv[1]); mode = sys.argv[2]
nest, bs, hier = bench.make_plan(T, size, size, size)
A = torch.empty(size*size, dtype=torch.float64, device='cuda'); T.fill_uniform_device(A, 1)
B = torch.empty(size*size, dtype=torch.float64, device='cuda'); T.fill_uniform_device(B, 2)
C = torch.empty(size*size, dtype=torch.float64, device='cuda'); T.fill_uniform_device(C, 3)
if 'dev' in mode:
    n2 = nest
    if 'other' in mode:
        n2, _, _ = bench.make_plan(T, size, size, size)
    T.execute(n2, A, B, C); torch.cuda.synchronize(); print("device ok", flush=True)
if 'free' in mode:
    del A, B, C; torch.cuda.empty_cache()
    A = torch.zeros(10, dtype=torch.float64, device='cuda')
    Ah = np.zeros(size*size); Bh = np.zeros(size*size); Ch = np.zeros(size*size)
elif 'pin' in mode:
    Ah = A.cpu().pin_memory().numpy(); Bh = B.cpu().pin_memory().numpy(); Ch = C.cpu().pin_memory().numpy()
else:
    Ah = A.cpu().numpy(); Bh = B.cpu().numpy(); Ch = C.cpu().numpy()
try:
    T.execute(nest, Ah, Bh, Ch); print(mode, "host ok", nest.last_launch(), flush=True)
except Exception as e:
    print(mode, "host FAIL", e, flush=True)
