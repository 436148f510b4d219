import sys, os
sys.path.insert(0, '/root/repo' if os.path.exists('/root/repo/bench.py') else '.')
import torch, numpy as np, paper_0912_4506_b200 as sp
lib = sp._native.lib()
for dt, nz in ((np.float64, 1024), (np.float32, 2048)):
    n = 1024
    g = sp.TwoGrid(sp.GridDims(n, n, nz), sp.FillPattern.dirichlet_box("random", (nz, n, n), (1, 0, .5, 0, .25, 0)), dtype=dt)
    for k1 in (1, 0):
        lib.sp_set_tuning(-1 if k1 else 0, 0)
        sp.sweeps(g, 2, depth=1); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); sp.sweeps(g, 20, depth=1); e1.record(); torch.cuda.synchronize()
        t = e0.elapsed_time(e1) / 1e3
        print(np.dtype(dt).name, "K1" if k1 else "K2(T=1)", round(n * n * nz * 20 / t / 1e9, 1), "GLUP/s")
    lib.sp_set_tuning(0, 0)
