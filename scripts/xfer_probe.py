"""Dev tool: TwoGrid.upload / download bandwidth at 1024^3 fp64 (alone and concurrently)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_0912_4506_b200 as sp  # noqa: E402

n = int(os.environ.get("N", "1024"))
d = sp.GridDims(n, n, n)
g1 = sp.TwoGrid(d, sp.FillPattern.constant(1.0))
g2 = sp.TwoGrid(d, sp.FillPattern.constant(2.0))
h_in = torch.empty(g1.host_shape(), dtype=torch.float64, pin_memory=True)
h_out = torch.empty(d.shape, dtype=torch.float64, pin_memory=True)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps


bi, bo = h_in.numel() * 8, h_out.numel() * 8
tu = timed(lambda: g1.upload(h_in, stream=s1.cuda_stream))
td = timed(lambda: g2.download(h_out, stream=s2.cuda_stream))
tb = timed(lambda: (g1.upload(h_in, stream=s1.cuda_stream), g2.download(h_out, stream=s2.cuda_stream)))
print(f"upload {bi / tu / 1e9:.1f} GB/s ({tu * 1e3:.0f} ms)  download {bo / td / 1e9:.1f} GB/s "
      f"({td * 1e3:.0f} ms)  both {tb * 1e3:.0f} ms")
tc = timed(lambda: sp.sweeps(g2, 100, depth=2), reps=2)
print(f"100 sweeps {tc * 1e3:.0f} ms")
