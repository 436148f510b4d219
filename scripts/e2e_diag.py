import os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch, torch.distributed as dist
import bench
import paper_0912_4506_b200 as sp
from paper_0912_4506_b200.dist import SlabRunner
dev = torch.device("cuda", 0); torch.cuda.set_device(0)
os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT="29533")
dist.init_process_group("nccl", rank=0, world_size=1, device_id=dev)
shape = (512, 1024, 1024)
pat = sp.FillPattern.dirichlet_box("random", shape, (1,0,0,0,0,0), seed=0)
for overlap in (True, False):
    rs = [SlabRunner(sp.GridDims(1024, 1024, 512), pat, h=4, depth=4, device=dev, transport="nccl", overlap=overlap) for _ in range(3)]
    for steps in (12, 24):
        e = bench.measure_e2e_dist(torch, dist, rs, [4]*25, dev, 1, 1024*1024*512, steps=steps)
        print("overlap", overlap, "steps", steps, e["value"], e["ms_per_step"], flush=True)
    for r in rs: r.close()
    del rs; torch.cuda.empty_cache()
g = sp.TwoGrid(sp.GridDims(1024, 1024, 512), pat)
e = bench.measure_e2e(sp, torch, np, g, np.float64, [4]*25, dev, torch.cuda.current_stream(), steps=24)
print("single", e["value"], e["ms_per_step"])
dist.destroy_process_group()
