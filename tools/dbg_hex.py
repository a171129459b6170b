import sys, time, numpy as np, torch
sys.path.insert(0, '.')
from paper_2308_09839_b200 import inputs as I, fem
fem.load()
print("loaded", flush=True)
for n in [(1,1,1), (3,2,2), (40,3,2)]:
    c, e, b = I.hex_box_mesh(*n, jitter=0.1)
    m = fem.HexMesh(torch.from_numpy(c).cuda(), torch.from_numpy(e).cuda(), torch.from_numpy(b).cuda())
    print("mesh ok", n, flush=True)
    op = fem.Operator(m, "scalar", 1)
    x = torch.rand(c.shape[0], dtype=torch.float64, device="cuda")
    t=time.time(); y = op.apply(x); torch.cuda.synchronize(); print("apply ok", n, time.time()-t, float(y.abs().sum()), flush=True)
