"""timing experiment: event-graph (time_apply) vs plain-graph passes, alternated"""
import sys, torch
sys.path.insert(0, '.')
from paper_2308_09839_b200 import fem, inputs as I
fem.load(build_if_missing=False)
cfg = I.CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 3]
nx, ny, nz = I.config_cells(cfg); kind = cfg["kind"]; c = I.ncomp(kind)
op = fem.Operator(fem.Mesh(nx, ny, nz, 1.0 / nx), kind, "dirichlet")
g = I.rng(I.SEED_BASE + 3)
if kind == "elastic":
    lam, mu = I.materials(g, nx, ny, nz); op.set_material(torch.from_numpy(lam).cuda(), torch.from_numpy(mu).cuda())
b = torch.from_numpy(I.interior_rhs(g, nx, ny, nz, c)).cuda(); x = torch.zeros_like(b)
K = 20
op.cg_begin(b, x, tol=0.0, maxit=1 << 30)
def run(timed):
    op.set_option("time_apply", 1 if timed else 0)
    op.cg_iterate(K); torch.cuda.synchronize(); op.apply_time()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(); op.cg_iterate(K); e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / K
    a, n = op.apply_time()
    return ms, (a / n if n else None)
for i in range(3):
    for timed in (1, 0):
        ms, a = run(timed)
        print("event-graph" if timed else "plain-graph", "step %.4f ms" % ms, "apply %s" % (("%.4f" % a) if a else "-"), flush=True)
