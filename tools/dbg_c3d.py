import sys, torch
sys.path.insert(0, '.')
from paper_2308_09839_b200 import fem, inputs as I
fem.load(build_if_missing=False)
kind = sys.argv[1]; n = int(sys.argv[2]); ug = int(sys.argv[3])
c = I.ncomp(kind); g = I.rng(5)
op = fem.Operator(fem.Mesh(n, n, n, 1.0 / n), kind, "dirichlet")
op.set_option("use_graph", ug)
b = torch.from_numpy(I.interior_rhs(g, n, n, n, c)).cuda()
q = op.apply(b); alpha = torch.dot(b, b) / torch.dot(b, q); xr = alpha * b
for rep in range(5):
    x = torch.zeros_like(b)
    op.cg_begin(b, x, tol=0.0, maxit=1); op.cg_iterate(1); info = op.cg_end()
    m = b != 0
    ratio = torch.ones_like(b); ratio[m] = x[m] / xr[m]
    bad = m & ((ratio - 1).abs() > 1e-6)
    print("rep", rep, "bad", int(bad.sum()), flush=True)
    if bad.sum() == 0: continue
    bn = (bad.nonzero().flatten() // c).unique()
    i = bn % (n + 1); j = (bn // (n + 1)) % (n + 1); k = bn // ((n + 1) ** 2)
    print("  i tiles(29):", torch.bincount(i // 29).cpu().tolist())
    print("  j tiles(7):", torch.bincount(j // 7).cpu().tolist())
    print("  k:", torch.bincount(k, minlength=n+1).cpu().tolist())
    print("  ratios sample", ratio[bad][:10].cpu().tolist())
