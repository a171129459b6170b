import sys, torch
sys.path.insert(0, '.')
from paper_2308_09839_b200 import fem, inputs as I
fem.load(build_if_missing=False)
kind = sys.argv[1]; n = int(sys.argv[2])
c = I.ncomp(kind); g = I.rng(5)
op = fem.Operator(fem.Mesh(n, n, n, 1.0 / n), kind, "dirichlet")
op.set_option("use_graph", 0)
b = torch.from_numpy(I.interior_rhs(g, n, n, n, c)).cuda()
for rep in range(3):
    x = torch.zeros_like(b)
    op.cg_begin(b, x, tol=0.0, maxit=1); op.cg_iterate(1); info = op.cg_end()
    m = b != 0
    ratio = torch.zeros_like(b); ratio[m] = x[m] / b[m]
    med = ratio[m].median()
    good = m & ((ratio - med).abs() <= 1e-9 * med.abs())
    bad = m & ~good
    print("rep", rep, "alpha_gpu(median ratio) %.12e" % float(med), "good", int(good.sum()), "bad", int(bad.sum()), flush=True)
    if bad.sum() == 0: continue
    bn = (bad.nonzero().flatten() // c)
    i = bn % (n + 1); j = (bn // (n + 1)) % (n + 1); k = bn // ((n + 1) ** 2)
    for name, v in (("i", i), ("j", j), ("k", k)):
        h = torch.bincount(v, minlength=n + 1).cpu().tolist()
        print(" ", name, "bad per index:", h[:12], "...", h[120:136], "...", h[-12:])
    gn = (good.nonzero().flatten() // c)
    gi = gn % (n + 1); gj = (gn // (n + 1)) % (n + 1); gk = gn // ((n + 1) ** 2)
    print("  good i", torch.bincount(gi, minlength=n+1).cpu().tolist()[:40])
    print("  good j", torch.bincount(gj, minlength=n+1).cpu().tolist()[:40])
    print("  good k", torch.bincount(gk, minlength=n+1).cpu().tolist()[:40])
