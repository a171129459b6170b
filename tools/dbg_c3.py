"""debug: vector Laplace fused CG vs textbook CG around fem_apply at several sizes"""
import sys, torch
sys.path.insert(0, '.')
from paper_2308_09839_b200 import fem, inputs as I
fem.load(build_if_missing=False)

def textbook(op, b, iters):
    xr = torch.zeros_like(b); r = b.clone(); p = r.clone(); rr = torch.dot(r, r)
    for _ in range(iters):
        q = op.apply(p); alpha = rr / torch.dot(p, q)
        xr += alpha * p; r -= alpha * q; rr_new = torch.dot(r, r)
        p = r + (rr_new / rr) * p; rr = rr_new
    return xr

for kind in sys.argv[1].split(','):
  for n in [int(v) for v in sys.argv[2].split(',')]:
    c = I.ncomp(kind)
    g = I.rng(5)
    op = fem.Operator(fem.Mesh(n, n, n, 1.0 / n), kind, "dirichlet")
    if kind == "elastic":
        lam, mu = I.materials(g, n, n, n)
        op.set_material(torch.from_numpy(lam).cuda(), torch.from_numpy(mu).cuda())
    b = torch.from_numpy(I.interior_rhs(g, n, n, n, c)).cuda()
    xin = torch.from_numpy(I.uniform_vector(g, n, n, n, c)).cuda()
    y1 = op.apply(xin)
    op.set_option("direct_tma", 0)
    y2 = op.apply(xin)
    op.set_option("direct_tma", 1)
    dapply = float((y1 - y2).abs().max() / y2.abs().max())
    res = []
    for opts in [dict(), dict(use_graph=0), dict(dot_mode=1)]:
        for k, v in opts.items(): op.set_option(k, v)
        for iters in (1, 3):
            x = torch.zeros_like(b)
            op.cg_begin(b, x, tol=0.0, maxit=iters); op.cg_iterate(iters); op.cg_end()
            xr = textbook(op, b, iters)
            res.append(float((x - xr).abs().max() / xr.abs().max()))
        for k, v in opts.items(): op.set_option(k, {"use_graph": 1, "dot_mode": 0}[k])
    print(kind, n, "apply pair-vs-bulk %.2e" % dapply, "cg", " ".join("%.1e" % v for v in res), flush=True)
    del op
