import sys, torch
sys.path.insert(0, '.')
from paper_2308_09839_b200 import fem, inputs as I
fem.load(build_if_missing=False)
kind = sys.argv[1]; n = int(sys.argv[2])
c = I.ncomp(kind); g = I.rng(5)
op = fem.Operator(fem.Mesh(n, n, n, 1.0 / n), kind, "dirichlet")
b = torch.from_numpy(I.interior_rhs(g, n, n, n, c)).cuda()
ys = [op.apply(b) for _ in range(4)]
print("apply mode 0 deterministic", [bool(torch.equal(ys[0], v)) for v in ys[1:]])
q = op.apply(b); alpha = torch.dot(b, b) / torch.dot(b, q); xr = alpha * b
for rep in range(6):
    x = torch.zeros_like(b)
    op.cg_begin(b, x, tol=0.0, maxit=1); op.cg_iterate(1); info = op.cg_end()
    d = float((x - xr).abs().max() / xr.abs().max())
    # x = alpha_gpu * p_gpu: compare direction (x / xr ratio) to separate alpha errors from p errors
    ratio = x[b != 0] / xr[b != 0]
    print("rep", rep, "d %.2e" % d, "nan", int(torch.isnan(x).sum()), "ratio min/max %.6f %.6f" % (float(ratio.min()), float(ratio.max())), flush=True)
    if d > 1e-9:
        bad = ((x - xr).abs() > 1e-9 * xr.abs().max()).nonzero().flatten()
        nodes = (bad // c).unique()
        i = nodes % (n + 1); j = (nodes // (n + 1)) % (n + 1); k = nodes // ((n + 1) ** 2)
        print("  bad dofs", bad.numel(), "i", int(i.min()), int(i.max()), "j", int(j.min()), int(j.max()),
              "k", int(k.min()), int(k.max()), [(int(a), int(bb), int(cc)) for a, bb, cc in zip(i[:6], j[:6], k[:6])])
