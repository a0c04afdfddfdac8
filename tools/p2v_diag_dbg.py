import numpy as np, sys
sys.path.insert(0, '.')
import paper_2404_08371_b200 as tm
for mesh, level in (("cube6", 3), ("cubes2", 2), ("cubes2", 3), ("single-tet", 4)):
    ctx = tm.Context(mesh, device=0)
    k = tm.Function(ctx, tm.SPACE_P2); k.fill_coefficient(level, tm.COEFF_K)
    op = tm.Operator(ctx, tm.FORM_P2V, [k])
    d = tm.Function(ctx, tm.SPACE_P2); op.diagonal(d, level); ctx.synchronize()
    rmap, nref = ctx.ref_map(tm.SPACE_P2, level)
    raw = d.download(level)
    sel = rmap >= 0
    vals = raw[sel]
    print(mesh, level, "diag min/max over stored copies", vals.min(), vals.max(), "n<=0:", int((vals <= 0).sum()), flush=True)
    xs = tm.Function(ctx, tm.SPACE_P2); xs.fill_seeded(level, 5, True)
    b = tm.Function(ctx, tm.SPACE_P2); op.apply(xs, b, level); b.mask_dirichlet(level)
    x = tm.Function(ctx, tm.SPACE_P2)
    try:
        print("  CG", op.cg_solve(b, x, level, rtol=1e-12, max_iter=3000), flush=True)
    except Exception as e:
        print("  CG failed", e)
    x = tm.Function(ctx, tm.SPACE_P2)
    try:
        print("  PCG", op.cg_solve(b, x, level, rtol=1e-12, max_iter=3000, diag=d), flush=True)
    except Exception as e:
        print("  PCG failed", e)
