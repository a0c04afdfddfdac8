"""P2V apply: kernel time (CUDA events) of the fold walk (variant 0), the
factored cube kernel (variant 2) and the first version (variant 1) at cube6
L7/L8, under the exact rule and quadrature(1..3), and their agreement.
usage: python tools/p2v_time.py [--rules]"""
import sys

import numpy as np

import paper_2404_08371_b200 as tm

rules = (0, 1, 2, 3) if "--rules" in sys.argv else (0,)
for mesh, L in (("cube6", 7), ("cube6", 8)):
    ctx = tm.Context(mesh, device=0)
    k = tm.Function(ctx, tm.SPACE_P2)
    k.fill_coefficient(L, tm.COEFF_K)
    x = tm.Function(ctx, tm.SPACE_P2)
    x.fill_seeded(L, 1)
    dofs = x.num_ref_dofs(L)
    for rule in rules:
        out = {}
        for v in ((0, 2, 1) if rule == 0 else (0, 2)):
            y = tm.Function(ctx, tm.SPACE_P2)
            op = tm.Operator(ctx, tm.FORM_P2V, [k])
            op.set_variant(v)
            op.set_quadrature(rule)
            for _ in range(3):
                op.apply(x, y, L)
            ctx.synchronize()
            op.profile(True)
            for _ in range(10):
                op.apply(x, y, L)
            ms, n = op.kernel_stats()
            op.profile(False)
            t = ms / n
            out[v] = y.download(L)
            print(f"{mesh} L{L} rule {rule} variant {v}: {dofs} DoFs, kernel {t:.3f} ms, "
                  f"{dofs / (t * 1e-3) / 1e9:.2f} GDoF/s", flush=True)
        ref = out[2]
        for v, a in out.items():
            print(f"  variant {v} vs 2: max rel diff {np.abs(a - ref).max() / np.abs(ref).max():.2e}")
