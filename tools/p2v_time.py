"""P2V apply: kernel time (CUDA events) of the factored kernel (variant 0)
and the first version (variant 1) at cube6 L7/L8, and their agreement.
usage: python tools/p2v_time.py"""
import numpy as np

import paper_2404_08371_b200 as tm

for mesh, L in (("cube6", 7), ("cube6", 8)):
    ctx = tm.Context(mesh, device=0)
    k = tm.Function(ctx, tm.SPACE_P2)
    k.fill_coefficient(L, tm.COEFF_K)
    x = tm.Function(ctx, tm.SPACE_P2)
    x.fill_seeded(L, 1)
    dofs = x.num_ref_dofs(L)
    out = {}
    for v in (0, 1):
        y = tm.Function(ctx, tm.SPACE_P2)
        op = tm.Operator(ctx, tm.FORM_P2V, [k])
        op.set_variant(v)
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
        print(f"{mesh} L{L} variant {v}: {dofs} DoFs, kernel {t:.3f} ms, {dofs / (t * 1e-3) / 1e9:.2f} GDoF/s",
              flush=True)
    d = np.abs(out[0] - out[1]).max() / np.abs(out[1]).max()
    print(f"{mesh} L{L}: max |y_v0 - y_v1| / max |y_v1| = {d:.3e}", flush=True)
