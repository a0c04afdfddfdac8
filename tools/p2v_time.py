"""Timing of the P2V apply (kernel events) at cube6 L7/L8: python tools/p2v_time.py"""
import paper_2404_08371_b200 as tm

for mesh, L in (("cube6", 7), ("cube6", 8)):
    ctx = tm.Context(mesh, device=0)
    k = tm.Function(ctx, tm.SPACE_P2)
    k.fill_coefficient(L, tm.COEFF_K)
    x, y = tm.Function(ctx, tm.SPACE_P2), tm.Function(ctx, tm.SPACE_P2)
    x.fill_seeded(L, 1)
    op = tm.Operator(ctx, tm.FORM_P2V, [k])
    for _ in range(3):
        op.apply(x, y, L)
    ctx.synchronize()
    op.profile(True)
    for _ in range(10):
        op.apply(x, y, L)
    ms, n = op.kernel_stats()
    dofs = x.num_ref_dofs(L)
    elems = 6 * 8 ** L
    t = ms / n
    print(f"{mesh} L{L}: {dofs} DoFs, kernel {t:.3f} ms, {dofs / (t * 1e-3) / 1e9:.2f} GDoF/s, "
          f"{1300.0 * elems / (t * 1e-3) / 1e12:.2f} TFLOP/s (1300 flop/element)", flush=True)
