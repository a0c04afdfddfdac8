"""K2 A/B: kernel time of P1 -div(k grad) variants and their agreement with
variant 3 (the round-2 walk) on several meshes / levels.
usage: python tools/k2_ab.py [--c2l-only] [variant ...]   (TETMF_LIB selects a build)"""
import sys

import numpy as np

import paper_2404_08371_b200 as tm

c2l_only = "--c2l-only" in sys.argv
variants = [int(v) for v in sys.argv[1:] if v != "--c2l-only"] or [0, 3]
cases = [] if c2l_only else [("single-tet", L) for L in range(0, 7)] + [("cube6", L) for L in range(1, 6)] + [("cubes2", 4)]
for mesh, L in cases:
    ctx = tm.Context(mesh, device=0)
    x, k = tm.Function(ctx, tm.SPACE_P1), tm.Function(ctx, tm.SPACE_P1)
    x.fill_seeded(L, 7)
    k.fill_coefficient(L, tm.COEFF_K)
    out = {}
    for v in variants:
        y = tm.Function(ctx, tm.SPACE_P1)
        y.fill_seeded(L, 99)  # scribble: every stored value must be overwritten
        op = tm.Operator(ctx, tm.FORM_P1K, [k])
        op.set_variant(v)
        op.apply(x, y, L)
        out[v] = y.download(L)
    ref = out[3] if 3 in out else out[variants[0]]
    scale = float(np.max(np.abs(ref)))
    print(mesh, f"L{L}", " ".join(f"v{v}: {float(np.max(np.abs(out[v] - ref))) / scale:.2e}" for v in variants),
          flush=True)

ctx = tm.Context("cube6", device=0)
L = 8
x, k = tm.Function(ctx, tm.SPACE_P1), tm.Function(ctx, tm.SPACE_P1)
x.fill_seeded(L, 7)
k.fill_coefficient(L, tm.COEFF_K)
for v in variants:
    y = tm.Function(ctx, tm.SPACE_P1)
    op = tm.Operator(ctx, tm.FORM_P1K, [k])
    op.set_variant(v)
    for _ in range(3):
        op.apply(x, y, L)
    ctx.synchronize()
    op.profile(True)
    for _ in range(20):
        op.apply(x, y, L)
    ms, cnt = op.kernel_stats()
    op.profile(False)
    t = ms / cnt
    print(f"c2l cube6 L8 variant {v}: kernel {t * 1e3:8.1f} us  {x.size(L) / (t * 1e-3) / 1e9:7.1f} GDoF/s "
          f"({24 * x.size(L) / (t * 1e-3) / 1e9:.0f} GB/s compulsory)", flush=True)
