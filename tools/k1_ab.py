"""K1 A/B: kernel time of P1 -Laplace variants on one mesh/level and bitwise
agreement with the default kernel (variant 0).
usage: python tools/k1_ab.py [mesh] [level] [variant ...]   (TETMF_LIB selects a build)"""
import sys

import numpy as np

import paper_2404_08371_b200 as tm

mesh = sys.argv[1] if len(sys.argv) > 1 else "cube6"
L = int(sys.argv[2]) if len(sys.argv) > 2 else 8
variants = [int(v) for v in sys.argv[3:]] or [0, 3]
ctx = tm.Context(mesh, device=0)
x = tm.Function(ctx, tm.SPACE_P1)
x.fill_seeded(L, 7)
ref = None
for v in variants:
    y = tm.Function(ctx, tm.SPACE_P1)
    op = tm.Operator(ctx, tm.FORM_P1)
    op.set_variant(v)
    for _ in range(3):
        op.apply(x, y, L)
    ctx.synchronize()
    op.profile(True)
    for _ in range(20):
        op.apply(x, y, L)
    ms, k = op.kernel_stats()
    op.profile(False)
    vals = y.download(L)
    if ref is None:
        ref = vals
    diff = float(np.max(np.abs(vals - ref)))
    print(f"{mesh} L{L} variant {v}: kernel {ms / k * 1e3:8.1f} us  {x.size(L) / (ms / k * 1e-3) / 1e9:7.1f} "
          f"GDoF/s  max|y - y_v{variants[0]}| = {diff:.3e}", flush=True)
