"""Repeat-apply stress test of the default K1 kernel: N applies of the same
input must be bitwise identical (the box kernel's TMA copy / mbarrier
pipeline must not race). usage: python tools/stress_k1.py [mesh] [level] [N]"""
import sys

import numpy as np

import paper_2404_08371_b200 as tm

mesh = sys.argv[1] if len(sys.argv) > 1 else "cube6"
L = int(sys.argv[2]) if len(sys.argv) > 2 else 8
N = int(sys.argv[3]) if len(sys.argv) > 3 else 200
ctx = tm.Context(mesh, device=0)
x, y = tm.Function(ctx, tm.SPACE_P1), tm.Function(ctx, tm.SPACE_P1)
op = tm.Operator(ctx, tm.FORM_P1)
x.fill_seeded(L, 17)
op.apply(x, y, L)
ref = y.download(L)
bad = 0
for i in range(N):
    y.fill_seeded(L, 1000 + i)  # scribble over the output first
    op.apply(x, y, L)
    if not np.array_equal(y.download(L), ref):
        bad += 1
print(f"{mesh} L{L}: {N} repeated applies, {bad} differ from the first")
sys.exit(1 if bad else 0)
