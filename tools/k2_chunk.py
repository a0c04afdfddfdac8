"""K2 cube-walk task size sweep: kernel time of P1 -div(k grad) per (mesh, level)
with rows = layers per task forced to 16 / 8 / 4 (TETMF_P1KC_CHUNK, read when a
level is first used) and with the default choice (p1k_cube_chunk); all bitwise
equal. usage: python tools/k2_chunk.py"""
import os
import sys

import numpy as np

import paper_2404_08371_b200 as tm

cases = [("single-tet", 5), ("single-tet", 6), ("single-tet", 7), ("single-tet", 8), ("cube6", 5), ("cube6", 6),
         ("cube6", 7), ("cube6", 8), ("cubes2", 5), ("cubes2", 6)]
for mesh, L in cases:
    res, ref = [], None
    for chunk in ("16", "8", "4", ""):
        if chunk:
            os.environ["TETMF_P1KC_CHUNK"] = chunk
        else:
            os.environ.pop("TETMF_P1KC_CHUNK", None)
        ctx = tm.Context(mesh if mesh != "cubes2" else "cubes2x2x2", device=0)
        x, k, y = (tm.Function(ctx, tm.SPACE_P1) for _ in range(3))
        x.fill_seeded(L, 7)
        k.fill_coefficient(L, tm.COEFF_K)
        y.fill_seeded(L, 99)
        op = tm.Operator(ctx, tm.FORM_P1K, [k])
        for _ in range(3):
            op.apply(x, y, L)
        ctx.synchronize()
        op.profile(True)
        for _ in range(20):
            op.apply(x, y, L)
        ms, cnt = op.kernel_stats()
        op.profile(False)
        out = y.download(L)
        if ref is None:
            ref = out
        same = bool(np.array_equal(out, ref))
        res.append(f"{chunk or 'auto'}: {ms / cnt * 1e3:7.1f} us{'' if same else ' DIFF'}")
    print(f"{mesh} L{L} ({x.size(L)} points)  " + "  ".join(res), flush=True)
