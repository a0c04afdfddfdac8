"""K3 fold-walk task length sweep: kernel time of N1 per (mesh, level) with the
steps per task forced (TETMF_N1F2_CHUNK_STEPS, read when a level is first
used) and with the default choice (n1_fold2_chunk); all bitwise equal.
The same for the P2V fold walk with --p2v (TETMF_P2VF_CHUNK_STEPS).
usage: python tools/k3_chunk.py [--p2v]"""
import os
import sys

import numpy as np

import paper_2404_08371_b200 as tm

p2v = "--p2v" in sys.argv
env = "TETMF_P2VF_CHUNK_STEPS" if p2v else "TETMF_N1F2_CHUNK_STEPS"
cases = [("single-tet", 4), ("single-tet", 5), ("single-tet", 6), ("single-tet", 7), ("cube6", 4), ("cube6", 5),
         ("cube6", 6), ("cubes2x2x2", 4), ("cubes2x2x2", 5)]
for mesh, L in cases:
    res, ref = [], None
    for chunk in ("32", "16", "8", "4", "2", ""):
        if chunk:
            os.environ[env] = chunk
        else:
            os.environ.pop(env, None)
        ctx = tm.Context(mesh, device=0)
        if p2v:
            x, y, k = (tm.Function(ctx, tm.SPACE_P2) for _ in range(3))
            k.fill_coefficient(L, tm.COEFF_K)
            op = tm.Operator(ctx, tm.FORM_P2V, [k])
        else:
            x, y = tm.Function(ctx, tm.SPACE_ND1), tm.Function(ctx, tm.SPACE_ND1)
            a, b = tm.Function(ctx, tm.SPACE_P1), tm.Function(ctx, tm.SPACE_P1)
            a.fill_coefficient(L, tm.COEFF_ALPHA)
            b.fill_coefficient(L, tm.COEFF_BETA)
            op = tm.Operator(ctx, tm.FORM_N1, [a, b])
        x.fill_seeded(L, 7)
        y.fill_seeded(L, 99)
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
    print(f"{mesh} L{L} ({x.size(L)} dofs)  " + "  ".join(res), flush=True)
