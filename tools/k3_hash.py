"""Prints a hash of N1 applies (pass 0 + pass 1 + interface sum) on small
meshes, for bitwise A/B of K3 builds: TETMF_LIB=... python tools/k3_hash.py"""
import hashlib
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2404_08371_b200 as tm  # noqa: E402

h = hashlib.sha256()
worst = 0.0
for mesh, L in [("cubes2", 5), ("cube6", 6), ("single-tet", 7), ("cubes1x1x2", 4)]:
    ctx = tm.Context(mesh, device=0)
    x, y = tm.Function(ctx, tm.SPACE_ND1), tm.Function(ctx, tm.SPACE_ND1)
    a, b = tm.Function(ctx, tm.SPACE_P1), tm.Function(ctx, tm.SPACE_P1)
    a.fill_coefficient(L, tm.COEFF_ALPHA)
    b.fill_coefficient(L, tm.COEFF_BETA)
    op = tm.Operator(ctx, tm.FORM_N1, [a, b])
    x.fill_seeded(L, 9)
    op.apply(x, y, L)
    got = y.download(L)
    h.update(got.tobytes())
    op.set_variant(1)  # the per-cube kernel (independent check)
    op.apply(x, y, L)
    ref = y.download(L)
    worst = max(worst, float(abs(got - ref).max() / abs(ref).max()))
print(os.path.basename(os.environ.get("TETMF_LIB", "default")), h.hexdigest()[:16], f"max rel diff vs variant 1: {worst:.2e}")
