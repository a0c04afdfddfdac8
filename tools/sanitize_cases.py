"""Small applies of every hand-written kernel for compute-sanitizer runs
(racecheck / memcheck / synccheck, ONE tool per gpurun call):

  compute-sanitizer --tool racecheck python tools/sanitize_cases.py

K1 box kernel (P1, TMA bulk copies + mbarrier), K2 gather (P1K), K3 fold
kernel (N1, cp.async ring, both parity passes), P2V cube kernel, the
operator diagonals, the interface sum (K4), at levels <= 4 on meshes with
several macros per geometry group. Checks each result against the C port
(oracle/port, test infrastructure) so a sanitizer-clean run is also a
correct one.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2404_08371_b200 as tm  # noqa: E402
import tempfile  # noqa: E402

from oracle.refapi import PortSystem, RefSystem, write_kuhn_mesh  # noqa: E402

CASES = [("cube6", "P1", 4), ("cubes2", "P1", 3), ("single-tet", "P1K", 4), ("cube6", "P1K", 3),
         ("cube6", "N1", 4), ("cubes2", "N1", 3), ("cube6", "P2V", 3)]
FID = {"P1": tm.FORM_P1, "P1K": tm.FORM_P1K, "N1": tm.FORM_N1, "P2V": tm.FORM_P2V}

worst = 0.0
for mesh, form, level in CASES:
    ctx = tm.Context(mesh, device=0)
    sid = tm.FORM_SPACE[FID[form]]
    x, y, d = tm.Function(ctx, sid), tm.Function(ctx, sid), tm.Function(ctx, sid)
    coeffs = []
    if form == "N1":
        a, b = tm.Function(ctx, tm.SPACE_P1), tm.Function(ctx, tm.SPACE_P1)
        a.fill_coefficient(level, tm.COEFF_ALPHA)
        b.fill_coefficient(level, tm.COEFF_BETA)
        coeffs = [a, b]
    elif form in ("P1K", "P2V"):
        k = tm.Function(ctx, tm.SPACE_P1 if form == "P1K" else tm.SPACE_P2)
        k.fill_coefficient(level, tm.COEFF_K)
        coeffs = [k]
    op = tm.Operator(ctx, FID[form], coeffs)
    x.fill_seeded(level, 42)
    op.apply(x, y, level)
    op.diagonal(d, level)
    w = y.export_ref(level)
    rmesh = mesh
    if mesh.startswith("cubes"):
        rmesh = write_kuhn_mesh(os.path.join(tempfile.gettempdir(), f"san_{mesh}.mesh"), int(mesh[5:]))
    ref = (RefSystem if form == "P2V" else PortSystem)(rmesh, form, level)
    c0, c1 = ref.coefficients()
    wr, _ = ref.apply(x.export_ref(level), c0, c1)  # the device's own seeded input
    err = float(np.abs(w - wr).max() / np.abs(wr).max())
    worst = max(worst, err)
    print(f"{mesh} {form} L{level}: rel err {err:.2e}", flush=True)
assert worst <= 1e-12, worst
print("sanitize cases OK")
