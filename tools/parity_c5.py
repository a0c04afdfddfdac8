"""Parity of the GPU apply against the reference's own FormSystem::apply
(oracle/_ref) at one level, x random in the reference numbering,
coefficients the reference's. Default mesh: config 5's (2x2x2 Kuhn cubes,
48 macros). usage: python tools/parity_c5.py LEVEL [FORM] [MESH]"""
import sys
import tempfile
import time

import numpy as np

import paper_2404_08371_b200 as tm
from oracle.refapi import RefSystem, write_kuhn_mesh

level = int(sys.argv[1]) if len(sys.argv) > 1 else 7
form = sys.argv[2] if len(sys.argv) > 2 else "N1"
mesh = sys.argv[3] if len(sys.argv) > 3 else "cubes2"
fid, sid = {"P1": (tm.FORM_P1, tm.SPACE_P1), "N1": (tm.FORM_N1, tm.SPACE_ND1), "P1K": (tm.FORM_P1K, tm.SPACE_P1),
            "P2V": (tm.FORM_P2V, tm.SPACE_P2)}[form]
path = mesh
if mesh.startswith("cubes"):
    path = tempfile.mktemp(suffix=".mesh")
    write_kuhn_mesh(path, int(mesh[5:]))
t0 = time.time()
r = RefSystem(path, form, level)
c0, c1 = r.coefficients()
x = np.random.default_rng(level).uniform(-1.0, 1.0, r.num_dofs)
w, _ = r.apply(x, c0, c1, degree=0)
t_ref = time.time() - t0
ctx = tm.Context(mesh, device=0)
xs, ys = tm.Function(ctx, sid), tm.Function(ctx, sid)
cf = []
if form == "N1":
    a, b = tm.Function(ctx, tm.SPACE_P1), tm.Function(ctx, tm.SPACE_P1)
    a.import_ref(level, c0)
    b.import_ref(level, c1)
    cf = [a, b]
elif form in ("P1K", "P2V"):
    k = tm.Function(ctx, tm.SPACE_P1 if form == "P1K" else tm.SPACE_P2)
    k.import_ref(level, c0)
    cf = [k]
op = tm.Operator(ctx, fid, cf)
xs.import_ref(level, x)
op.apply(xs, ys, level)
got = ys.export_ref(level)
err = np.abs(got - w).max() / np.abs(w).max()
print(f"{form} {mesh} L{level}: {r.num_dofs} DoFs, reference apply {t_ref:.1f} s, "
      f"max|y_gpu - y_ref| / max|y_ref| = {err:.3e} ({'PASS' if err <= 1e-12 else 'FAIL'} at 1e-12)")
