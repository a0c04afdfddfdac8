"""Generates tests/golden/*.npz from the REFERENCE itself (oracle/_ref).

Run here (where /root/reference exists and oracle/_ref is built):
    make -C oracle ref && python tests/golden/make_golden.py

Fixtures hold, per case: the seeded input x (reference numbering), the
coefficient vectors, the reference outputs w (reference_apply: P1/P1K
degree 2, N1 degree 5) from the fixed build (libtetmf_ref_fixed.so) and from
the verbatim build (libtetmf_ref.so, documents the fill_map defect), the
DoF geometry and the interior mask. Large configs (C2, C3) store
size-independent checksums of w instead of w itself.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle.refapi import RefSystem  # noqa: E402

SMALL = [(m, f, l) for m in ("single-tet", "cube6") for f in ("P1", "P1K", "N1") for l in (1, 2, 3)]
SEED = 42


def checksums(w: np.ndarray) -> np.ndarray:
    i = np.arange(w.size, dtype=np.float64)
    return np.array([w.sum(), (w * w).sum(), (w * np.cos(0.001 * i)).sum(), np.abs(w).max()])


def case(mesh, form, level, dirichlet=False, full=True):
    r = RefSystem(mesh, form, level, fixed=True)
    rv = RefSystem(mesh, form, level, fixed=False)
    x = r.seeded_input(SEED, dirichlet)
    c0, c1 = r.coefficients()
    w, _ = r.apply(x, c0, c1)
    wv, _ = rv.apply(x, c0, c1)
    kind, a, b = r.dof_geometry()
    d = dict(x=x, w=w, w_verbatim=wv, interior=r.interior(), num_dofs=np.int64(r.num_dofs),
             seed=np.int64(SEED), dirichlet=np.bool_(dirichlet), w_checksums=checksums(w))
    if c0 is not None:
        d["c0"] = c0
    if c1 is not None:
        d["c1"] = c1
    if full:
        d.update(kind=kind, a=a, b=b)
    else:
        for k in ("x", "w", "w_verbatim", "interior", "c0", "c1"):
            d.pop(k, None)
    return d


def main():
    out = {}
    for mesh, form, level in SMALL:
        out[f"{mesh}/{form}/L{level}"] = case(mesh, form, level)
    for key, d in out.items():
        fn = os.path.join(HERE, key.replace("/", "_") + ".npz")
        np.savez_compressed(fn, **d)
    # BASELINE config 1 in full (single-tet P1 L6, zero Dirichlet on x)
    np.savez_compressed(os.path.join(HERE, "config1_single-tet_P1_L6.npz"),
                        **case("single-tet", "P1", 6, dirichlet=True))
    # configs 2 and 3: checksums only (sizes 366,145 / 318,240)
    np.savez_compressed(os.path.join(HERE, "config2_single-tet_P1K_L7.npz"),
                        **case("single-tet", "P1K", 7, full=False))
    np.savez_compressed(os.path.join(HERE, "config3_single-tet_N1_L6.npz"),
                        **case("single-tet", "N1", 6, full=False))
    print("wrote", len(os.listdir(HERE)) - 1, "files")


if __name__ == "__main__":
    main()
