"""CPU tests of the CHECKERS: the plain-C restatement (oracle/port) pinned
against golden vectors produced by the reference itself
(tests/golden/make_golden.py), SPEC known-answer examples, and the
reference's fill_map defect."""
import glob
import os

import numpy as np
import pytest

from oracle.refapi import PortSystem, RefSystem, REF_LIB, REF_FIXED_LIB, seeded_values

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
HAVE_REF = os.path.exists(REF_LIB) and os.path.exists(REF_FIXED_LIB)
need_ref = pytest.mark.skipif(not HAVE_REF, reason="oracle/_ref not built (make -C oracle ref)")

SMALL = sorted(glob.glob(os.path.join(GOLDEN, "single-tet_*.npz")) + glob.glob(os.path.join(GOLDEN, "cube6_*.npz")))


def parse(fn):
    mesh, form, lev = os.path.basename(fn)[:-4].rsplit("_", 2)
    return mesh, form, int(lev[1:])


def rel(a, b):
    return np.abs(a - b).max() / max(np.abs(b).max(), 1e-300)


@pytest.mark.parametrize("fn", SMALL, ids=lambda f: os.path.basename(f)[:-4])
def test_port_matches_reference_golden(fn):
    g = np.load(fn)
    mesh, form, level = parse(fn)
    p = PortSystem(mesh, form, level)
    assert p.num_dofs == int(g["num_dofs"])
    kind, a, b = p.dof_geometry()
    assert np.array_equal(kind, g["kind"])
    assert np.allclose(a, g["a"], atol=0, rtol=0) and np.allclose(b, g["b"], atol=0, rtol=0)
    assert np.array_equal(p.interior(), g["interior"])
    x = p.seeded_input(int(g["seed"]))
    assert np.array_equal(x, g["x"])
    c0, c1 = p.coefficients()
    if "c0" in g:
        assert np.allclose(c0, g["c0"], rtol=1e-15, atol=1e-15)
    w, _ = p.apply(g["x"], g["c0"] if "c0" in g else None, g["c1"] if "c1" in g else None)
    assert rel(w, g["w"]) <= 1e-12


def test_port_config1_golden():
    g = np.load(os.path.join(GOLDEN, "config1_single-tet_P1_L6.npz"))
    p = PortSystem("single-tet", "P1", 6)
    x = p.seeded_input(42, dirichlet=True)
    assert np.array_equal(x, g["x"])
    assert int((g["interior"] == 1).sum()) == 39711
    w, _ = p.apply(x)
    assert rel(w, g["w"]) <= 1e-12


@pytest.mark.parametrize("name,mesh,form,level", [("config2_single-tet_P1K_L7", "single-tet", "P1K", 7),
                                                   ("config3_single-tet_N1_L6", "single-tet", "N1", 6)])
def test_port_config_checksums(name, mesh, form, level):
    g = np.load(os.path.join(GOLDEN, name + ".npz"))
    p = PortSystem(mesh, form, level)
    assert p.num_dofs == int(g["num_dofs"])
    x = p.seeded_input(42)
    c0, c1 = p.coefficients()
    w, _ = p.apply(x, c0, c1)
    i = np.arange(w.size, dtype=np.float64)
    cs = np.array([w.sum(), (w * w).sum(), (w * np.cos(0.001 * i)).sum(), np.abs(w).max()])
    ref = g["w_checksums"]
    scale = np.array([np.abs(w).sum(), (w * w).sum(), np.abs(w).sum(), np.abs(w).max()])
    assert np.all(np.abs(cs - ref) <= 1e-12 * scale)


# ---------------------------------------------------------------- SPEC KATs
@pytest.mark.parametrize("mesh,form,level,n", [("single-tet", "P1", 1, 10), ("single-tet", "P1", 2, 35),
                                               ("single-tet", "N1", 1, 25), ("cube6", "P1", 1, 27),
                                               ("single-tet", "N1", 6, 318240), ("single-tet", "P1", 7, 366145)])
def test_num_dofs_kat(mesh, form, level, n):
    assert PortSystem(mesh, form, level).num_dofs == n


def test_nd1_cube6_counts():
    # ND1 edges on cube6 L5 = 238,688
    assert PortSystem("cube6", "N1", 5).num_dofs == 238688


def test_seeded_values_orientation():
    # reversing an edge flips its value; vertex values are in [-1, 1]
    a = np.array([[0.0, 0, 0], [0.25, 0.5, 0]])
    b = np.array([[0.25, 0, 0], [0.25, 0.25, 0]])
    kind = np.array([1, 1], dtype=np.uint8)
    v = seeded_values(kind, a, b, 4, 42)
    vr = seeded_values(kind, b, a, 4, 42)
    assert np.array_equal(v, -vr)
    kv = seeded_values(np.zeros(100, np.uint8), np.random.default_rng(0).integers(0, 8, (100, 3)) / 8.0,
                       np.zeros((100, 3)), 8, 1)
    assert np.all(np.abs(kv) <= 1.0)


def test_p1_constant_annihilated():
    # SPEC forms example: interpolate(constant 1) -> w = 0 on interior DoFs
    p = PortSystem("cube6", "P1", 3)
    w, _ = p.apply(np.ones(p.num_dofs))
    assert np.abs(w[p.interior() == 1]).max() < 1e-13


def test_p1_linear_annihilated_port():
    # SPEC forms example: v = interpolate(x) on single-tet L2 -> w = 0 on interior DoFs
    p = PortSystem("single-tet", "P1", 2)
    kind, a, _ = p.dof_geometry()
    w, _ = p.apply(a[:, 0].copy())
    assert np.abs(w[p.interior() == 1]).max() < 1e-13


def test_symmetry_port():
    # SPEC exec property: <A u, v> = <u, A v>
    p = PortSystem("cube6", "N1", 2)
    rng = np.random.default_rng(3)
    c0, c1 = p.coefficients()
    u, v = rng.uniform(-1, 1, p.num_dofs), rng.uniform(-1, 1, p.num_dofs)
    au, _ = p.apply(u, c0, c1)
    av, _ = p.apply(v, c0, c1)
    assert abs(au @ v - u @ av) <= 1e-12 * abs(au @ v)


# ---------------------------------------------------------------- reference defect
@need_ref
def test_reference_fill_map_defect():
    """The verbatim reference aliases DoF ids at level >= 2 and so violates
    its own SPEC example (interior rows of A x for linear x must vanish, checked
    at L4: 455 interior DoFs); the one-line fixed build satisfies it and
    agrees with the port."""
    rv = RefSystem("single-tet", "P1", 4, fixed=False)
    rf = RefSystem("single-tet", "P1", 4, fixed=True)
    kind, a, _ = rf.dof_geometry()
    lin = a[:, 0].copy()
    inner = rf.interior() == 1
    wv, _ = rv.apply(lin)
    wf, _ = rf.apply(lin)
    assert np.abs(wv[inner]).max() > 1e-3      # defect
    assert np.abs(wf[inner]).max() < 1e-13     # fixed build: correct FE operator
    # level 1 P1 has no private carriers: verbatim == fixed there
    r1v, r1f = RefSystem("cube6", "P1", 1, fixed=False), RefSystem("cube6", "P1", 1, fixed=True)
    x = r1f.seeded_input(5)
    assert np.array_equal(r1v.apply(x)[0], r1f.apply(x)[0])


@need_ref
@pytest.mark.parametrize("mesh,form,level", [("cube6", "P1", 4), ("cube6", "N1", 3), ("single-tet", "P1K", 5),
                                             ("single-tet", "N1", 4)])
def test_port_matches_reference_live(mesh, form, level):
    r = RefSystem(mesh, form, level)
    p = PortSystem(mesh, form, level)
    x = r.seeded_input(1)
    c0, c1 = r.coefficients()
    w_r, _ = r.apply(x, c0, c1)
    w_p, _ = p.apply(x, c0, c1)
    assert rel(w_p, w_r) <= 1e-12


@need_ref
def test_reference_quadrature_exactness():
    # SPEC quadrature example: any rule with degree >= 3 integrates x^2 y to 1/360
    import ctypes
    from oracle.refapi import ref_lib
    L = ref_lib().L
    for deg in (3, 4, 5, 6):
        pts = np.empty(3 * 64)
        wts = np.empty(64)
        nq = L.ref_quadrature(deg, pts.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                              wts.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), 64)
        p = pts[:3 * nq].reshape(nq, 3)
        assert abs((wts[:nq] * p[:, 0] ** 2 * p[:, 1]).sum() - 1 / 360) < 1e-14
        assert abs(wts[:nq].sum() - 1 / 6) < 1e-14


@need_ref
def test_orientation_histogram_kat():
    import ctypes
    from oracle.refapi import ref_lib
    L = ref_lib().L
    buf = (ctypes.c_int * (4 * 64))()
    assert L.ref_enumerate(0, 2, buf, 64) == 64
    hist = np.bincount([buf[4 * i] for i in range(64)], minlength=6)
    assert hist.tolist() == [20, 4, 10, 10, 10, 10]  # WU 20, WD 4, others 10
