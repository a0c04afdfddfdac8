"""P2V: -div(k grad u) with u, k in P2 (forms.cpp:12), on
the GPU against the fixed reference build's FormSystem::reference_apply
(degree 6 >= the exact degree 4), on single-tet, cube6 and a Kuhn-cube mesh.
Seeded x: vertex values at vertex keys, edge-midpoint values at the
key-ascending edge keys (unsigned); k nodally interpolated at vertices and
edge midpoints (fespace.cpp:494-506)."""
import numpy as np
import pytest

from oracle.refapi import RefSystem, seeded_values, write_kuhn_mesh

pytestmark = pytest.mark.gpu


def _setup(tm, mesh, level, seed):
    ctx = tm.Context(mesh, device=0)
    k = tm.Function(ctx, tm.SPACE_P2)
    k.fill_coefficient(level, tm.COEFF_K)
    x = tm.Function(ctx, tm.SPACE_P2)
    x.fill_seeded(level, seed)
    return ctx, k, x, tm.Operator(ctx, tm.FORM_P2V, [k])


@pytest.mark.parametrize("mesh,level", [("single-tet", 0), ("cube6", 0), ("single-tet", 1), ("single-tet", 2), ("single-tet", 3), ("cube6", 1),
                                        ("cube6", 2), ("cubes2", 1), ("cubes2", 2)])
def test_p2v_parity_with_reference(tm, tmp_path, mesh, level):
    port_mesh = mesh
    if mesh.startswith("cubes"):
        port_mesh = str(tmp_path / "kuhn.mesh")
        write_kuhn_mesh(port_mesh, int(mesh[5:]))
    ctx, k, x, op = _setup(tm, mesh, level, 42)
    y = tm.Function(ctx, tm.SPACE_P2)
    op.apply(x, y, level)
    ctx.synchronize()
    ref = RefSystem(port_mesh, "P2V", level)
    kind, a, b = ref.dof_geometry()
    x_ref = seeded_values(kind, a, b, 1 << level, 42, signed_edges=False)
    assert np.array_equal(x.export_ref(level), x_ref)        # seeded input reproduced
    k_ref = ref.interpolate(2)
    assert np.abs(k.export_ref(level) - k_ref).max() <= 1e-15 * np.abs(k_ref).max()
    w, _ = ref.apply(x_ref, k_ref, None, degree=0)
    got = y.export_ref(level)
    assert np.abs(got - w).max() <= 1e-12 * np.abs(w).max()


def test_p2v_cg_recovers_known_solution(tm):
    level = 3
    ctx, k, xs, op = _setup(tm, "cube6", level, 3)
    xs.fill_seeded(level, 3, True)
    b = tm.Function(ctx, tm.SPACE_P2)
    op.apply(xs, b, level)
    b.mask_dirichlet(level)
    x = tm.Function(ctx, tm.SPACE_P2)
    it, rel, ok = op.cg_solve(b, x, level, rtol=1e-12, max_iter=3000)
    assert ok
    want, got = xs.export_ref(level), x.export_ref(level)
    assert np.abs(got - want).max() <= 1e-8 * np.abs(want).max()


@pytest.mark.parametrize("mesh,level", [("single-tet", 2), ("cube6", 1), ("cubes2", 1)])
def test_p2v_diagonal_matches_probed_reference(tm, tmp_path, mesh, level):
    """tetmf_op_diagonal for P2V: d_i = (A e_i)_i through the reference's
    apply, on the owner copies (interface copies hold the same summed value)."""
    port_mesh = mesh
    if mesh.startswith("cubes"):
        port_mesh = str(tmp_path / "kuhn.mesh")
        write_kuhn_mesh(port_mesh, int(mesh[5:]))
    ctx, k, _, op = _setup(tm, mesh, level, 1)
    ref = RefSystem(port_mesh, "P2V", level)
    k_ref = ref.interpolate(2)
    nd = len(k_ref)
    want = np.empty(nd)
    for i in range(nd):
        e = np.zeros(nd)
        e[i] = 1.0
        w, _ = ref.apply(e, k_ref, None, degree=0)
        want[i] = w[i]
    d = tm.Function(ctx, tm.SPACE_P2)
    op.diagonal(d, level)
    ctx.synchronize()
    rmap, nref = ctx.ref_map(tm.SPACE_P2, level)
    assert nref == nd
    raw = d.download(level)
    sel = (rmap >= 0) & ((rmap & 1) == 1)
    got = np.full(nd, np.nan)
    got[rmap[sel] >> 2] = raw[sel]
    assert np.abs(got - want).max() <= 1e-12 * np.abs(want).max()
    assert (want > 0).all()


def test_p2v_jacobi_pcg(tm):
    """Jacobi-PCG on P2V. cube6 (z <= 1): the BASELINE coefficient
    k = 1 + sin(2 pi x) cos(2 pi y) (1 + z) / 2 is >= 0 there; on the 2x2x2
    Kuhn mesh (z up to 2) it turns negative and the form is indefinite."""
    level = 3
    ctx, k, xs, op = _setup(tm, "cube6", level, 5)
    xs.fill_seeded(level, 5, True)
    b = tm.Function(ctx, tm.SPACE_P2)
    op.apply(xs, b, level)
    b.mask_dirichlet(level)
    d = tm.Function(ctx, tm.SPACE_P2)
    op.diagonal(d, level)
    x = tm.Function(ctx, tm.SPACE_P2)
    it, rel, ok = op.cg_solve(b, x, level, rtol=1e-12, max_iter=3000, diag=d)
    assert ok and rel <= 1e-12
    want, got = xs.export_ref(level), x.export_ref(level)
    assert np.abs(got - want).max() <= 1e-8 * np.abs(want).max()


@pytest.mark.parametrize("mesh,level", [("cube6", 6), ("cubes2", 5), ("single-tet", 7), ("cubes1x1x2", 4),
                                        ("single-tet", 0), ("single-tet", 1), ("single-tet", 2), ("cube6", 3),
                                        ("single-tet", 6)])
def test_p2v_factored_vs_first_version(tm, mesh, level):
    """A/B at sizes beyond the oracle's reach: the fold walk (variant 0),
    the factored cube kernel (variant 2) and the first-version table kernel
    (variant 1); every stored value overwritten (scribbled outputs), and the
    fold walk bitwise repeatable (no atomics: one store per DoF, fixed order)."""
    ctx, k, x, op = _setup(tm, mesh, level, 9)
    outs = {}
    for v in (0, 2, 1):
        y = tm.Function(ctx, tm.SPACE_P2)
        y.fill_seeded(level, 77)
        op.set_variant(v)
        op.apply(x, y, level)
        outs[v] = y.download(level)
    b = outs[1]
    assert np.abs(outs[0] - b).max() <= 1e-13 * np.abs(b).max()
    assert np.abs(outs[2] - b).max() <= 1e-13 * np.abs(b).max()
    op.set_variant(0)
    for rep in range(2):
        y = tm.Function(ctx, tm.SPACE_P2)
        y.fill_seeded(level, 100 + rep)
        op.apply(x, y, level)
        assert np.array_equal(y.download(level), outs[0]), f"launch {rep} differs"
