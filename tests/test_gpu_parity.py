"""GPU parity: the CUDA path (through the C ABI) against the reference's own
FormSystem::apply (oracle/_ref, compiled from the reference sources) on
identical seeded inputs. Tolerance: relative 1e-12 in FP64 (BASELINE.json
north_star), ||y_gpu - y_ref||_inf / ||y_ref||_inf.
"""
import numpy as np
import pytest

from oracle.refapi import RefSystem

RTOL = 1e-12

FORMS = {"P1": (0, 0), "N1": (2, 2), "P1K": (3, 0)}  # form id, space id


def gpu_apply(tm, mesh, form, level, seed, dirichlet=False, via_import=None, coeffs_ref=None):
    fid, sid = FORMS[form]
    ctx = tm.Context(mesh, device=0)
    x = tm.Function(ctx, sid)
    y = tm.Function(ctx, sid)
    cf = []
    if form == "N1":
        a = tm.Function(ctx, tm.SPACE_P1)
        b = tm.Function(ctx, tm.SPACE_P1)
        if coeffs_ref is None:
            a.fill_coefficient(level, tm.COEFF_ALPHA)
            b.fill_coefficient(level, tm.COEFF_BETA)
        else:
            a.import_ref(level, coeffs_ref[0])
            b.import_ref(level, coeffs_ref[1])
        cf = [a, b]
    elif form == "P1K":
        k = tm.Function(ctx, tm.SPACE_P1)
        if coeffs_ref is None:
            k.fill_coefficient(level, tm.COEFF_K)
        else:
            k.import_ref(level, coeffs_ref[0])
        cf = [k]
    op = tm.Operator(ctx, fid, cf)
    if via_import is not None:
        x.import_ref(level, via_import)
    else:
        x.fill_seeded(level, seed, dirichlet)
    op.apply(x, y, level)
    ctx.synchronize()
    return y.export_ref(level), x.export_ref(level)


def ref_apply(mesh, form, level, seed, dirichlet=False):
    r = RefSystem(mesh, form, level)
    x = r.seeded_input(seed, dirichlet)
    c0, c1 = r.coefficients()
    # exact rules: P1/P1K degree 2 (reference_apply), N1 degree 5 (reference_apply)
    w, _ = r.apply(x, c0, c1, degree=0)
    return w, x, (c0, c1)


def relerr(a, b):
    return np.abs(a - b).max() / max(np.abs(b).max(), 1e-300)


CASES = [
    ("single-tet", "P1", 0), ("cube6", "P1", 0), ("single-tet", "P1K", 0), ("cube6", "P1K", 0),
    ("single-tet", "N1", 0), ("cube6", "N1", 0),
    ("single-tet", "P1", 1), ("single-tet", "P1", 2), ("single-tet", "P1", 3), ("single-tet", "P1", 5),
    ("single-tet", "P1", 6),
    ("cube6", "P1", 1), ("cube6", "P1", 2), ("cube6", "P1", 4),
    ("single-tet", "P1K", 1), ("single-tet", "P1K", 3), ("single-tet", "P1K", 5),
    ("cube6", "P1K", 2), ("cube6", "P1K", 4),
    ("single-tet", "N1", 1), ("single-tet", "N1", 2), ("single-tet", "N1", 4),
    ("cube6", "N1", 1), ("cube6", "N1", 2), ("cube6", "N1", 3),
]


@pytest.mark.gpu
@pytest.mark.parametrize("mesh,form,level", CASES)
def test_parity_seeded(tm, mesh, form, level):
    w_ref, x_ref, _ = ref_apply(mesh, form, level, seed=42)
    w_gpu, x_gpu = gpu_apply(tm, mesh, form, level, seed=42)
    # the device generator reproduces the layout-independent seeded input
    assert np.array_equal(x_gpu, x_ref)
    assert relerr(w_gpu, w_ref) <= RTOL


@pytest.mark.gpu
@pytest.mark.parametrize("mesh,form,level", [("single-tet", "P1", 4), ("cube6", "N1", 2), ("cube6", "P1K", 3)])
def test_parity_import_export(tm, mesh, form, level):
    """Reference vectors in, reference vectors out (FormSystem::apply drop-in)."""
    w_ref, x_ref, coeffs = ref_apply(mesh, form, level, seed=7)
    w_gpu, _ = gpu_apply(tm, mesh, form, level, seed=0, via_import=x_ref, coeffs_ref=coeffs)
    assert relerr(w_gpu, w_ref) <= RTOL


@pytest.mark.gpu
def test_config1_dirichlet(tm):
    """BASELINE config 1: P1 -Laplace, single-tet L6, zero Dirichlet on x."""
    w_ref, x_ref, _ = ref_apply("single-tet", "P1", 6, seed=42, dirichlet=True)
    w_gpu, x_gpu = gpu_apply(tm, "single-tet", "P1", 6, seed=42, dirichlet=True)
    assert np.array_equal(x_gpu, x_ref)
    assert relerr(w_gpu, w_ref) <= RTOL


@pytest.mark.gpu
@pytest.mark.parametrize("mesh,form,level", [("cube6", "P1", 7), ("single-tet", "P1", 8), ("cubes1x1x2", "P1", 5),
                                             ("cube6", "N1", 6), ("single-tet", "N1", 7), ("cubes2", "N1", 4),
                                             ("cubes2", "N1", 6), ("cubes1x1x2", "N1", 7),
                                             ("cube6", "P1K", 6), ("single-tet", "P1K", 8)])
def test_optimized_vs_first_version(tm, mesh, form, level):
    """A/B: optimized kernels (variant 0) vs the first-version kernels
    (variant 1) on identical inputs at sizes beyond the oracle's reach."""
    fid, sid = FORMS[form]
    ctx = tm.Context(mesh, device=0)
    x, y0, y1 = tm.Function(ctx, sid), tm.Function(ctx, sid), tm.Function(ctx, sid)
    cf = []
    if form == "N1":
        a, b = tm.Function(ctx, tm.SPACE_P1), tm.Function(ctx, tm.SPACE_P1)
        a.fill_coefficient(level, tm.COEFF_ALPHA)
        b.fill_coefficient(level, tm.COEFF_BETA)
        cf = [a, b]
    elif form == "P1K":
        k = tm.Function(ctx, tm.SPACE_P1)
        k.fill_coefficient(level, tm.COEFF_K)
        cf = [k]
    op = tm.Operator(ctx, fid, cf)
    x.fill_seeded(level, 3)
    op.apply(x, y0, level)
    op.set_variant(1)
    op.apply(x, y1, level)
    a, b = y0.download(level), y1.download(level)
    assert np.abs(a - b).max() <= 1e-13 * np.abs(b).max()


@pytest.mark.gpu
@pytest.mark.parametrize("mesh,level", [("cube6", 8), ("single-tet", 9), ("cubes2", 6), ("cubes1x1x2", 5),
                                        ("single-tet", 1), ("single-tet", 0)])
def test_p1k_cube_kernel_vs_walk_and_gather(tm, mesh, level):
    """K2: the default cube walk (per-cube edge weights, dynamic task queue)
    against the round-2 row walk (variant 3) and the round-1 per-point gather
    (variant 2) on identical inputs, every stored value overwritten (scribbled
    outputs), and bitwise repeatable over launches (the task counters reset
    themselves; each vertex is summed by one task in a fixed order)."""
    ctx = tm.Context(mesh, device=0)
    x, k = tm.Function(ctx, tm.SPACE_P1), tm.Function(ctx, tm.SPACE_P1)
    x.fill_seeded(level, 21)
    k.fill_coefficient(level, tm.COEFF_K)
    op = tm.Operator(ctx, tm.FORM_P1K, [k])
    outs = {}
    for v in (0, 3, 2):
        y = tm.Function(ctx, tm.SPACE_P1)
        y.fill_seeded(level, 77)
        op.set_variant(v)
        op.apply(x, y, level)
        outs[v] = y.download(level)
    scale = np.abs(outs[2]).max()
    assert np.abs(outs[0] - outs[3]).max() <= 1e-13 * scale
    assert np.abs(outs[0] - outs[2]).max() <= 1e-13 * scale
    op.set_variant(0)
    y = tm.Function(ctx, tm.SPACE_P1)
    for rep in range(3):
        y.fill_seeded(level, 100 + rep)
        op.apply(x, y, level)
        assert np.array_equal(y.download(level), outs[0]), f"launch {rep} differs"


@pytest.mark.gpu
@pytest.mark.parametrize("variant", [5, 6, 9, 10])
@pytest.mark.parametrize("mesh,level", [("cube6", 8), ("single-tet", 7), ("cubes2", 6), ("cubes1x1x2", 5),
                                        ("single-tet", 2)])
def test_p1_kernel_variants_bitwise(tm, variant, mesh, level):
    """The K1 kernel variants kept for A/B (5 interior walk + L2 slab
    prefetch, 6 the default selected explicitly, 9 the round-1 two-plane
    walk, 10 persistent double-buffered boxes; 2-4 were removed in round 2,
    7/8 in round 2's second session)
    evaluate the same stencil sums in the same order as the default
    (variant 6: shared-memory boxes filled by per-row TMA bulk copies, face
    pass, diagonal gathers) -- bitwise for the pipelined kernels, over
    repeated runs (their copy pipelines must not race)."""
    ctx = tm.Context(mesh, device=0)
    x, y0, y1 = tm.Function(ctx, tm.SPACE_P1), tm.Function(ctx, tm.SPACE_P1), tm.Function(ctx, tm.SPACE_P1)
    op = tm.Operator(ctx, tm.FORM_P1)
    x.fill_seeded(level, 11)
    op.apply(x, y0, level)
    ref = y0.download(level)
    op.set_variant(variant)
    for _ in range(4):
        op.apply(x, y1, level)
        got = y1.download(level)
        assert np.array_equal(got, ref)


@pytest.mark.gpu
@pytest.mark.parametrize("mesh,form,level", [("cube6", "N1", 3), ("cube6", "P1", 4)])
def test_apply_ref_host_batch(tm, mesh, form, level):
    """tetmf_apply_ref_host_batch (pipelined H2D / apply / D2H over three
    streams, two staging buffers each way) gives every w_k bitwise equal to a
    synchronous tetmf_apply_ref_host of v_k, for more vectors than staging
    buffers; and the first one matches the reference's apply."""
    fid, sid = FORMS[form]
    ctx = tm.Context(mesh, device=0)
    src, dst = tm.Function(ctx, sid), tm.Function(ctx, sid)
    cf = []
    if form == "N1":
        a, b = tm.Function(ctx, tm.SPACE_P1), tm.Function(ctx, tm.SPACE_P1)
        a.fill_coefficient(level, tm.COEFF_ALPHA)
        b.fill_coefficient(level, tm.COEFF_BETA)
        cf = [a, b]
    op = tm.Operator(ctx, fid, cf)
    src.fill_seeded(level, 3)
    nd = src.export_ref(level).size
    rng = np.random.default_rng(5)
    vs = [rng.uniform(-1.0, 1.0, nd) for _ in range(5)]
    ws = [np.zeros(nd) for _ in range(5)]
    op.apply_ref_host_batch(src, dst, level, vs, ws)
    for v, w in zip(vs, ws):
        one = np.zeros(nd)
        op.apply_ref_host(src, dst, level, v, one)
        assert np.array_equal(w, one)
    r = RefSystem(mesh, form, level)
    c0, c1 = r.coefficients()
    wr, _ = r.apply(vs[0], c0, c1, degree=0)
    assert relerr(ws[0], wr) <= RTOL


@pytest.mark.gpu
@pytest.mark.parametrize("mesh,level,reps", [("cube6", 8, 30), ("single-tet", 5, 100)])
def test_k1_repeated_applies_bitwise(tm, mesh, level, reps):
    """The default K1 kernel (per-row TMA copies on one mbarrier per box,
    face CTAs in the same launch) gives bitwise-identical outputs over
    repeated applies, with the output scribbled over in between (no copy /
    barrier race, every output point written every apply)."""
    ctx = tm.Context(mesh, device=0)
    x, y = tm.Function(ctx, tm.SPACE_P1), tm.Function(ctx, tm.SPACE_P1)
    op = tm.Operator(ctx, tm.FORM_P1)
    x.fill_seeded(level, 17)
    op.apply(x, y, level)
    ref = y.download(level)
    for i in range(reps):
        y.fill_seeded(level, 1000 + i)
        op.apply(x, y, level)
        assert np.array_equal(y.download(level), ref)


@pytest.mark.gpu
@pytest.mark.parametrize("form,level", [("N1", 2), ("N1", 4), ("N1", 6), ("P1", 4), ("P1", 7), ("P1K", 5)])
def test_parity_config5_mesh(tm, tmp_path, form, level):
    """Config 5's mesh (2x2x2 Kuhn cubes = 48 macros, many interface
    carriers shared by up to 24 macros) against the reference's own apply on
    the same mesh file: x and the coefficient fields are the reference's,
    imported through the reference numbering."""
    from oracle.refapi import write_kuhn_mesh
    path = str(tmp_path / "kuhn.mesh")
    write_kuhn_mesh(path, 2)
    r = RefSystem(path, form, level)
    c0, c1 = r.coefficients()
    x = np.random.default_rng(level).uniform(-1.0, 1.0, r.num_dofs)
    w, _ = r.apply(x, c0, c1, degree=0)
    got, _ = gpu_apply(tm, "cubes2", form, level, 0, via_import=x, coeffs_ref=(c0, c1))
    assert relerr(got, w) <= RTOL


@pytest.mark.gpu
@pytest.mark.parametrize("mesh,form,level,index,delta", [
    ("cube6", "N1", 3, 24, 1e-9),    # one Gram metric entry g of orientation WU, group 0
    ("cube6", "N1", 3, 21, 1.0),     # kappa = 7200/vol of orientation WU (curl-curl scale, ~2.2e7)
    ("cube6", "P1", 4, 0, 1e-9),     # the centre weight of the interior stencil
    ("single-tet", "P1K", 3, 256 + 1, 1e-9),  # one packed stiffness entry K_o
])
def test_negative_control_corrupted_table(tm, mesh, form, level, index, delta):
    """SPEC.md:599's negative control: a deliberately corrupted table entry
    must make the parity check fail, and restoring it must make it pass --
    the 1e-12 comparison is sensitive to the tables the kernels read."""
    fid, sid = FORMS[form]
    w_ref, x_ref, coeffs = ref_apply(mesh, form, level, seed=42)
    ctx = tm.Context(mesh, device=0)
    x, y = tm.Function(ctx, sid), tm.Function(ctx, sid)
    cf = []
    if form == "N1":
        a, b = tm.Function(ctx, tm.SPACE_P1), tm.Function(ctx, tm.SPACE_P1)
        a.fill_coefficient(level, tm.COEFF_ALPHA)
        b.fill_coefficient(level, tm.COEFF_BETA)
        cf = [a, b]
    elif form == "P1K":
        k = tm.Function(ctx, tm.SPACE_P1)
        k.fill_coefficient(level, tm.COEFF_K)
        cf = [k]
    op = tm.Operator(ctx, fid, cf)
    x.fill_seeded(level, 42)
    op.apply(x, y, level)
    assert relerr(y.export_ref(level), w_ref) <= RTOL
    op.debug_perturb_table(level, index, delta)
    op.apply(x, y, level)
    assert relerr(y.export_ref(level), w_ref) > RTOL  # corrupted -> parity fails
    op.debug_perturb_table(level, index, -delta)
    op.apply(x, y, level)
    assert relerr(y.export_ref(level), w_ref) <= RTOL  # restored -> passes again


@pytest.mark.gpu
def test_apply_ref_host_batch_pinned(tm):
    """The pinned-memory path bench.py measures: host vectors in
    page-locked memory from tetmf_host_alloc, distinct outputs per vector,
    nvec = 6 > the two staging buffers each way -- every w_k bitwise equal to
    the synchronous tetmf_apply_ref_host of v_k."""
    import ctypes
    mesh, form, level = "cube6", "N1", 4
    fid, sid = FORMS[form]
    ctx = tm.Context(mesh, device=0)
    src, dst = tm.Function(ctx, sid), tm.Function(ctx, sid)
    a, b = tm.Function(ctx, tm.SPACE_P1), tm.Function(ctx, tm.SPACE_P1)
    a.fill_coefficient(level, tm.COEFF_ALPHA)
    b.fill_coefficient(level, tm.COEFF_BETA)
    op = tm.Operator(ctx, fid, [a, b])
    nd = src.num_ref_dofs(level)
    nvec = 6
    hv = [tm.host_alloc(8 * nd) for _ in range(nvec)]
    hw = [tm.host_alloc(8 * nd) for _ in range(nvec)]
    try:
        view = lambda p: np.ctypeslib.as_array(ctypes.cast(ctypes.c_void_p(p), ctypes.POINTER(ctypes.c_double)),
                                               shape=(nd,))
        rng = np.random.default_rng(11)
        for p in hv:
            view(p)[:] = rng.uniform(-1.0, 1.0, nd)
        for p in hw:
            view(p)[:] = np.nan
        op.apply_ref_host_batch(src, dst, level, hv, hw)
        for p, q in zip(hv, hw):
            one = np.zeros(nd)
            op.apply_ref_host(src, dst, level, view(p).copy(), one)
            assert np.array_equal(view(q), one)
    finally:
        for p in hv + hw:
            tm.host_free(p)


@pytest.mark.gpu
def test_removed_variants_are_rejected(tm):
    ctx = tm.Context("cube6", device=0)
    x, y = tm.Function(ctx, tm.SPACE_P1), tm.Function(ctx, tm.SPACE_P1)
    op = tm.Operator(ctx, tm.FORM_P1)
    x.fill_seeded(2, 1)
    with pytest.raises(tm.InvalidArgument, match="unknown kernel variant"):
        op.set_variant(11)
    for v in (2, 3, 4, 7, 8):
        op.set_variant(v)
        with pytest.raises(tm.InvalidArgument, match="does not exist"):
            op.apply(x, y, 2)
