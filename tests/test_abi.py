"""CPU tests of the product's host side through the C ABI (no GPU): the
library loads and exports every declared symbol, the reference numbering
and interface groups of the layout, the per-orientation tables against the
reference's FormSystem::local_matrix, and the error model."""
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "tetmf_b200.h")


def header_symbols():
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"^(?:int|const char\*)\s+(tetmf_\w+)\(", txt, flags=re.M)))


def test_exports_every_declared_symbol(tm):
    syms = header_symbols()
    assert len(syms) >= 30
    L = tm.lib()
    for s in syms:
        assert hasattr(L, s), s
    assert set(syms) <= set(tm.exported_symbols()) | {"tetmf_ctx_create", "tetmf_version"}
    assert b"sm_100a" in L.tetmf_version()


def lattice_points(n):
    return np.array([(x, y, z) for z in range(n + 1) for y in range(n + 1 - z) for x in range(n + 1 - z - y)])


def macro_geometry(mesh):
    if mesh == "single-tet":
        return np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1.0]]), [[0, 1, 2, 3]]
    V = np.array([[x, y, z] for z in range(2) for y in range(2) for x in range(2)], float)
    T = []
    for p in [(0, 1, 2), (0, 2, 1), (1, 0, 2), (1, 2, 0), (2, 0, 1), (2, 1, 0)]:
        a = [0, 0, 0]
        a[p[0]] = 1
        b = list(a)
        b[p[1]] = 1
        t = [0, a[0] + 2 * a[1] + 4 * a[2], b[0] + 2 * b[1] + 4 * b[2], 7]
        P = V[t]
        if np.linalg.det((P[1:] - P[0]).T) < 0:
            t[2], t[3] = t[3], t[2]
        T.append(t)
    return V, T


DIRS = np.array([[1, 0, 0], [0, 1, 0], [0, 0, 1], [1, -1, 0], [1, 0, -1], [0, 1, -1], [1, 1, -1]])
BASE = np.array([[0, 0, 0], [0, 0, 0], [0, 0, 0], [0, 1, 0], [0, 0, 1], [0, 0, 1], [0, 0, 1]])


def slot_geometry(ctx, space, level, mesh):
    """World geometry of every storage slot: (macro-local index, base, tip)."""
    V, T = macro_geometry(mesh)
    n = 1 << level
    ms, cs = ctx.layout(space, level)
    out = []
    for li, m in enumerate(ctx.local_macros()):
        v0 = V[T[m][0]]
        E = np.array([V[T[m][c + 1]] - v0 for c in range(3)])
        if space == 0:
            pts = lattice_points(n)
            out.append((li * ms + np.arange(len(pts)), v0 + pts @ E / n, None))
        else:
            eoff = 0
            if space == 1:  # P2: vertex block (32-padded) before the edge blocks
                pts = lattice_points(n)
                out.append((li * ms + np.arange(len(pts)), v0 + pts @ E / n, None))
                eoff = -(-len(pts) // 32) * 32
            for c in range(7):
                pts = lattice_points(n - 1)
                valid = np.ones(len(pts), bool) if c < 6 else pts.sum(1) <= n - 2
                idx = li * ms + eoff + c * cs + np.arange(len(pts))
                P = pts + BASE[c]
                out.append((idx[valid], (v0 + P @ E / n)[valid], (v0 + (P + DIRS[c]) @ E / n)[valid]))
    return out


@pytest.mark.parametrize("mesh", ["single-tet", "cube6"])
@pytest.mark.parametrize("form", ["P1", "N1"])
@pytest.mark.parametrize("level", [1, 2, 3])
def test_ref_numbering_matches_reference_geometry(tm, mesh, form, level):
    from oracle.refapi import PortSystem
    space = tm.SPACE_ND1 if form == "N1" else tm.SPACE_P1
    ctx = tm.Context(mesh, device=-1)
    m, nd = ctx.ref_map(space, level)
    ref = PortSystem(mesh, form, level)  # pinned to the reference by test_oracle.py
    assert nd == ref.num_dofs
    kind, a, b = ref.dof_geometry()
    owners = np.zeros(nd, int)
    for idx, base, tip in slot_geometry(ctx, space, level, mesh):
        e = m[idx]
        assert (e >= 0).all()
        ids = e >> 2
        neg = (e & 2) != 0
        if tip is None:
            assert np.allclose(a[ids], base)
        else:
            assert np.allclose(a[ids[~neg]], base[~neg]) and np.allclose(b[ids[~neg]], tip[~neg])
            assert np.allclose(a[ids[neg]], tip[neg]) and np.allclose(b[ids[neg]], base[neg])
        np.add.at(owners, ids[(e & 1) == 1], 1)
    assert (owners == 1).all()


@pytest.mark.parametrize("mesh", ["single-tet", "cube6", "cubes2", "cubes2x1x3"])
@pytest.mark.parametrize("form", ["P1", "N1"])
def test_dirichlet_mask_matches_reference_interior(tm, tmp_path, mesh, form):
    """Dirichlet carriers = boundary flag OR-merged over every macro holding the
    carrier (fespace.cpp:207-214, 226). Kuhn-cube meshes have macros that
    touch the domain boundary only along an edge or a vertex."""
    from oracle.refapi import PortSystem, write_kuhn_mesh
    space = tm.SPACE_ND1 if form == "N1" else tm.SPACE_P1
    level = 2
    ctx = tm.Context(mesh, device=-1)
    port_mesh = mesh
    if mesh.startswith("cubes"):
        dims = [int(v) for v in mesh[5:].split("x")]
        port_mesh = str(tmp_path / "kuhn.mesh")
        write_kuhn_mesh(port_mesh, *dims)
    want = PortSystem(port_mesh, form, level).interior()
    got = ctx.interior(space, level)
    assert got.shape == want.shape
    assert np.array_equal(got, want), (int((got != want).sum()), got.size)


@pytest.mark.parametrize("mesh", ["single-tet", "cube6"])
@pytest.mark.parametrize("level", [1, 2, 3])
def test_p2_ref_numbering_matches_reference_geometry(tm, mesh, level):
    """P2 (the P2V form's space): vertex + unsigned edge-midpoint DoFs in the
    reference's record order (fespace.cpp:233-307), against the fixed
    reference build's DoF geometry."""
    from oracle.refapi import RefSystem
    ctx = tm.Context(mesh, device=-1)
    m, nd = ctx.ref_map(tm.SPACE_P2, level)
    ref = RefSystem(mesh, "P2V", level)
    assert nd == ref.num_dofs
    kind, a, b = ref.dof_geometry()
    owners = np.zeros(nd, int)
    for idx, base, tip in slot_geometry(ctx, tm.SPACE_P2, level, mesh):
        e = m[idx]
        assert (e >= 0).all()
        assert not (e & 2).any()  # no orientation signs on P2 edges
        ids = e >> 2
        if tip is None:
            assert (kind[ids] == 0).all() and np.allclose(a[ids], base)
        else:
            assert (kind[ids] == 1).all()
            same = np.isclose(a[ids], base).all(1) & np.isclose(b[ids], tip).all(1)
            swap = np.isclose(a[ids], tip).all(1) & np.isclose(b[ids], base).all(1)
            assert (same | swap).all()
        np.add.at(owners, ids[(e & 1) == 1], 1)
    assert (owners == 1).all()


@pytest.mark.parametrize("space", [0, 1, 2])
def test_interface_groups_are_geometric_copies(tm, space):
    ctx = tm.Context("cube6", device=-1)
    level = 3
    off, cp = ctx.local_groups(space, level)
    geo = np.zeros((ctx.layout(space, level)[0] * 6, 6))
    for idx, base, tip in slot_geometry(ctx, space, level, "cube6"):
        geo[idx, :3] = base
        geo[idx, 3:] = base if tip is None else tip
    assert len(off) > 1
    for g in range(len(off) - 1):
        c = cp[off[g]:off[g + 1]]
        assert len(c) >= 2
        st = c >> 1
        neg = (c & 1) == 1
        # every copy is the same carrier; sign = orientation relative to the first copy's owner
        for k in range(len(c)):
            a, b = geo[st[k], :3], geo[st[k], 3:]
            if neg[k]:
                a, b = b, a
            a0, b0 = geo[st[0], :3], geo[st[0], 3:]
            if neg[0]:
                a0, b0 = b0, a0
            if space == 1:  # P2 edge DoFs are unsigned: same carrier, any direction, no sign
                assert not neg.any()
                assert (np.allclose(a, a0) and np.allclose(b, b0)) or (np.allclose(a, b0) and np.allclose(b, a0))
            else:
                assert np.allclose(a, a0) and np.allclose(b, b0)


@pytest.mark.parametrize("mesh", ["single-tet", "cube6"])
def test_tables_match_reference_local_matrix(tm, mesh):
    """Per-orientation exact tables vs the reference's local_matrix (degree 3
    for N1: local_matrix's fixed 16-entry arrays overflow for the 27-point
    rule, forms.cpp:148-149)."""
    import ctypes
    from oracle.refapi import REF_FIXED_LIB, RefSystem, ref_fixed_lib
    if not os.path.exists(REF_FIXED_LIB):
        pytest.skip("oracle/_ref not built")
    L = ref_fixed_lib().L
    L.ref_local_matrix.restype = ctypes.c_int
    dp = ctypes.POINTER(ctypes.c_double)
    L.ref_local_matrix.argtypes = [ctypes.c_void_p] + [ctypes.c_int] * 5 + [dp, dp, ctypes.c_int, dp]
    ctx = tm.Context(mesh, device=-1)
    level = 2
    for form, fid, nloc, deg in [("P1", tm.FORM_P1, 4, 2), ("N1", tm.FORM_N1, 6, 3)]:
        ref = RefSystem(mesh, form, level)
        p1 = RefSystem(mesh, "P1", level)
        nc = int(ref.lib.coeff_num_dofs(ref.h))
        rng = np.random.default_rng(0)
        c0, c1 = rng.uniform(1, 2, nc), rng.uniform(1, 2, nc)
        for m in range(ctx.num_macros()[0]):
            for o in range(6):
                out = np.empty(nloc * nloc)
                rc = L.ref_local_matrix(ref.h, m, o, 0, 0, 0, c0.ctypes.data_as(dp), c1.ctypes.data_as(dp), deg,
                                        out.ctypes.data_as(dp))
                assert rc == nloc
                ids = (ctypes.c_longlong * 10)()
                sg = (ctypes.c_double * 10)()
                L.ref_local_dofs(p1.h, m, o, 0, 0, 0, ids, sg)
                cid = np.array(list(ids)[:4])
                B = ctx.local_matrix(fid, level, m, o, c0[cid], c1[cid]) if form == "N1" else \
                    ctx.local_matrix(fid, level, m, o)
                A = out.reshape(nloc, nloc)
                assert np.abs(A - B).max() <= 1e-14 * np.abs(A).max()


@pytest.mark.parametrize("mesh", ["single-tet", "cube6"])
def test_p2v_tables_match_reference_local_matrix(tm, mesh):
    """P2V exact tables (k in P2, degree-4 integrand) vs the reference's
    local_matrix with the degree-4 (Keast, 11-point) rule; local DoF order
    vertices then edges (0,1),(0,2),(0,3),(1,2),(1,3),(2,3) (fespace.hpp:27-28)."""
    import ctypes
    from oracle.refapi import REF_FIXED_LIB, RefSystem, ref_fixed_lib
    if not os.path.exists(REF_FIXED_LIB):
        pytest.skip("oracle/_ref not built")
    L = ref_fixed_lib().L
    L.ref_local_matrix.restype = ctypes.c_int
    dp = ctypes.POINTER(ctypes.c_double)
    L.ref_local_matrix.argtypes = [ctypes.c_void_p] + [ctypes.c_int] * 5 + [dp, dp, ctypes.c_int, dp]
    ctx = tm.Context(mesh, device=-1)
    level = 2
    ref = RefSystem(mesh, "P2V", level)
    nc = int(ref.lib.coeff_num_dofs(ref.h))
    k = np.random.default_rng(1).uniform(1, 2, nc)
    for m in range(ctx.num_macros()[0]):
        for o in range(6):
            for (x, y, z) in [(0, 0, 0), (1, 0, 0)]:
                out = np.empty(100)
                rc = L.ref_local_matrix(ref.h, m, o, x, y, z, k.ctypes.data_as(dp), None, 4, out.ctypes.data_as(dp))
                assert rc == 10
                ids = (ctypes.c_longlong * 10)()
                sg = (ctypes.c_double * 10)()
                assert L.ref_local_dofs(ref.h, m, o, x, y, z, ids, sg) == 10
                B = ctx.local_matrix(tm.FORM_P2V, level, m, o, k[np.array(list(ids))], None)
                A = out.reshape(10, 10)
                assert np.abs(A - B).max() <= 1e-13 * np.abs(A).max()


def test_stencil_properties(tm):
    ctx = tm.Context("single-tet", device=-1)
    S = ctx.stencil(4, 0)
    assert abs(S[0].sum()) < 1e-14                # interior rows of -Laplace sum to zero
    assert np.count_nonzero(np.abs(S[0]) > 1e-14) == 15
    # corner (0,0,0) of the reference tet at L4 touches only the WU element:
    # vol = 1/(6*16^3), grad = 16 * reference gradients
    assert np.allclose(S[7][[0, 1, 3, 5]], [768 / 24576, -256 / 24576, -256 / 24576, -256 / 24576])
    assert np.count_nonzero(np.abs(S[7]) > 1e-14) == 4


def test_error_model(tm):
    with pytest.raises(tm.InvalidArgument):
        tm.Context("no-such-mesh-file", device=-1)
    ctx = tm.Context("cube6", device=-1)
    with pytest.raises(tm.InvalidArgument):
        tm.Operator(ctx, tm.FORM_N1, [])           # N1 expects 2 coefficient fields
    with pytest.raises(tm.InvalidArgument):
        tm.Operator(ctx, tm.FORM_P2V, [])          # P2V expects k in P2
    x = tm.Function(ctx, tm.SPACE_P1)
    e = tm.Function(ctx, tm.SPACE_ND1)
    with pytest.raises(tm.InvalidArgument):
        tm.Operator(ctx, tm.FORM_P1K, [])          # P1K expects k
    with pytest.raises(tm.InvalidArgument):
        tm.Operator(ctx, tm.FORM_N1, [x, e])        # coefficients live in P1
    with pytest.raises(tm.InvalidArgument):
        ctx.layout(tm.SPACE_ND1, 15)               # levels 0..14
    assert ctx.layout(tm.SPACE_ND1, 0) is not None  # level 0: one anchor per edge class
    with pytest.raises(tm.InvalidArgument):
        x.size(3)                                  # planning-only context owns no device memory


def test_host_bodies(tm):
    # K4 body: copies summed in order, written back with signs
    y = np.array([1.0, 2.0, 3.0, 4.0])
    off = np.array([0, 3], dtype=np.int64)
    cp = np.array([0 << 1, (1 << 1) | 1, 2 << 1], dtype=np.int64)
    tm.host_local_sum(off, cp, y)
    assert y.tolist() == [2.0, -2.0, 2.0, 4.0]
    send = tm.host_pack(np.array([5.0, 6.0]), np.array([(1 << 1) | 1, 0], dtype=np.int64))
    assert send.tolist() == [-6.0, 5.0]
    y = np.array([1.0, 10.0])
    tm.host_combine(y, np.array([2.0]), np.array([0, 2], dtype=np.int64),
                    np.array([(0 << 2), (0 << 2) | 2], dtype=np.int64))
    assert y.tolist() == [3.0, 10.0]


@pytest.mark.gpu
def test_set_stream_switch_orders_pending_work(tm):
    """switching streams must order the old stream's pending work
    before the new stream's (tetmf_ctx_set_stream records an event on the old
    stream and makes the new one wait); NULL selects the context's own stream."""
    import torch
    level = 7
    ctx = tm.Context("cube6", device=0)
    a, b = tm.Function(ctx, tm.SPACE_ND1), tm.Function(ctx, tm.SPACE_ND1)
    al, be = tm.Function(ctx, tm.SPACE_P1), tm.Function(ctx, tm.SPACE_P1)
    al.fill_coefficient(level, tm.COEFF_ALPHA)
    be.fill_coefficient(level, tm.COEFF_BETA)
    op = tm.Operator(ctx, tm.FORM_N1, [al, be])
    a.fill_seeded(level, 3)
    op.apply(a, b, level)
    ctx.synchronize()
    want = b.download(level)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    for _ in range(3):
        ctx.set_stream(s1.cuda_stream)
        op.apply(a, b, level)           # queued on s1
        ctx.set_stream(s2.cuda_stream)  # download runs on s2: must see the finished apply
        assert np.array_equal(b.download(level), want)
        ctx.set_stream(None)            # back to the context's own stream
        op.apply(a, b, level)
        assert np.array_equal(b.download(level), want)
