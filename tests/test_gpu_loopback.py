"""Multi-rank apply on ONE B200 through the loopback transport.

P virtual ranks (tetmf_ctx_create_loopback), one host thread each, run the
product's multi-rank path end to end: element kernels on the rank's macros,
K4 for rank-local interface groups, the exchange pack kernel, the transfer
(device-to-device copies between the ranks' buffers instead of NCCL
send/recv), the combine kernel, and the solver's scalar all-gather. The
results must be bitwise equal to the single-rank apply (every interface sum
runs in ascending global macro order, exchange.hpp; the P2V apply too -- its
fold walk has no atomics -- and the P2V operator diagonal, whose kernel
scatters with FP64 atomics, to 1e-13), and within 1e-12 of the
reference's FormSystem::apply (oracle/_ref) after reassembly.

Partitions: contiguous macro ranges (runtime.cpp partition_macros); cube6
over 8 ranks leaves two ranks without macros (they still take part in every
collective step).
"""
import numpy as np
import pytest

from oracle.refapi import RefSystem, write_kuhn_mesh

pytestmark = pytest.mark.gpu

FORMS = {"P1": (0, 0), "P1K": (3, 0), "N1": (2, 2), "P2V": (1, 1)}


def _setup(tm, ctx, form, level, seed=42):
    fid, sid = FORMS[form]
    x, y = tm.Function(ctx, sid), tm.Function(ctx, sid)
    cf = []
    if form == "N1":
        a, b = tm.Function(ctx, tm.SPACE_P1), tm.Function(ctx, tm.SPACE_P1)
        a.fill_coefficient(level, tm.COEFF_ALPHA)
        b.fill_coefficient(level, tm.COEFF_BETA)
        cf = [a, b]
    elif form in ("P1K", "P2V"):
        k = tm.Function(ctx, tm.SPACE_P1 if form == "P1K" else tm.SPACE_P2)
        k.fill_coefficient(level, tm.COEFF_K)
        cf = [k]
    op = tm.Operator(ctx, fid, cf)
    x.fill_seeded(level, seed)
    y.size(level)
    return x, y, op, cf


def _single(tm, mesh, form, level):
    ctx = tm.Context(mesh, device=0)
    x, y, op, cf = _setup(tm, ctx, form, level)
    op.apply(x, y, level)
    d = tm.Function(ctx, FORMS[form][1])
    op.diagonal(d, level)
    ms, _ = ctx.layout(FORMS[form][1], level)
    return ctx, y.download(level).reshape(-1, ms), d.download(level).reshape(-1, ms), ms


def _virtual(tm, mesh, form, level, nranks):
    group = tm.LoopbackGroup(nranks)
    ctxs = group.contexts(mesh, device=0)
    objs = [_setup(tm, c, form, level) for c in ctxs]

    def rank_body(r):
        x, y, op, _ = objs[r]
        op.apply(x, y, level)
        d = tm.Function(ctxs[r], FORMS[form][1])
        op.diagonal(d, level)
        ctxs[r].synchronize()
        return y.download(level), d.download(level)

    res = tm.run_ranks(rank_body, nranks)
    return ctxs, res


CASES = [("cubes2", "N1", 4, 2), ("cubes2", "N1", 5, 4), ("cubes2", "N1", 4, 8), ("cube6", "P1", 6, 2),
         ("cube6", "P1", 6, 4), ("cube6", "P1", 5, 8), ("cubes2", "P1K", 4, 8), ("cube6", "N1", 3, 8),
         ("cube6", "P2V", 3, 4), ("cubes1x1x2", "P1", 5, 3)]


@pytest.mark.parametrize("mesh,form,level,nranks", CASES)
def test_virtual_ranks_bitwise_equal_single_rank(tm, mesh, form, level, nranks):
    ctx1, y1, d1, ms = _single(tm, mesh, form, level)
    ctxs, res = _virtual(tm, mesh, form, level, nranks)
    seen = []
    for c, (y, d) in zip(ctxs, res):
        macros = c.local_macros()
        seen += macros
        assert "loopback virtual rank" in c.transport_info()
        if not macros:
            continue
        if form == "P2V":  # the fold walk apply is atomic-free (bitwise); the diagonal kernel uses atomics
            assert np.array_equal(y.reshape(-1, ms), y1[macros]), f"rank {c.rank}: apply differs"
            assert np.abs(d.reshape(-1, ms) - d1[macros]).max() <= 1e-13 * np.abs(d1).max(), f"rank {c.rank}"
        else:
            assert np.array_equal(y.reshape(-1, ms), y1[macros]), f"rank {c.rank}: apply differs"
            assert np.array_equal(d.reshape(-1, ms), d1[macros]), f"rank {c.rank}: diagonal differs"
    assert sorted(seen) == list(range(ctx1.num_macros()[0]))


@pytest.mark.parametrize("mesh,form,level,nranks", [("cubes2", "N1", 4, 4), ("cube6", "P1", 4, 8),
                                                    ("cubes2", "P1K", 3, 2)])
def test_virtual_ranks_match_reference(tm, tmp_path, mesh, form, level, nranks):
    """Reassemble the ranks' storage into one single-rank function, export it
    in reference numbering and compare with the reference's apply."""
    ctxs, res = _virtual(tm, mesh, form, level, nranks)
    ctx = tm.Context(mesh, device=0)
    x, y, _, _ = _setup(tm, ctx, form, level)
    ms, _ = ctx.layout(FORMS[form][1], level)
    full = np.zeros((ctx.num_macros()[0], ms))
    for c, (yr, _) in zip(ctxs, res):
        if c.local_macros():
            full[c.local_macros()] = yr.reshape(-1, ms)
    y.upload(level, full.ravel())
    got = y.export_ref(level)
    rmesh = write_kuhn_mesh(str(tmp_path / "k.mesh"), int(mesh[5:])) if mesh.startswith("cubes") else mesh
    ref = RefSystem(rmesh, form, level)
    c0, c1 = ref.coefficients()
    want, _ = ref.apply(x.export_ref(level), c0, c1)
    assert np.abs(got - want).max() <= 1e-12 * np.abs(want).max()


def test_virtual_ranks_cg_and_dot(tm):
    """The solver's all-gather through the loopback transport: inner products
    equal the single-rank ones to rounding, CG converges in the same number of
    iterations to the same solution."""
    mesh, form, level, nranks = "cubes2", "P1", 3, 4
    ctx = tm.Context(mesh, device=0)
    xs, b, op, _ = _setup(tm, ctx, form, level, seed=5)
    xs.fill_seeded(level, 5, True)
    op.apply(xs, b, level)
    b.mask_dirichlet(level)
    dot1 = b.dot(b, level)
    x1 = tm.Function(ctx, 0)
    it1, _, ok1 = op.cg_solve(b, x1, level, rtol=1e-10, max_iter=500)
    assert ok1
    ms, _ = ctx.layout(0, level)
    sol1 = x1.download(level).reshape(-1, ms)

    group = tm.LoopbackGroup(nranks)
    ctxs = group.contexts(mesh, device=0)

    def body(r):
        xr, br, opr, _ = _setup(tm, ctxs[r], form, level, seed=5)
        xr.fill_seeded(level, 5, True)
        opr.apply(xr, br, level)
        br.mask_dirichlet(level)
        dot = br.dot(br, level)
        sol = tm.Function(ctxs[r], 0)
        it, _, ok = opr.cg_solve(br, sol, level, rtol=1e-10, max_iter=500)
        return dot, it, ok, sol.download(level)

    out = tm.run_ranks(body, nranks)
    for c, (dot, it, ok, sol) in zip(ctxs, out):
        assert ok and abs(dot - dot1) <= 1e-13 * abs(dot1)
        assert abs(it - it1) <= 1
        assert np.abs(sol.reshape(-1, ms) - sol1[c.local_macros()]).max() <= 1e-8 * np.abs(sol1).max()
    assert len({o[0] for o in out}) == 1  # every rank sees the same scalar


@pytest.mark.parametrize("mesh,level,nranks", [("cube6", 6, 2), ("cube6", 6, 4), ("cube6", 7, 8), ("cubes2", 5, 8),
                                               ("cube6", 8, 8)])
def test_slab_partition_virtual_ranks_bitwise(tm, mesh, level, nranks):
    """Config 4's strong-scaling partition on one GPU: (macro, z-slab) units
    (TETMF_PARTITION_SLAB), the K1 box kernel restricted to each rank's
    planes, the exchange of macro-interface copies between slabs through the
    loopback transport. Every rank's owned points equal the single-rank apply
    bitwise."""
    ctx1, y1, _, ms = _single(tm, mesh, "P1", level)
    group = tm.LoopbackGroup(nranks)
    ctxs = group.contexts(mesh, device=0, partition=tm.PARTITION_SLAB)
    objs = [_setup(tm, c, "P1", level) for c in ctxs]

    def body(r):
        x, y, op, _ = objs[r]
        op.apply(x, y, level)
        ctxs[r].synchronize()
        return y.download(level)

    res = tm.run_ranks(body, nranks)
    n = 1 << level
    tet = lambda k: (k + 1) * (k + 2) * (k + 3) // 6
    starts = np.array([tet(n) - tet(n - z) for z in range(n + 1)])
    zslot = np.searchsorted(starts, np.arange(ms), side="right") - 1
    real = np.arange(ms) < tet(n)
    nmac = ctx1.num_macros()[0]
    owned = np.zeros((nmac, ms), dtype=int)
    for r, y in enumerate(res):
        y = y.reshape(nmac, ms)
        for m, za, zb in tm.slab_units(nmac, level, nranks, r):
            sel = (zslot >= za) & (zslot < zb) & real
            owned[m] += sel
            assert np.array_equal(y[m][sel], y1[m][sel]), f"rank {r} macro {m} planes [{za}, {zb})"
    assert (owned[:, real] == 1).all()  # every point computed by exactly one rank


def test_slab_partition_rejects_other_forms(tm):
    group = tm.LoopbackGroup(2)
    ctx = tm.Context.loopback(group, "cube6", 0, device=0, partition=tm.PARTITION_SLAB)
    a, b = tm.Function(ctx, tm.SPACE_P1), tm.Function(ctx, tm.SPACE_P1)
    with pytest.raises(tm.InvalidArgument, match="slab partition"):
        tm.Operator(ctx, tm.FORM_N1, [a, b])


@pytest.mark.parametrize("mesh,form,level,nranks", [("cubes2", "N1", 4, 4), ("cube6", "P1", 5, 8),
                                                    ("cubes2", "P1K", 4, 3), ("cubes1x1x2", "N1", 4, 2)])
def test_owned_reference_slices(tm, mesh, form, level, nranks):
    """Multi-rank host I/O in reference numbering (tetmf_fn_import_ref_owned /
    export_ref_owned): the ranks' owned slices tile the global vector; import
    of the slices (ghost copies from their owners through the exchange) gives
    every rank the single-rank storage bitwise; the exported slices of the
    apply concatenate to the single-rank export_ref bitwise."""
    ctx = tm.Context(mesh, device=0)
    x, y, op, _ = _setup(tm, ctx, form, level)
    ms, _ = ctx.layout(FORMS[form][1], level)
    xr = x.export_ref(level)
    op.apply(x, y, level)
    w1 = y.export_ref(level)
    xs1 = x.download(level).reshape(-1, ms)

    group = tm.LoopbackGroup(nranks)
    ctxs = group.contexts(mesh, device=0)
    objs = [_setup(tm, c, form, level) for c in ctxs]

    def body(r):
        xx, yy, oo, _ = objs[r]
        lo, hi = xx.owned_ref_range(level)
        xx.fill_seeded(level, 999)  # overwritten by the import
        xx.import_ref_owned(level, np.ascontiguousarray(xr[lo:hi]))
        oo.apply(xx, yy, level)
        return lo, hi, xx.download(level), yy.export_ref_owned(level)

    out = tm.run_ranks(body, nranks)
    pieces = sorted(((lo, hi, w) for lo, hi, _, w in out if hi > lo), key=lambda t: t[0])  # ranks without macros own nothing
    assert pieces[0][0] == 0 and pieces[-1][1] == w1.size
    for (lo, hi, _), (lo2, _, _) in zip(pieces, pieces[1:]):
        assert hi == lo2
    assert np.array_equal(np.concatenate([w for _, _, w in pieces]), w1)
    for c, (_, _, xl, _) in zip(ctxs, out):
        if c.local_macros():
            assert np.array_equal(xl.reshape(-1, ms), xs1[c.local_macros()])


def _modes_run(tm, mesh, form, level, nranks, partition, seeds=(42, 43, 44)):
    """Applies with consecutive seeds (the put mode's window halves alternate)
    under both exchange modes; the level is created inside the rank threads
    because opening a put channel is collective."""
    out = {}
    for mode in (tm.EXCHANGE_SENDRECV, tm.EXCHANGE_PUT, tm.EXCHANGE_PUT_PACK, tm.EXCHANGE_PUT_FUSED):
        group = tm.LoopbackGroup(nranks)
        ctxs = group.contexts(mesh, device=0, partition=partition)
        for c in ctxs:
            c.set_exchange_mode(mode)

        def body(r):
            x, y, op, _ = _setup(tm, ctxs[r], form, level)
            res = []
            for sd in seeds:
                x.fill_seeded(level, sd)
                op.apply(x, y, level)
                ctxs[r].synchronize()
                res.append(y.download(level))
            return res

        out[mode] = tm.run_ranks(body, nranks)
        del ctxs, group
    return out


@pytest.mark.parametrize("mesh,form,level,nranks", [("cubes2", "N1", 4, 2), ("cubes2", "N1", 5, 4),
                                                    ("cubes2", "N1", 4, 8), ("cube6", "P1", 6, 8),
                                                    ("cubes2", "P1K", 4, 3), ("cube6", "P2V", 3, 4),
                                                    ("cubes2", "P1", 5, 3)])
def test_put_exchange_equals_sendrecv(tm, mesh, form, level, nranks):
    """TETMF_EXCHANGE_PUT (the pack kernel stores straight into the peers'
    receive windows; TETMF_EXCHANGE_PUT_FUSED, P1: the K1 stencil kernel
    stores each shared value as it computes it; loopback: device pointers,
    host barrier as the fence)
    gives the send/recv exchange's results bitwise, apply after apply (each
    apply uses the other window half), and the single-rank apply's."""
    out = _modes_run(tm, mesh, form, level, nranks, tm.PARTITION_MACRO)
    for r in range(nranks):
        for k in range(3):
            a = out[tm.EXCHANGE_SENDRECV][r][k]
            for mode in (tm.EXCHANGE_PUT, tm.EXCHANGE_PUT_PACK, tm.EXCHANGE_PUT_FUSED):
                assert np.array_equal(a, out[mode][r][k]), f"mode {mode} rank {r} apply {k}"
    # and the same as one rank (seed 42)
    ctx1, y1, _, ms = _single(tm, mesh, form, level)
    group = tm.LoopbackGroup(nranks)
    ctxs = group.contexts(mesh, device=0)
    for r in range(nranks):
        mac = ctxs[r].local_macros()
        got = out[tm.EXCHANGE_PUT][r][0].reshape(-1, ms) if len(mac) else np.zeros((0, ms))
        for li, m in enumerate(mac):
            assert np.array_equal(got[li], y1[m]), f"rank {r} macro {m}"


@pytest.mark.parametrize("mesh,level,nranks", [("cube6", 6, 4), ("cube6", 7, 8)])
def test_put_exchange_slab_partition(tm, mesh, level, nranks):
    """Config 4's strong-scaling partition with the put exchange: every rank's
    owned points equal the send/recv exchange's bitwise."""
    out = _modes_run(tm, mesh, "P1", level, nranks, tm.PARTITION_SLAB)
    n = 1 << level
    tet = lambda k: (k + 1) * (k + 2) * (k + 3) // 6
    ctx1 = tm.Context(mesh, device=0)
    ms, _ = ctx1.layout(tm.SPACE_P1, level)
    starts = np.array([tet(n) - tet(n - z) for z in range(n + 1)])
    zslot = np.searchsorted(starts, np.arange(ms), side="right") - 1
    real = np.arange(ms) < tet(n)
    nmac = ctx1.num_macros()[0]
    for r in range(nranks):
        for m, za, zb in tm.slab_units(nmac, level, nranks, r):
            sel = (zslot >= za) & (zslot < zb) & real
            for k in range(3):
                a = out[tm.EXCHANGE_SENDRECV][r][k].reshape(nmac, ms)[m][sel]
                for mode in (tm.EXCHANGE_PUT, tm.EXCHANGE_PUT_PACK, tm.EXCHANGE_PUT_FUSED):
                    b = out[mode][r][k].reshape(nmac, ms)[m][sel]
                    assert np.array_equal(a, b), f"mode {mode} rank {r} macro {m} apply {k}"


def test_put_mode_cg_matches_sendrecv(tm):
    """The solver over put-mode virtual ranks (applies through the put
    exchange, inner products through the transport's all-gather)."""
    res = {}
    for mode in (tm.EXCHANGE_SENDRECV, tm.EXCHANGE_PUT):
        group = tm.LoopbackGroup(3)
        ctxs = group.contexts("cubes2", device=0)
        for c in ctxs:
            c.set_exchange_mode(mode)

        def body(r, ctxs=ctxs):
            x, b, op, _ = _setup(tm, ctxs[r], "P1", 3, seed=5)
            x.fill_seeded(3, 5, True)
            op.apply(x, b, 3)
            b.mask_dirichlet(3)
            u = tm.Function(ctxs[r], tm.SPACE_P1)
            it, _, ok = op.cg_solve(b, u, 3, rtol=1e-10, max_iter=500)
            assert ok
            return u.download(3), it

        res[mode] = tm.run_ranks(body, 3)
    for r in range(3):
        assert res[0][r][1] == res[1][r][1]
        assert np.array_equal(res[0][r][0], res[1][r][0])


def test_exchange_mode_set_before_first_level(tm):
    group = tm.LoopbackGroup(2)
    ctx = tm.Context.loopback(group, "cube6", 0, device=0)
    with pytest.raises(tm.InvalidArgument):
        ctx.set_exchange_mode(7)
    ctx.set_exchange_mode(tm.EXCHANGE_SENDRECV)  # (a send/recv exchange opens without the peer)
    f = tm.Function(ctx, tm.SPACE_P1)
    f.size(3)
    with pytest.raises(tm.InvalidArgument, match="before the context's first level"):
        ctx.set_exchange_mode(tm.EXCHANGE_PUT)


def test_nccl_put_channel_selftest(tm):
    """The NCCL device-API path on one B200: a 1-rank communicator,
    ncclMemAlloc + symmetric window registration, a device communicator with
    an LSA barrier, and the LSA barrier kernel (no peers on one GPU)."""
    tm.selftest_nccl_put(0, rounds=4)
