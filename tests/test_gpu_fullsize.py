"""Parity at BASELINE's full sizes through size-independent properties
(the oracle cannot run these sizes): C4 = cube6 L8 P1 (17.0 M DoFs), C5 =
48 macros L8 N1 (942 M DoFs), and the config-2 form P1K at cube6 L8.

* symmetry      <A x, y> = <x, A y>   (x, y with zero Dirichlet values; masked
                inner product of the solver, each interior DoF once)
* positivity    <A x, x> > 0
* linearity     A (x + 2 y) = A x + 2 A y   (entrywise, 1e-12)
* A/B           optimized kernels == first-version kernels (entrywise, 1e-12)
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

CASES = [("cube6", "P1", 8), ("cube6", "P1K", 8), ("cubes2x2x2", "N1", 8)]
FORMS = {"P1": (0, 0), "N1": (2, 2), "P1K": (3, 0)}


class _DevArray:
    """__cuda_array_interface__ view of a library buffer (torch: plumbing only)."""

    def __init__(self, ptr, n):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<f8", "data": (ptr, False), "version": 3}


def _view(fn, level):
    import torch
    return torch.as_tensor(_DevArray(fn.device_ptr(level), fn.size(level)), device="cuda")


def _setup(tm, mesh, form, level):
    fid, sid = FORMS[form]
    ctx = tm.Context(mesh, device=0)
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
    return ctx, tm.Operator(ctx, fid, cf), sid


@pytest.mark.parametrize("mesh,form,level", CASES)
def test_fullsize_symmetry_linearity_positivity(tm, mesh, form, level):
    import torch
    ctx, op, sid = _setup(tm, mesh, form, level)
    x, y, ax, ay, z, az = (tm.Function(ctx, sid) for _ in range(6))
    x.fill_seeded(level, 1, True)
    y.fill_seeded(level, 2, True)
    op.apply(x, ax, level)
    op.apply(y, ay, level)
    s1, s2 = ax.dot(y, level), x.dot(ay, level)
    # scale: sum of |terms| (masked dot of the absolute values)
    ctx.synchronize()
    a_abs, y_abs = tm.Function(ctx, sid), tm.Function(ctx, sid)
    _view(a_abs, level).copy_(_view(ax, level).abs())
    _view(y_abs, level).copy_(_view(y, level).abs())
    torch.cuda.synchronize()
    scale = a_abs.dot(y_abs, level)
    assert abs(s1 - s2) <= 1e-12 * scale, (s1, s2, scale)
    assert ax.dot(x, level) > 0.0
    # linearity
    _view(z, level).copy_(_view(x, level) + 2.0 * _view(y, level))
    torch.cuda.synchronize()
    op.apply(z, az, level)
    ctx.synchronize()
    want = _view(ax, level) + 2.0 * _view(ay, level)
    err = (_view(az, level) - want).abs().max().item()
    assert err <= 1e-12 * want.abs().max().item()


@pytest.mark.parametrize("mesh,form,level", CASES)
def test_fullsize_optimized_vs_first_version(tm, mesh, form, level):
    import torch
    ctx, op, sid = _setup(tm, mesh, form, level)
    x, y0, y1 = (tm.Function(ctx, sid) for _ in range(3))
    x.fill_seeded(level, 3)
    op.apply(x, y0, level)
    op.set_variant(1)
    op.apply(x, y1, level)
    ctx.synchronize()
    a, b = _view(y0, level), _view(y1, level)
    assert (a - b).abs().max().item() <= 1e-12 * b.abs().max().item()
    torch.cuda.synchronize()


@pytest.mark.gpu
@pytest.mark.parametrize("level", [10])
def test_p1_large_level_matches_round1_walk(tm, level):
    """Levels past BASELINE's L8 (single-tet L10: 180 M points per vector):
    the default K1 box kernel (32-bit lattice offsets formed in 64 bits)
    equals the round-1 row walk (variant 9) bitwise."""
    ctx = tm.Context("single-tet", device=0)
    x, y0, y1 = tm.Function(ctx, tm.SPACE_P1), tm.Function(ctx, tm.SPACE_P1), tm.Function(ctx, tm.SPACE_P1)
    op = tm.Operator(ctx, tm.FORM_P1)
    x.fill_seeded(level, 23)
    op.apply(x, y0, level)
    op.set_variant(9)
    op.apply(x, y1, level)
    a, b = y0.download(level), y1.download(level)
    assert np.array_equal(a, b)
    assert np.abs(a).max() > 0.0
