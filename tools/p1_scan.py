"""Throughput of the P1 stencil apply vs working set (mesh x level).
usage: python tools/p1_scan.py"""
import torch
import paper_2404_08371_b200 as tm

for mesh, L in (("single-tet", 7), ("single-tet", 8), ("cube6", 7), ("cubes1x1x2", 7), ("single-tet", 9),
                ("cube6", 8), ("cubes1x1x2", 8), ("cubes2", 7)):
    ctx = tm.Context(mesh, device=0)
    x, y = tm.Function(ctx, 0), tm.Function(ctx, 0)
    x.fill_seeded(L, 1)
    op = tm.Operator(ctx, 0)
    for _ in range(3):
        op.apply(x, y, L)
    ctx.synchronize()
    op.profile(True)
    for _ in range(20):
        op.apply(x, y, L)
    ms, k = op.kernel_stats()
    pts = x.size(L)
    print(f"{mesh:12s} L{L}: storage {pts * 8 * 2 / 1e6:8.1f} MB (x+y)  kernel {ms / k * 1e3:8.1f} us  "
          f"{pts / (ms / k * 1e-3) / 1e9:7.1f} Gpt/s", flush=True)
