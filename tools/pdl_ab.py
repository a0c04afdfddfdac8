"""Back-to-back applies (no events between kernels, no flush): the per-apply
time with programmatic dependent launch on or off (TETMF_PDL=1 / 0, read once
per process). bench.py's timed region records events between the kernels, which
keeps them from overlapping; this is the stream a solver loop sees.
usage: TETMF_PDL=0|1 python tools/pdl_ab.py [config ...]"""
import os
import sys

import torch

import bench
import paper_2404_08371_b200 as tm

keys = sys.argv[1:] or ["c4", "c1", "c2", "c2l"]
torch.cuda.set_stream(torch.cuda.Stream())  # a real stream: NULL would select the context's own
for key in keys:
    cfg = bench.CONFIGS[key]
    ctx = tm.Context(cfg["mesh"], device=0)
    stream = torch.cuda.current_stream()
    ctx.set_stream(stream.cuda_stream)
    op, x, y, _ = bench.make_operator(tm, ctx, cfg["form"], cfg["level"], cfg.get("dirichlet", False))
    n = 200
    for _ in range(20):
        op.apply(x, y, cfg["level"])
    best = 1e9
    for rep in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(n):
            op.apply(x, y, cfg["level"])
        e1.record(stream)
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) / n)
    print(f"{key} TETMF_PDL={os.environ.get('TETMF_PDL', '1')}: {1e3 * best:.2f} us per apply (best of 5 x {n} back-to-back)", flush=True)
    del op, x, y, ctx
