"""Kernel launches of P1 applies over loopback virtual ranks in one exchange
mode (run under `ncu --metrics gpu__time_duration.sum --csv` to list them):
with TETMF_EXCHANGE_PUT_FUSED the K1 stencil kernel issues the exchange's puts
(no exchange_put pack kernel); TETMF_EXCHANGE_PUT_PACK launches it.

    python tools/fused_put_launches.py --mode 3 --partition slab
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2404_08371_b200 as tm  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--mode", type=int, default=tm.EXCHANGE_PUT_FUSED)
    ap.add_argument("--partition", choices=("macro", "slab"), default="slab")
    ap.add_argument("--mesh", default="cube6")
    ap.add_argument("--level", type=int, default=6)
    ap.add_argument("--ranks", type=int, default=2)
    ap.add_argument("--applies", type=int, default=2)
    a = ap.parse_args()
    part = tm.PARTITION_SLAB if a.partition == "slab" else tm.PARTITION_MACRO
    group = tm.LoopbackGroup(a.ranks)
    ctxs = group.contexts(a.mesh, device=0, partition=part)
    for c in ctxs:
        c.set_exchange_mode(a.mode)

    def body(r):
        x, y = tm.Function(ctxs[r], tm.SPACE_P1), tm.Function(ctxs[r], tm.SPACE_P1)
        op = tm.Operator(ctxs[r], 0, [])
        x.fill_seeded(a.level, 42)
        y.size(a.level)
        for _ in range(a.applies):
            op.apply(x, y, a.level)
        ctxs[r].synchronize()
        return float(abs(y.download(a.level)).sum())

    print("mode", a.mode, "checksums", tm.run_ranks(body, a.ranks))


if __name__ == "__main__":
    main()
