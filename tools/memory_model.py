"""Memory-volume model of the apply kernels on B200 (the
paper's M_lower / M_upper / layer-condition estimate, PAPER.md section
"Memory Volume and Layer Conditions", restated for this library's loops and
the B200 L2) against the DRAM bytes ncu measured (committed profiles).

  M_lower  every stored DoF / coefficient read once, every output written once
  M_upper  every micro-element reloads all of its DoFs and coefficients and
           read-modify-writes its outputs (no reuse at all)
  M_lc     layer-condition estimate: data is reused from L2 iff the "tail"
           (bytes the whole GPU touches between two uses of the same data)
           fits in the 126 MB L2; otherwise it is reloaded

usage: python tools/memory_model.py  (prints the table in profiles/r2_memory_model.txt)
"""

L2 = 126e6  # bytes (B200)
SMS = 148


def tet(k):
    return (k + 1) * (k + 2) * (k + 3) // 6 if k >= 0 else 0


def sizes(macros, level):
    n = 1 << level
    pts = macros * tet(n)                 # P1 points (stored closure copies)
    edges = macros * 7 * tet(n - 1)       # ND1 / P2-edge slots (7 class blocks)
    elems = macros * n ** 3
    return n, pts, edges, elems


def k1(macros, level, measured):
    """P1 -Laplace, two-plane row walk (k_p1_stencil2.cu). Per point: x
    read, y written. A plane is read by two plane-pair tasks (as A/B and as
    L/U); tasks run z-pairs innermost, so the tail between the two reads is
    the footprint of the resident warps (16 per SM, 4 planes x 10 rows x 34
    entries each) -- far below L2: layer condition holds."""
    n, pts, _, elems = sizes(macros, level)
    lower = 8.0 * 2 * pts
    upper = 8.0 * elems * (4 + 2 * 4)     # 4 vertex reads + 4 RMW of y per element
    tail = SMS * 16 * 4 * 10 * 34 * 8.0
    lc = lower if tail < L2 else 8.0 * (2 * pts + pts)   # fails: x read twice
    return dict(kernel="K1 P1 row walk", config=f"cube6 L{level}" if macros == 6 else f"{macros} macros L{level}",
                lower=lower, upper=upper, lc=lc, tail=tail, measured=measured)


def k3(macros, level, measured):
    """N1 folded cube walk (k_n1_fold.cu), two parity passes. Pass 0 (even
    layers) reads x on planes z, z+1 and alpha / beta, stores y; pass 1 (odd
    layers) reads them again and read-modify-writes y. The tail between a
    plane's pass-0 and pass-1 reads is a whole pass (all planes): the layer
    condition fails, so x, alpha, beta are read twice and y three times."""
    n, pts, edges, elems = sizes(macros, level)
    x = y = 8.0 * edges
    coef = 8.0 * 2 * pts
    lower = x + y + coef
    upper = 8.0 * elems * (6 + 8 + 2 * 6)  # 6 edges + 4 alpha + 4 beta + 6 RMW
    tail = (x + coef + y) / 2              # one pass
    lc = (2 * (x + coef) + 3 * y) if tail >= L2 else lower + y
    return dict(kernel="K3 N1 fold, 2 passes", config=f"{macros} macros L{level}", lower=lower, upper=upper,
                lc=lc, tail=tail, measured=measured)


def p2v(macros, level, measured):
    """P2V factored cube kernel (k_p2v.cu v2): thread per cube, operands
    read per element through L1 / L2, outputs by FP64 atomics at L2 after a
    memset. The tail between two cubes sharing a DoF (the next plane of
    anchors, ~n^2/2 cubes later) is ~ a plane of cube data (27 x + 27 k per
    cube): far below L2, so x and k come from DRAM once; y costs the memset
    write, the first atomic's line fill (read) and the final write-back."""
    n, pts, edges, elems = sizes(macros, level)
    dofs = pts + edges
    x = k = y = 8.0 * dofs
    lower = x + k + y
    upper = 8.0 * elems * (10 + 10 + 2 * 10)
    tail = (n * n / 2) * 27 * 2 * 8.0
    lc = x + k + 2 * y if tail < L2 else 2 * (x + k) + 2 * y
    return dict(kernel="P2V factored cubes", config=f"cube6 L{level}",
                lower=lower, upper=upper, lc=lc, tail=tail, measured=measured)


def k2(macros, level, measured):
    """P1 -div(k grad) column walk (k_p1k_gather.cu p1k_walk_kernel). A warp
    walks 32 rows of one plane; its window holds rows y-1..y+1 of planes
    z-1..z+1 (x and k). Plane z is read as the centre plane by its own tasks
    and as a neighbour plane by the tasks of z-1 and z+1; tasks run z-major,
    so the tail between those reads is about two planes of x and k of the
    whole mesh (6 macros x ~n^2/2 points x 16 B), below L2 at L8."""
    n, pts, _, elems = sizes(macros, level)
    lower = 8.0 * 3 * pts                 # x, k read once, y written once
    upper = 8.0 * elems * (4 + 4 + 2 * 4)
    tail = 2 * macros * (n * n / 2) * 16.0
    lc = lower if tail < L2 else 8.0 * (3 * 2 + 1) * pts
    return dict(kernel="K2 P1K column walk", config=f"cube6 L{level}", lower=lower, upper=upper, lc=lc, tail=tail,
                measured=measured)


ROWS = [
    # measured: ncu dram__bytes_read.sum + dram__bytes_write.sum of the kernel launch(es) of one apply
    k1(6, 8, (138.851328e6 + 100.060416e6, "profiles/r1_k1_rowwalk_ncu_summary.txt")),
    k3(48, 8, (34092914432.0, "profiles/r1_traffic.json (both pass launches, ncu --set full)")),
    p2v(6, 7, (413.534720e6 + 112.126208e6, "profiles/r1_p2v_v2_ncu_summary.txt")),
    k2(6, 8, (275.180288e6 + 117.081600e6, "profiles/r2_k2_walk_ncu_summary.txt")),
]


def main():
    print(f"{'kernel':40s} {'config':16s} {'M_lower':>10s} {'M_lc':>10s} {'M_upper':>10s} {'measured':>10s} "
          f"{'M/M_lower':>9s} {'M/M_lc':>7s} {'tail':>10s}  layer condition (L2 126 MB)")
    for r in ROWS:
        m, src = r["measured"]
        cond = "holds" if r["tail"] < L2 else "fails"
        print(f"{r['kernel']:40s} {r['config']:16s} {r['lower'] / 1e9:9.3f}G {r['lc'] / 1e9:9.3f}G "
              f"{r['upper'] / 1e9:9.3f}G {m / 1e9:9.3f}G {m / r['lower']:9.2f} {m / r['lc']:7.2f} "
              f"{r['tail'] / 1e6:8.1f}MB  {cond}")
    print()
    for r in ROWS:
        print(f"{r['kernel']}: measured from {r['measured'][1]}")


if __name__ == "__main__":
    main()
