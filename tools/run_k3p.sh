export PYTHONPATH=$PWD
# K3: smem tables (default) vs parameter-bank tables (N1 variant 2): C5 time, bitwise agreement on a small mesh
run() { python bench.py --steps 8 --warmup 3 --no-e2e --no-cpu-baseline --no-fp64-peak $2 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', round(d['value'],2), round(d['roofline']['kernel_ms'],3), d['roofline']['frac'])"; }
run default ""
run ptab "--variant 2"
python - <<'PY'
import numpy as np, paper_2404_08371_b200 as tm
for mesh, L in [("cube6", 5), ("cubes2", 4), ("single-tet", 6)]:
    ctx = tm.Context(mesh, device=0)
    x, y0, y1 = tm.Function(ctx, tm.SPACE_ND1), tm.Function(ctx, tm.SPACE_ND1), tm.Function(ctx, tm.SPACE_ND1)
    a, b = tm.Function(ctx, tm.SPACE_P1), tm.Function(ctx, tm.SPACE_P1)
    a.fill_coefficient(L, tm.COEFF_ALPHA); b.fill_coefficient(L, tm.COEFF_BETA)
    op = tm.Operator(ctx, tm.FORM_N1, [a, b])
    x.fill_seeded(L, 9)
    op.apply(x, y0, L)
    op.set_variant(2)
    op.apply(x, y1, L)
    print(mesh, L, "bitwise", np.array_equal(y0.download(L), y1.download(L)))
PY
