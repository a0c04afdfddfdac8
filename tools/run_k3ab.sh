export PYTHONPATH=$PWD
# K3 A/B: C5 kernel time of the default build and tuning builds (tools/build_variant.sh NAME k_n1_fold.cu ...)
run() { python bench.py --steps 8 --warmup 3 --no-e2e --no-cpu-baseline --no-fp64-peak 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', round(d['value'],2), round(d['roofline']['kernel_ms'],3))"; }
run default
for v in "$@"; do TETMF_LIB=paper_2404_08371_b200/_lib/variants/libtetmf_$v.so run $v; done
