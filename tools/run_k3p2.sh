export PYTHONPATH=$PWD
run() { python bench.py --steps 8 --warmup 3 --no-e2e --no-cpu-baseline --no-fp64-peak $2 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', round(d['value'],2), round(d['roofline']['kernel_ms'],3))"; }
export TETMF_LIB=paper_2404_08371_b200/_lib/variants/libtetmf_k3mb2.so
run mb2_smem ""
run mb2_ptab "--variant 2"
