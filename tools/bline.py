"""Print the key fields of bench.py JSON lines: python tools/bline.py FILE [FILE...]"""
import json, sys
for f in sys.argv[1:]:
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        r = d.get("roofline") or {}
        print(f"{f}: ms/step {d['ms_per_step']:.4f} value {d['value']:.2f} {d['unit']} kernel_ms {r.get('kernel_ms', 0):.4f} frac {r.get('frac')}")
    except Exception as e:  # noqa: BLE001
        print(f"{f}: unreadable ({e})")
