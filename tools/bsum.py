"""One-line summary of bench.py JSON lines: python tools/bsum.py LOG..."""
import json
import sys

for f in sys.argv[1:]:
    lines = [ln for ln in open(f) if ln.startswith("{")]
    if not lines:
        print(f, "no JSON line")
        continue
    d = json.loads(lines[-1])
    e2e = (d.get("e2e") or {}).get("value")
    rf = d.get("roofline") or {}
    print(f"{f}: value={d.get('value'):.1f} {d.get('unit')} ms/step={d.get('ms_per_step'):.4f} e2e={e2e} "
          f"roofline={rf.get('achieved')}/{rf.get('peak')} frac={rf.get('frac')}")
    ks = d.get("kernels") or {}
    print("   " + "  ".join(f"{k}={v['avg_us']:.1f}" for k, v in ks.items()))
