"""One-line summary of bench JSON lines: python tools/bsum.py f1.json [f2.json ...]"""
import json
import sys

for f in sys.argv[1:]:
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:  # noqa: BLE001
        print(f, "unreadable", e)
        continue
    r = d.get("roofline", {})
    o = r.get("other_kernel", {})
    print(f"{f}: {d['value'] / 1e9:.3f} G pt-steps/s  {d['ms_per_step']:.3f} ms/step  "
          f"{r.get('kernel')} {r.get('avg_launch_ms', 0):.3f} ms  {o.get('name')} "
          f"{o.get('avg_launch_ms', 0):.3f} ms  clk {d.get('clocks', {}).get('sm_mhz')}  "
          f"diag {d.get('diagnostics', {}).get('ms_per_call')}")
