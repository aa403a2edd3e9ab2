"""Summarise a bench.py JSON line from stdin: label, ms/step, value, roofline fractions, clocks."""
import json
import sys

label = sys.argv[1] if len(sys.argv) > 1 else ""
for line in sys.stdin:
    line = line.strip()
    if not line.startswith("{"):
        continue
    d = json.loads(line)
    r = d.get("roofline") or {}
    kt = d.get("kernel_timing") or {}
    ks = " ".join(f"{k}={v['ms'] / max(v['launches'], 1) * 1e3:.1f}us" for k, v in kt.items())
    print(f"{label}: {d['ms_per_step'] * 1e3:.1f} us/step  {d['value']:.3e} upd/s  kernel_frac {r.get('frac')}  "
          f"step_frac {r.get('step_frac_of_roofline')}  sm_mhz {d['clocks']['sm_mhz']} {d['clocks']['reasons']}  [{ks}]")
