#!/usr/bin/env python
"""Print the headline fields of bench.py JSON lines found in log files: python tools/show_bench.py FILE..."""
import json
import sys

for fn in sys.argv[1:]:
    try:
        lines = [l for l in open(fn) if l.startswith("{")]
    except OSError as e:
        print(fn, e)
        continue
    if not lines:
        print(fn, "no JSON line;", "".join(open(fn).readlines()[-3:]).strip()[-300:])
        continue
    d = json.loads(lines[-1])
    r = d.get("roofline") or {}
    e = d.get("e2e") or {}
    print(f"{fn}: {d['value']:.2f} TF {d['ms_per_step']:.1f} ms frac {r.get('frac', 0):.3f} "
          f"e2e {e.get('value')} hpl3 {d.get('hpl3'):.3g} clk {d['clocks']['sm_mhz']} "
          f"{d['clocks']['reasons']} {r.get('per_class_ms')}")
