"""Summarise a bench.py JSON line (stdin) in one line."""
import json
import sys

for line in sys.stdin:
    if not line.startswith("{"):
        continue
    d = json.loads(line)
    r, c = d["roofline"], d["clocks"]
    print(f"value={d['value']:.2f} kernel_ms={r['kernel_ms']:.2f} split_ms={r['split_ms']:.2f} "
          f"fp8_tf={r['achieved']:.0f} sm_mhz={c['sm_mhz']} power={c.get('power_w')} {c['reasons']}")
