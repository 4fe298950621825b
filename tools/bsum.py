"""Summarise bench.py JSON lines from stdin: one compact line each."""
import json
import sys

for line in sys.stdin:
    line = line.strip()
    if not line.startswith("{"):
        continue
    d = json.loads(line)
    tag = " ".join(sys.argv[1:])
    if d.get("impl") == "reference":
        print(f"{tag} reference {d['value']:.1f} us/layer cores={d['cpu_baseline']['cores']}")
        continue
    rf, dn = d["roofline"], d.get("dense", {})
    print(f"{tag} value={d['value']:.2f}us kernel={rf['kernel_us']:.2f}us {rf['achieved']:.0f}GB/s "
          f"frac={rf['frac']:.3f} dense={dn.get('us_per_layer', 0):.1f}us ({dn.get('achieved_gbs', 0):.0f}GB/s) "
          f"e2e={d['e2e']['value']:.1f}us clocks={d['clocks'].get('sm_mhz')}")
