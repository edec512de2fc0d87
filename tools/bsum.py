"""Summarise bench JSON lines: value, e2e, roofline kernel, top kernels."""
import json
import sys

for f in sys.argv[1:]:
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:  # noqa: BLE001
        print(f, "ERR", e)
        continue
    print(f, d.get("value"), (d.get("e2e") or {}).get("value"), (d.get("roofline") or {}).get("kernel"),
          (d.get("roofline") or {}).get("frac"), d.get("vcycles_per_step"), d.get("setup_ms_mean"))
    for k, v in list((d.get("kernels") or {}).items())[:8]:
        print("   ", k, v)
