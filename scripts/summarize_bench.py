"""Print a one-line summary per bench JSON file."""
import json
import sys

for f in sys.argv[1:]:
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:  # noqa: BLE001
        print(f, "unreadable", e)
        continue
    r = d.get("roofline") or {}
    print(f"{d['config']['workload'][:3]} ms/step {d['ms_per_step']:.3f}  evals/s {d['value']:.3e}  "
          f"frac {r.get('frac', 0):.3f}  kernels " + str({k: round(v, 3) for k, v in (r.get('kernel_ms') or {}).items()}))
