"""Print ms/step and the per-kernel-kind table of bench JSON lines (quick A/B reading)."""
import json
import sys

for path in sys.argv[1:]:
    try:
        d = json.loads(open(path).read().strip().splitlines()[-1])
    except Exception as e:  # noqa: BLE001
        print(path, "unreadable:", e)
        continue
    r = d.get("roofline", {})
    print(f"{path}: {d.get('config', {}).get('workload')} {d.get('ms_per_step'):.3f} ms/step, "
          f"solve frac {r.get('solve', {}).get('frac')}")
    for k, v in sorted(r.get("kernels", {}).items(), key=lambda kv: -kv[1]["ms_per_step"]):
        print(f"   {k:14s} {v['ms_per_step']:7.3f} ms  share {v['share']:.3f}  frac {v.get('frac')}")
