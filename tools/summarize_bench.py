"""Print the per-transform lines of bench.py JSON outputs."""
import json
import sys

for f in sys.argv[1:]:
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:  # noqa: BLE001
        print(f, "unreadable", e)
        continue
    print("%s value=%.0f %s ms/step=%.3f roof=%s %.3f" % (f, d["value"], d["unit"][:40], d["ms_per_step"],
          d["roofline"].get("kernel"), d["roofline"]["frac"]))
    for k, v in (d.get("per_transform") or {}).items():
        print("   %-24s %12.0f img/s %7.3f ms frac %.3f" % (k, v["images_per_s"], v["ms_per_apply"], v["frac_of_peak"]))
