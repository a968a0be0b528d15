"""Print the per-transform lines of bench.py JSON outputs (and the composed configs)."""
import json
import sys


def show(tag, d):
    r = d["roofline"]
    print("%s value=%.0f %s ms/step=%.3f roof=%s %.3f e2e=%s" % (
        tag, d["value"], d["unit"][:40], d["ms_per_step"], r.get("kernel"), r["frac"],
        (d.get("e2e") or {}).get("value")))
    if d.get("trials"):
        print("   trials median %.0f img/s of %s" % (d["trials"]["median"], d["trials"]["images_per_s"]))
    for k, v in (d.get("per_transform") or {}).items():
        print("   %-24s %12.0f img/s %7.3f ms frac %.3f%s" % (
            k, v["images_per_s"], v["ms_per_apply"], v["frac_of_peak"],
            "  graph %.3f ms frac %.3f" % (v["ms_per_apply_graph"], v["frac_of_peak_graph"])
            if "ms_per_apply_graph" in v else ""))


for f in sys.argv[1:]:
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:  # noqa: BLE001
        print(f, "unreadable", e)
        continue
    show(f, d)
    for k, v in (d.get("composed") or {}).items():
        show("  " + k, v)
    if d.get("clocks"):
        print("   clocks", d["clocks"])
