"""Run selected cfg2-menu transforms (or cfg3/4/5 pipelines) a few times on the
full cfg2 corpus -- a small command for ncu captures (tools only)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from synth import configs as C  # noqa: E402
from synth import gen  # noqa: E402
from paper_1809_06839_b200 import Layout, Pipeline, Plan  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--ops", default="Rotate,Resize512,ShiftHSV,Grayscale")
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--n", type=int, default=2000)
a = ap.parse_args()
sizes = gen.cfg2_sizes(a.n)
b = gen.gen_images(sizes, seed=0, device="cuda")
inl = Layout(b.desc, 3)
for name in a.ops.split(","):
    specs = C.EXTRA_OPS.get(name) or C.CFG2_MENU[name]
    p = Pipeline(specs)
    osz = [p.output_shape(h, w) for h, w in sizes]
    ob = gen.empty_batch(osz, 3, "cuda")
    plan = Plan(p, inl, Layout(ob.desc, 3))
    ws = plan.workspace()
    for r in range(a.reps):
        plan.apply(r, 0, b.buf, ob.buf, workspace=ws)
torch.cuda.synchronize()
print("ok")
