"""Run selected cfg2-menu transforms, or the composed configs, a few times --
a small command for ncu captures (tools only).

    python tools/profile_ops.py --ops Rotate,Resize512,cfg3:Rotate,cfg4,cfg5 [--reps R] [--n N]

cfg2 names run on the first N images of the cfg2 corpus; "cfg3:<op>" runs the
cfg3 op on 256 512x512 images with masks, "cfg4" the fused Compose on 1024
500x375 images, "cfg5" the co-transform on 512 1024x1024 images with masks and
boxes (the bench workloads)."""
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
ap.add_argument("--time", type=int, default=0, help="also time this many applies (CUDA events) after the reps")
a = ap.parse_args()


def run(specs, sizes, masks=False, boxes=False):
    n = len(sizes)
    b = gen.gen_images(sizes, seed=0, device="cuda")
    p = Pipeline(specs)
    osz = [p.output_shape(h, w) for h, w in sizes]
    norm = specs[-1]["kind"] == "Normalize"
    ob = None if norm else gen.empty_batch(osz, 3, "cuda")
    nchw = torch.empty((n, 3) + tuple(osz[0]), device="cuda") if norm else None
    mi = mo = None
    bx = None
    if masks:
        bxs, lb, cnt, mi = gen.gen_boxes(sizes, seed=0)
        mi = mi.to("cuda")
        mo = gen.empty_batch(osz, 1, "cuda")
        if boxes:
            bx = [torch.from_numpy(t).cuda() for t in (bxs, lb, cnt)]
    plan = Plan(p, Layout(b.desc, 3), None if norm else Layout(ob.desc, 3),
                None if mi is None else Layout(mi.desc, 1), None if mo is None else Layout(mo.desc, 1),
                C.CFG5_MAX_BOXES if bx else 0, C.CFG5_MIN_VISIBILITY if bx else 0.0)
    ws = plan.workspace()
    bo = [torch.empty_like(t) for t in bx] if bx else [None] * 3
    bi = bx or [None] * 3
    def apply(r):
        plan.apply(r, 0, b.buf, None if ob is None else ob.buf, nchw, None if mi is None else mi.buf,
                   None if mo is None else mo.buf, bi[0], bi[1], bi[2], bo[0], bo[1], bo[2], workspace=ws)
    for r in range(a.reps):
        apply(r)
    torch.cuda.synchronize()
    if a.time:
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        for r in range(a.time):
            apply(r)
        e1.record()
        torch.cuda.synchronize()
        print("time %s %d images: %.3f ms per apply" % (specs[0]["kind"] if len(specs) == 1 else "compose", n,
                                                         e0.elapsed_time(e1) / a.time))


for name in a.ops.split(","):
    if name.startswith("cfg3:"):
        run(C.CFG3_OPS[name[5:]], [(512, 512)] * C.CONFIGS[3]["n"], masks=True)
    elif name == "cfg4":
        run(C.CFG4_OPS, [(375, 500)] * C.CONFIGS[4]["n"])
    elif name == "cfg5":
        run(C.CFG5_OPS, [(1024, 1024)] * C.CONFIGS[5]["n"], masks=True, boxes=True)
    else:
        specs = C.EXTRA_OPS.get(name) or C.CFG2_MENU[name]
        run(specs, gen.cfg2_sizes(a.n))
print("ok")
