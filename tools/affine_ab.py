"""A/B of the affine fast path: k_affine_rt (default) vs k_affine_pipe
(ALB_AFFINE_PIPE=1) on the cfg2 corpus -- outputs must be equal byte for byte
(same coordinate and blend arithmetic), then CUDA-event timing of both."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from synth import configs as C  # noqa: E402
from synth import gen  # noqa: E402
from paper_1809_06839_b200 import Layout, Pipeline, Plan  # noqa: E402

n = int(os.environ.get("AB_N", "2000"))
sizes = gen.cfg2_sizes(n)
b = gen.gen_images(sizes, seed=0, device="cuda")
nbytes = sum(h * w * 3 for h, w in sizes)
inl = Layout(b.desc, 3)


def timeit(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def mode(pipe):
    if pipe:
        os.environ["ALB_AFFINE_PIPE"] = "1"
    else:
        os.environ.pop("ALB_AFFINE_PIPE", None)


SSR = C.CFG2_MENU["ShiftScaleRotate"]
AB = {"SSRfused": SSR + [C.op("VerticalFlip"), C.op("HorizontalFlip", p=0.5),
                         C.op("BrightnessContrast", lo=[0.8, 0.8], hi=[1.2, 1.2])],
      "SSRcrop": SSR + [C.op("RandomCrop", size=(200, 200))],
      "SSRhsv": SSR + [C.op("ShiftHSV", lo=[-20.0, -0.1, -0.1], hi=[20.0, 0.1, 0.1])],
      "RotConst": [C.op("Rotate", lo=[-90.0], hi=[90.0], interp="bilinear", border="constant")]}
names = sys.argv[1:] or ["Rotate", "ShiftScaleRotate"]
ok = True
for name in names:
    specs = AB.get(name) or C.EXTRA_OPS.get(name) or C.CFG2_MENU[name]
    p = Pipeline(specs)
    ob = [gen.empty_batch([p.output_shape(h, w) for h, w in sizes], 3, "cuda") for _ in range(2)]
    plan = Plan(p, inl, Layout(ob[0].desc, 3))
    ws = plan.workspace()
    for seed in (1, 2, 3):
        for k, pipe in enumerate((True, False)):
            mode(pipe)
            ob[k].buf.fill_(0x5A)
            plan.apply(seed, 0, b.buf, ob[k].buf, workspace=ws)
        torch.cuda.synchronize()
        diff = (ob[0].buf != ob[1].buf).sum().item()
        print("%-18s seed %d: bytes differing rt vs pipe = %d" % (name, seed, diff))
        ok = ok and diff == 0
    for pipe in (True, False, True, False):
        mode(pipe)
        t = timeit(lambda: plan.apply(1, 0, b.buf, ob[0].buf, workspace=ws))
        print("%-18s %-5s apply %.3f ms  %.1f GB/s" % (name, "pipe" if pipe else "rt", t, 2 * nbytes / t / 1e6))
mode(False)
print("AB_EQUAL" if ok else "AB_DIFF")
