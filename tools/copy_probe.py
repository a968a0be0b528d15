"""Reference points for the streaming kernels: torch copy_ of the cfg2 corpus
vs our single-op applies (CUDA events, L2 > corpus avoided by size)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from synth import configs as C  # noqa: E402
from synth import gen  # noqa: E402
from paper_1809_06839_b200 import Layout, Pipeline, Plan  # noqa: E402

sizes = gen.cfg2_sizes(2000)
b = gen.gen_images(sizes, seed=0, device="cuda")
nbytes = sum(h * w * 3 for h, w in sizes)
out = torch.empty_like(b.buf)


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


t = timeit(lambda: out.copy_(b.buf))
print("torch copy_ corpus: %.3f ms  %.1f GB/s (alg %.1f GB/s)" % (t, 2 * b.buf.numel() / t / 1e6, 2 * nbytes / t / 1e6))
inl = Layout(b.desc, 3)
EXTRA = C.EXTRA_OPS
for name in sys.argv[1:] or ["Brightness", "HorizontalFlip", "Grayscale"]:
    specs = EXTRA.get(name) or C.CFG2_MENU[name]
    p = Pipeline(specs)
    ob = gen.empty_batch([p.output_shape(h, w) for h, w in sizes], 3, "cuda")
    plan = Plan(p, inl, Layout(ob.desc, 3))
    ws = plan.workspace()
    t = timeit(lambda: plan.apply(1, 0, b.buf, ob.buf, workspace=ws))
    print("%-16s apply %.3f ms  %.1f GB/s" % (name, t, 2 * nbytes / t / 1e6))
