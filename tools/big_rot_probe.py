"""Probe: Rotate on large single images (debugging helper)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from synth import gen  # noqa: E402
from tests.harness import run_gpu  # noqa: E402

h, w, ang = int(sys.argv[1]), int(sys.argv[2]), float(sys.argv[3])
specs = [{"kind": "Rotate", "lo": [ang], "hi": [ang], "interp": "bilinear", "border": "reflect_101"}]
b = gen.gen_images([(h, w)], seed=12, first_image_index=77, device="cuda")
res = run_gpu(specs, b, seed=5, first=77)
torch.cuda.synchronize()
print("OK", h, w, ang, os.environ.get("ALB_AFFINE_PIPE"))
