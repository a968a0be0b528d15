"""GPU input front-end measurement: N cfg2-sized
synthetic images encoded as JPEG (cv2, quality Q, host memory), then
  * nvJPEG batch decode into the ragged layout (hardware / CUDA backend),
  * decode -> cfg4 fused pipeline (RSC -> Resize224 -> HFlip -> HSV -> BC -> Normalize),
  * CPU reference: cv2.imdecode on T threads,
reported as images/s (CUDA events around the device work; wall clock for CPU).

    python tools/decode_probe.py [--n 2000] [--q 90] [--reps 5]
"""
import argparse
import os
import sys
import time
from concurrent.futures import ThreadPoolExecutor

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import cv2  # noqa: E402
import numpy as np  # noqa: E402
import torch  # noqa: E402

from synth import configs as C  # noqa: E402
from synth import gen  # noqa: E402
from paper_1809_06839_b200 import Decoder, Layout, Pipeline, Plan  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=2000)
ap.add_argument("--q", type=int, default=90)
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--threads", type=int, default=os.cpu_count())
ap.add_argument("--json", default="", help="write the end-to-end line (JSON) to this file")
a = ap.parse_args()

sizes = gen.cfg2_sizes(a.n)
b = gen.gen_images(sizes, seed=0, device="cpu")


def enc(i):
    ok, buf = cv2.imencode(".jpg", np.ascontiguousarray(b.image(i)[:, :, ::-1]), [cv2.IMWRITE_JPEG_QUALITY, a.q])
    return buf.tobytes()


with ThreadPoolExecutor(a.threads) as ex:
    streams = list(ex.map(enc, range(a.n)))
nbytes = sum(len(s) for s in streams)
px = sum(h * w for h, w in sizes)
print("corpus: %d images, %.1f Mpx, %.1f MB JPEG (q=%d, %.2f bits/px)" % (a.n, px / 1e6, nbytes / 1e6, a.q,
                                                                         8 * nbytes / px))
out = gen.empty_batch(sizes, 3, "cuda")
lay = Layout(out.desc, 3)
pipe = Pipeline(C.CFG4_OPS)
plan = Plan(pipe, lay, None)
ws = plan.workspace()
nchw = torch.empty((a.n, 3, 224, 224), dtype=torch.float32, device="cuda")


def timed(fn, reps):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


dec_rate = {}
for hw in (True, False):
    dec = Decoder(hw)
    t = timed(lambda: dec.decode(streams, lay, out.buf), a.reps)
    dec_rate.setdefault(dec.backend, round(a.n / t * 1e3, 1))
    print("nvJPEG %-8s decode        %8.2f ms  %9.0f img/s  %6.2f Gpx/s" % (
        {1: "hardware", 2: "gpu-huff", 0: "default"}[dec.backend], t, a.n / t * 1e3, px / t / 1e6))

    def both():
        dec.decode(streams, lay, out.buf)
        plan.apply(1, 0, out.buf, None, nchw, workspace=ws)

    t2 = timed(both, a.reps)
    print("nvJPEG %-8s decode + cfg4 %8.2f ms  %9.0f img/s" % ({1: "hardware", 2: "gpu-huff", 0: "default"}[dec.backend], t2,
                                                                a.n / t2 * 1e3))
t = timed(lambda: plan.apply(1, 0, out.buf, None, nchw, workspace=ws), a.reps)
print("cfg4 augment alone            %8.2f ms  %9.0f img/s" % (t, a.n / t * 1e3))

# end to end (the GPU does the input work): host JPEG bitstreams ->
# nvJPEG (bitstreams copied to the device inside the decode) -> cfg4 on the GPU ->
# fp32 NCHW batch back into pinned host memory, all inside the timed region
import json  # noqa: E402
from bench import Clocks  # noqa: E402
dec = Decoder(True)
host_out = torch.empty(nchw.shape, dtype=torch.float32).pin_memory()


def e2e():
    dec.decode(streams, lay, out.buf)
    plan.apply(1, 0, out.buf, None, nchw, workspace=ws)
    host_out.copy_(nchw, non_blocking=True)


e2e()
torch.cuda.synchronize()
clk = Clocks(0)
clk.start()
time.sleep(0.3)
te = timed(e2e, a.reps)
clk.stop()
line = {"metric": "images/s end to end: host JPEG -> nvJPEG decode -> cfg4 Compose -> fp32 NCHW in host memory",
        "value": round(a.n / te * 1e3, 1), "unit": "images/s", "ms_per_batch": round(te, 3),
        "batch": a.n, "jpeg_quality": a.q, "jpeg_mb": round(nbytes / 1e6, 1),
        "h2d_bytes_per_batch": nbytes, "d2h_bytes_per_batch": host_out.numel() * 4,
        "decoder_backend": {1: "hardware", 2: "gpu-assisted huffman", 0: "default"}[dec.backend],
        "context": {"decode_only_img_s": dec_rate.get(dec.backend), "cfg4_alone_img_s": round(a.n / t * 1e3, 1),
                    "cv2_imdecode_threads": a.threads},
        "clocks": clk.summary(), "data": "synthetic cfg2-size gradient+noise images, JPEG-encoded by cv2"}
print(json.dumps(line))
if a.json:
    with open(a.json, "w") as f:
        f.write(json.dumps(line) + "\n")
t0 = time.perf_counter()
with ThreadPoolExecutor(a.threads) as ex:
    list(ex.map(lambda s: cv2.imdecode(np.frombuffer(s, np.uint8), cv2.IMREAD_COLOR), streams))
dt = time.perf_counter() - t0
print("cv2.imdecode x %d threads       %8.2f ms  %9.0f img/s" % (a.threads, dt * 1e3, a.n / dt))
