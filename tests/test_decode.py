"""GPU input front-end: nvJPEG batch decode of host
bitstreams into the ragged layout alb_apply consumes.  The decoder is a
library (no oracle function of the method); its output is checked against an
independent CPU decoder (libjpeg via cv2.imdecode) on the same bitstreams
within IDCT/upsampling tolerance, and the decode -> augment composition is
checked against the oracle on the decoded pixels."""
import cv2
import numpy as np
import pytest
import torch

from synth import gen
from tests.harness import cmp_interp, run_oracle

pytestmark = pytest.mark.gpu

SIZES = [(45, 130), (70, 17), (129, 300), (1, 1), (333, 500), (16, 16), (2, 257)]


def encode(img, quality=95, sampling=None):
    params = [cv2.IMWRITE_JPEG_QUALITY, quality]
    if sampling is not None:
        params += [cv2.IMWRITE_JPEG_SAMPLING_FACTOR, sampling]
    ok, buf = cv2.imencode(".jpg", np.ascontiguousarray(img[:, :, ::-1]), params)
    assert ok
    return buf.tobytes()


def cpu_decode(data):
    return cv2.imdecode(np.frombuffer(data, np.uint8), cv2.IMREAD_COLOR)[:, :, ::-1]


def decode_gpu(streams, prefer_hardware):
    from paper_1809_06839_b200 import Decoder, Layout
    dec = Decoder(prefer_hardware)
    sizes = [dec.info(s) for s in streams]
    out = gen.empty_batch(sizes, 3, "cuda")
    dec.decode(streams, Layout(out.desc, 3), out.buf)
    torch.cuda.synchronize()
    return dec, out, sizes


@pytest.mark.parametrize("hw", [True, False])
@pytest.mark.parametrize("sampling", ["444", "420"])
def test_decode_matches_libjpeg(hw, sampling):
    b = gen.gen_images(SIZES, seed=1, first_image_index=0, device="cpu")
    imgs = [b.image(i) for i in range(len(SIZES))]
    sf = cv2.IMWRITE_JPEG_SAMPLING_FACTOR_444 if sampling == "444" else cv2.IMWRITE_JPEG_SAMPLING_FACTOR_420
    streams = [encode(im, 95, sf) for im in imgs]
    dec, out, sizes = decode_gpu(streams, hw)
    assert sizes == [tuple(s) for s in SIZES]
    tot = err = 0
    worst = 0
    for i, s in enumerate(streams):
        g = out.image(i).astype(np.int32)
        r = cpu_decode(s).astype(np.int32)
        assert g.shape == r.shape
        d = np.abs(g - r)
        worst = max(worst, int(d.max()))
        tot += d.size
        err += int(d.sum())
    mean = err / tot
    print("backend hw=%s (got %s) sampling %s: mean |d| %.4f max %d" % (hw, dec.hardware, sampling, mean, worst))
    # same bitstream, two IDCT / colour-conversion implementations
    assert mean <= (0.6 if sampling == "444" else 3.0) and worst <= (6 if sampling == "444" else 40)


def test_decode_errors():
    from paper_1809_06839_b200 import Decoder, Layout
    from paper_1809_06839_b200._lib import AlbError
    dec = Decoder(True)
    img = gen.gen_images([(20, 30)], seed=0, device="cpu").image(0)
    s = encode(img)
    wrong = gen.empty_batch([(21, 30)], 3, "cuda")
    with pytest.raises(AlbError) as e:
        dec.decode([s], Layout(wrong.desc, 3), wrong.buf)
    assert e.value.code == -4
    ok = gen.empty_batch([(20, 30)], 3, "cuda")
    with pytest.raises(AlbError):
        dec.decode([b"not a jpeg at all"], Layout(ok.desc, 3), ok.buf)
    with pytest.raises(AlbError):
        dec.info(b"\xff\xd8\xff")


def test_decode_then_augment_matches_oracle():
    """decode -> cfg4-style fused pipeline: the GPU output equals the oracle
    applied to the GPU-decoded pixels (cfg4 tolerance)."""
    from paper_1809_06839_b200 import Layout, Pipeline, Plan
    from synth import configs as C
    sizes = [(375, 500)] * 6 + [(300, 400)] * 2
    b = gen.gen_images(sizes, seed=4, first_image_index=0, device="cpu")
    streams = [encode(b.image(i), 90) for i in range(len(sizes))]
    dec, dec_out, _ = decode_gpu(streams, True)
    decoded = [dec_out.image(i) for i in range(len(sizes))]
    specs = C.CFG4_OPS
    pipe = Pipeline(specs)
    nchw = torch.empty((len(sizes), 3, 224, 224), dtype=torch.float32, device="cuda")
    plan = Plan(pipe, Layout(dec_out.desc, 3), None)
    plan.apply(9, 0, dec_out.buf, None, nchw)
    torch.cuda.synchronize()
    ref = np.stack([o["nchw"] for o in run_oracle(specs, decoded, seed=9, first=0)])
    g = nchw.cpu().numpy()
    assert (g == ref).mean() >= 0.999
