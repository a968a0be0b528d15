"""GPU parity of the co-transformed targets (Fig. 2: "a
horizontal flip and a random sized crop ... on both bounding box and instance
mask annotations") and of Normalize alone, through the C ABI against the
oracle:

  images   exact ops byte-equal; resampling ops <= 1 LSB, >= 99.9% exact
  masks    nearest: label-exact except inside the oracle's
           1e-4 px tie band, where either neighbour is accepted (R20)
  boxes    same keep set and labels, normalized coordinates within 1e-5
           (readings R18, R19)
  Normalize  fp32 bit-equal and <= 1e-6 relative given the same u8 input
           (BASELINE.json north_star; O12 / R16)
"""
import numpy as np
import pytest
import torch

from synth import configs as C
from synth import gen
from tests.harness import (cmp_boxes, cmp_cand, cmp_exact, cmp_interp, cmp_resize, random_masks,
                           run_gpu, run_oracle, run_oracle_cand)

pytestmark = pytest.mark.gpu

MEAN, STD = C.IMAGENET_MEAN, C.IMAGENET_STD


@pytest.fixture(scope="module", autouse=True)
def _build():
    from paper_1809_06839_b200 import build
    build.build()
    assert torch.cuda.is_available()


def _targets(sizes, first, seed=0):
    b = gen.gen_images(sizes, seed=seed, first_image_index=first, device="cuda")
    bx, lb, cnt, masks = gen.gen_boxes(sizes, seed=seed, first_image_index=first)
    return b, bx, lb, cnt, masks.to("cuda")


def _run_all(specs, sizes, first, seed, min_vis, image_cmp):
    """image + mask + boxes through one plan, each against the oracle."""
    b, bx, lb, cnt, masks = _targets(sizes, first)
    n = len(sizes)
    res = run_gpu(specs, b, seed=seed, first=first, masks=masks, boxes=bx, labels=lb, count=cnt,
                  max_boxes=bx.shape[1], min_visibility=min_vis)
    imgs = [b.image(i) for i in range(n)]
    mk = [masks.image(i) for i in range(n)]
    ref = run_oracle(specs, imgs, seed=seed, first=first, masks=mk, boxes=bx, labels=lb,
                     count=cnt, min_visibility=min_vis)
    cand = run_oracle_cand(specs, imgs, seed=seed, first=first, masks=mk)
    if image_cmp == "resize":  # one Resize op: exact .5 ties of structured ratios (R33)
        cmp_resize(res["images"], [o["image"] for o in ref], imgs)
    else:
        image_cmp(res["images"], [o["image"] for o in ref])
    cmp_cand(res["masks"], cand, "mask")
    cmp_boxes(res, ref)
    return res, ref


# ------------------------------------------- the paper's Fig. 2 combination

FIG2_CASES = {
    "hflip_then_rsc": [C.op("HorizontalFlip", p=0.5),
                       C.op("RandomSizedCrop", side=(64, 300), size=(256, 256), interp="bilinear")],
    "rsc_then_hflip": [C.op("RandomSizedCrop", side=(64, 375), size=(224, 224), interp="bilinear"),
                       C.op("HorizontalFlip", p=0.5)],
    "rsc_nearest_hflip_p1": [C.op("RandomSizedCrop", side=(100, 200), size=(320, 240),
                                  interp="nearest"),
                             C.op("HorizontalFlip")],
}


@pytest.mark.parametrize("name", list(FIG2_CASES))
@pytest.mark.parametrize("min_vis", [0.0, 0.3])
def test_fig2_hflip_random_sized_crop_image_mask_boxes(name, min_vis):
    """PAPER.md:76-80 (Fig. 2): horizontal flip + random sized crop applied
    consistently to the image, its instance mask and its boxes."""
    specs = FIG2_CASES[name]
    sizes = gen.cfg2_sizes(24, first_image_index=300)
    nearest = specs[0].get("interp") == "nearest"
    _run_all(specs, sizes, 300, 17, min_vis, cmp_exact if nearest else cmp_interp)


# ------------------------------------------------ masks through single ops

MASK_OPS = {
    "RandomCrop64": ([C.op("RandomCrop", size=(64, 64))], "exact"),
    "PadToSize512": ([C.op("PadToSize", size=(512, 512), fill=(9, 8, 7), mask_fill=5)], "exact"),
    "Crop": ([C.op("Crop", origin=(13, 7), size=(200, 150))], "exact"),
    "VerticalFlip": ([C.op("VerticalFlip")], "exact"),
    "Resize512": ([C.op("Resize", size=(512, 512), interp="bilinear")], "interp"),
    "Resize_down": ([C.op("Resize", size=(173, 131), interp="bilinear")], "interp"),
    "Resize_nearest": ([C.op("Resize", size=(390, 277), interp="nearest")], "cand"),
    "RandomSizedCrop64-512": ([C.op("RandomSizedCrop", side=(64, 512), size=(512, 512),
                                    interp="bilinear")], "interp"),
    "Rotate_nearest": ([C.op("Rotate", lo=[-90.0], hi=[90.0], interp="nearest",
                             border="reflect_101")], "cand"),
    "SSR_constant": ([C.op("ShiftScaleRotate", lo=C.SSR_LO, hi=C.SSR_HI, interp="bilinear",
                           border="constant", fill=(1, 2, 3), mask_fill=7)], "interp"),
}


@pytest.mark.parametrize("name", list(MASK_OPS))
def test_random_label_masks_through_op(name):
    """Masks of independent random labels through crop, pad, resize, RSC and
    the warps: every nearest decision is visible in the labels.  Window ops
    are byte-exact; resampling ops exact outside the oracle's tie band."""
    specs, kind = MASK_OPS[name]
    sizes = gen.cfg2_sizes(16, first_image_index=500)
    b = gen.gen_images(sizes, seed=0, first_image_index=500, device="cuda")
    masks, mk = random_masks(sizes, seed=9)
    res = run_gpu(specs, b, seed=23, first=500, masks=masks)
    imgs = [b.image(i) for i in range(len(sizes))]
    ref = run_oracle_cand(specs, imgs, seed=23, first=500, masks=mk)
    if kind == "exact":
        cmp_exact(res["images"], [o["image"] for o in ref])
        cmp_exact(res["masks"], [o["mask"] for o in ref])
    else:
        if kind == "cand":
            cmp_cand(res["images"], ref, "image")
        else:
            cmp_interp(res["images"], [o["image"] for o in ref])
        cmp_cand(res["masks"], ref, "mask")


# ------------------------------------------------ boxes through single ops

BOX_OPS = {
    "HorizontalFlip": [C.op("HorizontalFlip")],
    "VerticalFlip": [C.op("VerticalFlip")],
    "PadToSize512": [C.op("PadToSize", size=(512, 512))],
    "Resize512": [C.op("Resize", size=(512, 512), interp="bilinear")],
    "Resize_aniso": [C.op("Resize", size=(300, 120), interp="bilinear")],
    "RandomSizedCrop64-512": [C.op("RandomSizedCrop", side=(64, 512), size=(512, 512),
                                   interp="bilinear")],
    "Rotate": [C.op("Rotate", lo=[-90.0], hi=[90.0], **C.WARP)],
    "Rotate_fixed_30": [C.op("Rotate", lo=[30.0], hi=[30.0], **C.WARP)],
    "ShiftScaleRotate": [C.op("ShiftScaleRotate", lo=C.SSR_LO, hi=C.SSR_HI, **C.WARP)],
    "RandomCrop64": [C.op("RandomCrop", size=(64, 64))],
    "Crop": [C.op("Crop", origin=(40, 30), size=(250, 200))],
    "VFlip_Pad_Crop": [C.op("VerticalFlip", p=0.5), C.op("PadToSize", size=(520, 400)),
                       C.op("RandomCrop", size=(300, 300))],
}


@pytest.mark.parametrize("name", list(BOX_OPS))
@pytest.mark.parametrize("min_vis", [0.0, 0.3])
def test_boxes_image_mask_through_op(name, min_vis):
    """SPEC.md:179, 187 (flips), 232/241 (crops), 250 (pad), 259 (resize),
    268 (RSC), 214 (rotate), 220-224 (SSR): boxes clipped once at the end and
    kept iff clipped area >= min_visibility * unclipped area (R19)."""
    specs = BOX_OPS[name]
    sizes = gen.cfg2_sizes(20, first_image_index=700)
    exact = all(s["kind"] in ("HorizontalFlip", "VerticalFlip", "PadToSize", "RandomCrop", "Crop")
                for s in specs)
    resize = len(specs) == 1 and specs[0]["kind"] == "Resize"
    _run_all(specs, sizes, 700, 31, min_vis, "resize" if resize else cmp_exact if exact else cmp_interp)


# ---------------------------------------------------------------- Normalize

@pytest.mark.parametrize("sizes", [[(224, 224)] * 8, [(37, 61)] * 3, [(1, 1)] * 2,
                                   [(375, 500)] * 4])
def test_normalize_only_bit_equal_and_relative(sizes):
    """Normalize alone on identical u8 input: fp32 NCHW equal to the oracle's
    (float)((v/255 - mean)/std) bit for bit, hence within 1e-6 relative
    (BASELINE.json north_star); every value of the 3x256 table is exercised
    by the gradient+noise inputs."""
    specs = [C.op("Normalize", mean=MEAN, std=STD)]
    b = gen.gen_images(sizes, seed=4, first_image_index=0, device="cuda")
    g = run_gpu(specs, b, seed=0)["nchw"]
    r = np.stack([o["nchw"] for o in run_oracle(specs, [b.image(i) for i in range(len(sizes))])])
    assert g.shape == r.shape == (len(sizes), 3) + sizes[0]
    assert np.array_equal(g, r)
    rel = np.abs(g.astype(np.float64) - r) / np.maximum(np.abs(r.astype(np.float64)), 1e-30)
    assert rel.max() <= 1e-6


def test_normalize_table_every_value_closed_form():
    """A 1 x 256 ramp image holds every u8 value in every channel: the GPU's
    Normalize output equals the closed form (v/255 - m)/s rounded once to
    fp32, computed here with Python fractions (no oracle involved)."""
    from fractions import Fraction
    ramp = np.stack([np.arange(256, dtype=np.uint8)] * 3, 1)[None]  # (1, 256, 3)
    from tests.harness import to_device_batch
    b = to_device_batch([ramp])
    g = run_gpu([C.op("Normalize", mean=MEAN, std=STD)], b)["nchw"][0]
    for c in range(3):
        m, s = Fraction(MEAN[c]), Fraction(STD[c])
        want = np.array([float((Fraction(v, 255) - m) / s) for v in range(256)], np.float32)
        assert np.array_equal(g[c, 0], want), c


# ---------------------------- fused resample stage programs (quad-column kernel)

STAGE_PROGRAMS = {
    "lut": [C.op("Brightness", lo=[0.8], hi=[1.2])],
    "hsv": [C.op("ShiftHSV", lo=[-20.0, -0.1, -0.1], hi=[20.0, 0.1, 0.1])],
    "gray": [C.op("Grayscale", p=0.5)],
    "hsv_lut": [C.op("ShiftHSV", lo=[-20.0, -0.1, -0.1], hi=[20.0, 0.1, 0.1]),
                C.op("BrightnessContrast", lo=[0.8, 0.8], hi=[1.2, 1.2])],
    "lut_hsv": [C.op("Gamma", lo=[0.8], hi=[1.2]),
                C.op("ShiftHSV", lo=[-20.0, -0.1, -0.1], hi=[20.0, 0.1, 0.1], p=0.7)],
}


@pytest.mark.parametrize("norm", [False, True])
@pytest.mark.parametrize("prog", list(STAGE_PROGRAMS))
def test_resample_stage_programs_fused_equals_unfused(prog, norm):
    """A resize followed by a pointwise program (and Normalize) runs as ONE
    kernel; it must equal the chain of single-op GPU applies with the drawn
    parameters fixed, bit for bit (reading R21 (i)), and the oracle at >= 99.9%
    exact (R21 (iii))."""
    from paper_1809_06839_b200 import Pipeline
    rs = C.op("Resize", size=(256, 192), interp="bilinear")
    tail = [C.op("Normalize", mean=MEAN, std=STD)] if norm else []
    specs = [rs] + STAGE_PROGRAMS[prog] + tail
    sizes = gen.cfg2_sizes(6, first_image_index=900)
    b = gen.gen_images(sizes, seed=0, first_image_index=900, device="cuda")
    fused = run_gpu(specs, b, seed=41, first=900)
    prm, fired = Pipeline(specs).sample_params(41, 900, sizes)
    imgs = [b.image(i) for i in range(len(sizes))]
    from tests.harness import to_device_batch
    for i in range(len(sizes)):
        x = run_gpu([rs], to_device_batch([imgs[i]]))["out_batch"]
        for k, o in enumerate(STAGE_PROGRAMS[prog], start=1):
            if not fired[i, k]:
                continue
            q = [float(v) for v in prm[i, k, :3]]
            fixed = dict(o, p=1.0, lo=q[:len(o.get("lo", []))], hi=q[:len(o.get("lo", []))])
            x = run_gpu([fixed], x)["out_batch"]
        if norm:
            got = run_gpu(tail, x)["nchw"][0]
            assert np.array_equal(got, fused["nchw"][i]), i
        else:
            assert np.array_equal(x.image(0), fused["images"][i]), i
    ref = run_oracle(specs, imgs, seed=41, first=900)
    if norm:
        g = fused["nchw"]
        r = np.stack([o["nchw"] for o in ref])
        assert (g == r).mean() >= 0.999
    else:
        cmp_interp(fused["images"], [o["image"] for o in ref], max_abs=8 if "hsv" in prog else 1)


# ----------------------------------------- CUDA-graph capture with side streams

@pytest.mark.parametrize("cfg", ["cfg3", "cfg5"])
def test_masked_boxed_apply_captures_into_cuda_graph(cfg):
    """alb_apply forks label / box work onto the plan's side stream and joins
    it back; captured into a CUDA graph (fork / join become graph edges) and
    replayed, images, masks and boxes equal the eager results."""
    from paper_1809_06839_b200 import Layout, Pipeline, Plan
    from tests.harness import out_batch
    specs = C.CFG3_OPS["ShiftScaleRotate"] if cfg == "cfg3" else C.CFG5_OPS
    sizes = [(512, 512)] * 4 if cfg == "cfg3" else [(1024, 1024)] * 3
    b, bx, lb, cnt, masks = _targets(sizes, 60)
    pipe = Pipeline(specs)
    osz = [pipe.output_shape(h, w) for h, w in sizes]
    ob, mo = out_batch(osz, 3), out_batch(osz, 1)
    nb = bx.shape[1] if cfg == "cfg5" else 0
    plan = Plan(pipe, Layout(b.desc, 3), Layout(ob.desc, 3), Layout(masks.desc, 1), Layout(mo.desc, 1), nb,
                C.CFG5_MIN_VISIBILITY)
    ws = plan.workspace()
    bi = [torch.from_numpy(t).cuda() for t in (bx, lb, cnt)] if nb else [None] * 3
    bo = [torch.full_like(t, -1) for t in bi] if nb else [None] * 3

    def go(stream=None):
        plan.apply(9, 60, b.buf, ob.buf, None, masks.buf, mo.buf, bi[0], bi[1], bi[2], bo[0], bo[1], bo[2],
                   workspace=ws, stream=stream)

    go()
    torch.cuda.synchronize()
    want = [ob.buf.clone(), mo.buf.clone()] + ([t.clone() for t in bo] if nb else [])
    ob.buf.fill_(0xAB)
    mo.buf.fill_(0xAB)
    for t in (bo if nb else []):
        t.fill_(-1)
    s = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        go(stream=s)
    g.replay()
    torch.cuda.synchronize()
    got = [ob.buf, mo.buf] + (list(bo) if nb else [])
    for x, y in zip(got, want):
        assert torch.equal(x, y)


@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2, reason="needs two GPUs")
def test_plan_on_second_device_same_process():
    """Launch caches (dynamic shared-memory attribute, occupancy, SM count) are
    per device: a Rotate plan (large dynamic shared memory) on cuda:1 after one
    on cuda:0 in the same process runs and matches cuda:0 bit for bit."""
    from paper_1809_06839_b200 import Layout, Pipeline, Plan
    specs = C.CFG2_MENU["Rotate"]
    sizes = gen.cfg2_sizes(4)
    outs = []
    for dev in ("cuda:0", "cuda:1"):
        with torch.cuda.device(dev):
            b = gen.gen_images(sizes, seed=0, device=dev)
            pipe = Pipeline(specs)
            from tests.harness import out_batch
            ob = out_batch([pipe.output_shape(h, w) for h, w in sizes], 3, device=dev)
            plan = Plan(pipe, Layout(b.desc, 3), Layout(ob.desc, 3))
            plan.apply(3, 0, b.buf, ob.buf, workspace=plan.workspace(dev))
            torch.cuda.synchronize(dev)
            outs.append(ob.buf.cpu())
    assert torch.equal(outs[0], outs[1])
