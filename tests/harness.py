"""Shared test helpers: run a pipeline through the C ABI on the GPU and through
the oracle on the CPU, and compare at the DESIGN.md tolerances."""
from __future__ import annotations

import numpy as np
import torch

from synth import gen


def to_device_batch(images, channels=3, pitch_pad=0, align=256, shift=0, device="cuda"):
    """Pack numpy images into one flat device buffer.  shift moves every image
    by `shift` bytes (to test unaligned offsets)."""
    sizes = [im.shape[:2] for im in images]
    desc, total = gen.layout(sizes, channels, align, pitch_pad)
    desc[:, 0] += shift
    buf = torch.zeros(total + shift + 64, dtype=torch.uint8)
    for i, im in enumerate(images):
        off, h, w, pitch = [int(v) for v in desc[i]]
        v = buf[off:off + h * pitch].view(h, pitch)
        v[:, :w * channels] = torch.from_numpy(np.ascontiguousarray(im).reshape(h, w * channels))
    return gen.Batch(buf.to(device), desc, channels)


def out_batch(sizes, channels=3, device="cuda", align=256, pitch_pad=0, shift=0, fill=0xAB):
    desc, total = gen.layout(sizes, channels, align, pitch_pad)
    desc[:, 0] += shift
    buf = torch.full((total + shift + 64,), fill, dtype=torch.uint8, device=device)
    return gen.Batch(buf, desc, channels)


def run_gpu(specs, batch, seed=0, first=0, masks=None, boxes=None, labels=None, count=None,
            max_boxes=0, min_visibility=0.0, out_pitch_pad=0, out_shift=0, return_plan=False):
    from paper_1809_06839_b200 import Layout, Pipeline, Plan
    pipe = Pipeline(specs)
    n = batch.n
    in_l = Layout(batch.desc, 3)
    sizes = [pipe.output_shape(int(h), int(w)) for _, h, w, _ in batch.desc]
    ends_norm = len(specs) > 0 and specs[-1]["kind"] == "Normalize"
    out = out_l = nchw = None
    if ends_norm:
        oh, ow = sizes[0]
        nchw = torch.full((n, 3, oh, ow), float("nan"), dtype=torch.float32, device="cuda")
    else:
        out = out_batch(sizes, 3, pitch_pad=out_pitch_pad, shift=out_shift)
        out_l = Layout(out.desc, 3)
    mi_l = mo_l = mout = None
    if masks is not None:
        mi_l = Layout(masks.desc, 1)
        mout = out_batch(sizes, 1)
        mo_l = Layout(mout.desc, 1)
    bo = lo = co = bi = li = ci = None
    if max_boxes:
        bi = torch.from_numpy(boxes).cuda()
        li = torch.from_numpy(labels).cuda()
        ci = torch.from_numpy(count).cuda()
        bo = torch.full_like(bi, -1.0)
        lo = torch.full_like(li, -1)
        co = torch.full_like(ci, -1)
    plan = Plan(pipe, in_l, out_l, mi_l, mo_l, max_boxes, min_visibility)
    plan.apply(seed, first, batch.buf, None if out is None else out.buf, nchw,
               None if masks is None else masks.buf, None if mout is None else mout.buf,
               bi, li, ci, bo, lo, co)
    torch.cuda.synchronize()
    res = {"images": None if out is None else [out.image(i) for i in range(n)],
           "nchw": None if nchw is None else nchw.cpu().numpy(),
           "masks": None if mout is None else [mout.image(i) for i in range(n)],
           "out_batch": out, "mask_batch": mout}
    if max_boxes:
        res["boxes"] = bo.cpu().numpy()
        res["labels"] = lo.cpu().numpy()
        res["count"] = co.cpu().numpy()
    if return_plan:
        res["plan"] = plan
    return res


def run_oracle(specs, images, seed=0, first=0, masks=None, boxes=None, labels=None, count=None,
               min_visibility=0.0, threads=8):
    from oracle import albref as A
    bl = None if boxes is None else [boxes[i, :count[i]] for i in range(len(images))]
    ll = None if labels is None else [labels[i, :count[i]] for i in range(len(images))]
    return A.apply_batch(specs, seed, first, images, masks, bl, ll, min_visibility, threads)


def cmp_interp(gpu, ref, min_exact=0.999, max_abs=1):
    """Interpolating/HSV tolerance: max |d| <= 1 and >= 99.9% exact (per batch)."""
    tot = eq = 0
    worst = 0
    for g, r in zip(gpu, ref):
        assert g.shape == r.shape, (g.shape, r.shape)
        d = np.abs(g.astype(np.int32) - r.astype(np.int32))
        worst = max(worst, int(d.max()) if d.size else 0)
        tot += d.size
        eq += int((d == 0).sum())
    frac = eq / max(1, tot)
    assert worst <= max_abs, "max abs diff %d > %d" % (worst, max_abs)
    assert frac >= min_exact, "exact fraction %.6f < %.4f" % (frac, min_exact)
    return frac, worst


def cmp_exact(gpu, ref):
    for i, (g, r) in enumerate(zip(gpu, ref)):
        assert g.shape == r.shape, (i, g.shape, r.shape)
        if not np.array_equal(g, r):
            bad = np.argwhere(g != r)
            raise AssertionError("image %d differs at %d positions, first %s: gpu %s ref %s" % (
                i, len(bad), bad[0].tolist(), g[tuple(bad[0])], r[tuple(bad[0])]))


def run_oracle_cand(specs, images, seed=0, first=0, masks=None, threads=8):
    """Oracle outputs plus nearest-tie candidate sets (albref_apply_cand)."""
    from oracle import albref as A
    return A.apply_batch_cand(specs, seed, first, images, masks, threads)


def cmp_cand(gpu, ref, which="mask", min_exact=0.999):
    """Nearest-sample tolerance (SURVEY.md §8(c) "Mask nearest", R20): every
    pixel equals the oracle's, except where the oracle flagged a source
    coordinate within 1e-4 px of a .5 tie -- there the GPU value must be one
    of the oracle's candidate values (either neighbour) -- and >= min_exact
    of the pixels are exact.  `which` is "mask" or "image"."""
    tot = eq = 0
    for i, (g, o) in enumerate(zip(gpu, ref)):
        r, cv, cn = o[which], o[which + "_cand"], o[which + "_cand_n"]
        assert g.shape == r.shape, (i, g.shape, r.shape)
        g3 = g.reshape(g.shape[0], g.shape[1], -1)
        r3 = r.reshape(g3.shape)
        cv = cv.reshape(g3.shape[0], g3.shape[1], cv.shape[2], -1)
        diff = (g3 != r3).any(-1)
        tot += diff.size
        eq += int((~diff).sum())
        for y, x in np.argwhere(diff):
            n = int(cn[y, x])
            ok = n == 0 or any(np.array_equal(cv[y, x, k], g3[y, x]) for k in range(n))
            assert ok, ("image %d (%d,%d): gpu %s, oracle %s, outside the tie band (candidates %s)"
                        % (i, y, x, g3[y, x].tolist(), r3[y, x].tolist(),
                           cv[y, x, :n].tolist()))
    frac = eq / max(1, tot)
    assert frac >= min_exact, "exact fraction %.6f < %.4f" % (frac, min_exact)
    return frac


def random_masks(sizes, seed=0, device="cuda", levels=256):
    """Label planes of independent random labels per pixel: every neighbour
    differs, so any wrong nearest decision shows up as a wrong label."""
    rng = np.random.default_rng(seed)
    ims = [rng.integers(0, levels, size=(h, w), dtype=np.uint8) for h, w in sizes]
    return to_device_batch([m[:, :, None] for m in ims], channels=1, device=device), ims


def cmp_boxes(res, ref, tol=1e-5):
    """Box co-transform: same keep set and labels, coordinates within tol."""
    for i in range(len(ref)):
        k = int(res["count"][i])
        assert k == len(ref[i]["labels"]), (i, k, len(ref[i]["labels"]))
        assert np.array_equal(res["labels"][i, :k], ref[i]["labels"]), i
        assert np.abs(res["boxes"][i, :k] - ref[i]["boxes"]).max(initial=0) <= tol, i


def resize_exact_ties(img, nh, nw):
    """Per output element of a bilinear Resize of `img` (h, w, c) to nh x nw
    (R9), True where the exact rational blend value is k + 1/2:
    x_s = ((2d+1) W - nw) / (2 nw), so the value is N / (4 nw nh) with integer
    N (integer arithmetic, no floating point).  At these ties round-half-up
    is decided by each implementation's rounding of its inexact weights
    (reading R33), so either neighbour is a correct result."""
    img = img.astype(np.int64)
    H, W = img.shape[:2]

    def icoord(n_src, n_dst):
        d = np.arange(n_dst)
        num = (2 * d + 1) * n_src - n_dst
        x0 = np.where(num <= 0, 0, num // (2 * n_dst))
        wgt = np.where(num <= 0, 0, num % (2 * n_dst))
        cl = x0 >= n_src - 1
        return np.where(cl, n_src - 1, x0), np.where(cl, 0, wgt)

    y0, wy = icoord(H, nh)
    x0, wx = icoord(W, nw)
    y1, x1 = np.minimum(y0 + 1, H - 1), np.minimum(x0 + 1, W - 1)
    D = 4 * nw * nh
    h0 = (2 * nw - wx)[None, :, None] * img[y0][:, x0] + wx[None, :, None] * img[y0][:, x1]
    h1 = (2 * nw - wx)[None, :, None] * img[y1][:, x0] + wx[None, :, None] * img[y1][:, x1]
    N = (2 * nh - wy)[:, None, None] * h0 + wy[:, None, None] * h1
    return (2 * N) % (2 * D) == D


def cmp_resize(gpu, ref, inputs, min_exact=0.999):
    """Resize tolerance: max |d| <= 1 and >= min_exact exact, OR (structured
    ratios, R33) every difference sits on an exact .5 tie of the blend."""
    try:
        return cmp_interp(gpu, ref, min_exact)
    except AssertionError:
        for g, r, im in zip(gpu, ref, inputs):
            d = g.astype(np.int32) - r.astype(np.int32)
            assert np.abs(d).max(initial=0) <= 1
            tie = resize_exact_ties(im, g.shape[0], g.shape[1])
            assert not ((d != 0) & ~tie).any(), int(((d != 0) & ~tie).sum())
        return None
