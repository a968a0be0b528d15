"""Pins of the CPU oracle against things other than itself (CPU only).

Each test pins one oracle function to a value the paper/SPEC prints, a closed
form, an invariant, brute force, or an independent library routine (cv2,
numpy, colorsys, fractions, CUDA's own curand Philox).  Citations: PAPER.md /
SPEC.md lines and DESIGN.md readings.
"""
import colorsys
import json
import os
import shutil
import subprocess
import tempfile
from fractions import Fraction

import cv2
import numpy as np
import pytest

from oracle import albref as A

GOLD = os.path.join(os.path.dirname(__file__), "golden")
RNG = np.random.default_rng(1234)


def rand_img(h, w, c=3, rng=RNG):
    return rng.integers(0, 256, size=(h, w, c), dtype=np.uint8)


def run(ops, img, seed=0, idx=0, **kw):
    return A.apply(ops, seed, idx, img, **kw)


# ------------------------------------------------------------------ O1 RNG

def test_philox_kat():
    """Random123 known-answer vectors (tests/golden/philox_kat.txt)."""
    n = 0
    for line in open(os.path.join(GOLD, "philox_kat.txt")):
        if line.startswith("#") or not line.strip():
            continue
        lhs, rhs = line.split(":")
        v = [int(t, 16) for t in lhs.split()]
        want = [int(t, 16) for t in rhs.split()]
        assert A.philox(v[:4], v[4:6]) == want
        n += 1
    assert n == 3


@pytest.mark.skipif(shutil.which("nvcc") is None, reason="nvcc not available")
def test_philox_matches_curand_host():
    """Vendor pin: CUDA's curand_Philox4x32_10 (curand_philox4x32_x.h, compiled
    for the host) agrees with the oracle on 2000 random (ctr, key) pairs."""
    src = r"""
#define QUALIFIERS static inline __host__ __device__
#include <curand_philox4x32_x.h>
#include <cstdio>
int main() {
  unsigned c0, c1, c2, c3, k0, k1;
  while (scanf("%u %u %u %u %u %u", &c0, &c1, &c2, &c3, &k0, &k1) == 6) {
    uint4 c = make_uint4(c0, c1, c2, c3); uint2 k = make_uint2(k0, k1);
    uint4 o = curand_Philox4x32_10(c, k);
    printf("%u %u %u %u\n", o.x, o.y, o.z, o.w);
  }
  return 0;
}
"""
    d = tempfile.mkdtemp()
    try:
        with open(os.path.join(d, "p.cu"), "w") as f:
            f.write(src)
        exe = os.path.join(d, "p")
        subprocess.check_call(["nvcc", "-o", exe, os.path.join(d, "p.cu")],
                              stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)
        rng = np.random.default_rng(7)
        vals = rng.integers(0, 2**32, size=(2000, 6), dtype=np.uint64)
        inp = "\n".join(" ".join(str(int(x)) for x in row) for row in vals) + "\n"
        out = subprocess.run([exe], input=inp, capture_output=True, text=True, check=True).stdout
        rows = [list(map(int, l.split())) for l in out.strip().split("\n")]
        for row, got in zip(vals, rows):
            assert A.philox(row[:4], row[4:6]) == got
    finally:
        shutil.rmtree(d)


def test_u53_range_and_extremes():
    assert A.u53(0, 0) == 0.0
    assert A.u53(0xFFFFFFFF, 0xFFFFFFFF) == 1.0 - 2.0 ** -53
    # the low 5 / 6 bits are discarded; one step of b>>6 is exactly 2^-53
    assert A.u53(0, 64) == 2.0 ** -53
    assert A.u53(32, 0) == 2.0 ** -27


def test_gate_rate_statistical():
    """a p=0.5 transform fires 5000 +- 200 times over 10 000 seeds."""
    ops = [{"kind": "HorizontalFlip", "p": 0.5}]
    fired = sum(int(A.sample_params(ops, s, 0, 4, 4)[1][0]) for s in range(10000))
    assert 4800 <= fired <= 5200


def test_draws_uniform_chisq():
    """u53 draws are uniform: chi-square over 20 bins, 20000 draws."""
    u = np.array([A.draw(3, i, 0, 1) for i in range(20000)])
    assert u.min() >= 0 and u.max() < 1
    cnt = np.histogram(u, bins=20, range=(0, 1))[0]
    chi2 = ((cnt - 1000.0) ** 2 / 1000.0).sum()
    assert chi2 < 50  # 19 dof, p ~ 1e-4


def test_random_crop_coverage():
    """over 10 000 seeds an 8x8 -> 4x4 crop hits every x0 in 0..4."""
    ops = [{"kind": "RandomCrop", "size": (4, 4)}]
    xs, ys = set(), set()
    for s in range(10000):
        prm, _ = A.sample_params(ops, s, 0, 8, 8)
        xs.add(int(prm[0][0]))
        ys.add(int(prm[0][1]))
    assert xs == set(range(5)) and ys == set(range(5))


def test_param_ranges_and_gate_stability():
    """Params stay in [lo,hi]; changing params of a slot never changes the gates
    (SPEC.md:503), because the gate is always draw 0 of its own slot."""
    a = [{"kind": "Brightness", "p": 0.5, "lo": [0.8], "hi": [1.2]},
         {"kind": "Rotate", "p": 0.3, "lo": [-90], "hi": [90]}]
    b = [{"kind": "Brightness", "p": 0.5, "lo": [0.1], "hi": [0.2]},
         {"kind": "Rotate", "p": 0.3, "lo": [0], "hi": [1]}]
    for i in range(300):
        pa, fa = A.sample_params(a, 11, i, 10, 10)
        pb, fb = A.sample_params(b, 11, i, 10, 10)
        assert (fa == fb).all()
        assert 0.8 <= pa[0][0] <= 1.2 and -90 <= pa[1][0] <= 90


# --------------------------------------------------------- golden examples

def test_spec_examples():
    n = 0
    for line in open(os.path.join(GOLD, "spec_examples.jsonl")):
        e = json.loads(line)
        fn = e["fn"]
        if fn == "clip_round":
            assert A.clip_round(e["in"]) == e["out"], e["cite"]
        elif fn == "reflect101":
            assert A.reflect101(*e["in"]) == e["out"], e["cite"]
        elif fn == "lut":
            lut = A.build_lut(e["kind"], e["params"])
            assert (lut[:, e["v"]] == e["out"]).all(), e["cite"]
        elif fn == "rgb_to_hsv":
            assert np.allclose(A.rgb_to_hsv(*e["in"]), e["out"], atol=1e-12), e["cite"]
        elif fn == "grayscale":
            img = np.array(e["in"], np.uint8).reshape(1, 1, 3)
            assert (run([{"kind": "Grayscale"}], img)["image"] == e["out"]).all(), e["cite"]
        elif fn == "box":
            h, w = e["hw"]
            r = run(e["ops"], rand_img(h, w), boxes=np.array([e["box"]], np.float32),
                    labels=np.array([3], np.int32))
            assert r["boxes"].shape == (1, 4) and r["labels"][0] == 3, e["cite"]
            assert np.allclose(r["boxes"][0], e["out"], atol=1e-6), e["cite"]
        else:
            raise AssertionError(fn)
        n += 1
    assert n >= 20


def test_reflect101_matches_cv2():
    """Reflect-101 equals cv2.borderInterpolate(BORDER_REFLECT_101)."""
    for n in [1, 2, 3, 5, 16]:
        for i in range(-40, 40):
            assert A.reflect101(i, n) == cv2.borderInterpolate(i, n, cv2.BORDER_REFLECT_101)


# ------------------------------------------------------------------ O2 flips

def test_flips_vs_numpy_and_involution():
    img = rand_img(7, 9)
    m = RNG.integers(0, 5, size=(7, 9), dtype=np.uint8)
    h = run([{"kind": "HorizontalFlip"}], img, mask=m)
    v = run([{"kind": "VerticalFlip"}], img, mask=m)
    assert (h["image"] == img[:, ::-1]).all() and (h["mask"] == m[:, ::-1]).all()
    assert (v["image"] == img[::-1]).all() and (v["mask"] == m[::-1]).all()
    assert (h["image"] == cv2.flip(img, 1)).all() and (v["image"] == cv2.flip(img, 0)).all()
    for k in ["HorizontalFlip", "VerticalFlip"]:
        assert (run([{"kind": k}, {"kind": k}], img)["image"] == img).all()
    ab = np.array([[[1, 1, 1], [2, 2, 2]]], np.uint8)
    assert (run([{"kind": "HorizontalFlip"}], ab)["image"] == ab[:, ::-1]).all()


# ------------------------------------------------------------- O7 affine

def _ramp(h, w):
    y, x = np.mgrid[0:h, 0:w]
    return np.stack([x, y, x * y], 2).astype(np.uint8)


def _cv2_inverse(h, w, dx, dy, s, theta):
    M = cv2.getRotationMatrix2D(((w - 1) / 2.0, (h - 1) / 2.0), theta, s)
    M[0, 2] += dx * w
    M[1, 2] += dy * h
    return cv2.invertAffineTransform(M)


@pytest.mark.parametrize("dx,dy,s,theta", [(0, 0, 1, 30.0), (0.06, -0.04, 1.07, -17.0),
                                            (-0.05, 0.03, 0.91, 71.5), (0, 0, 1, -90.0)])
def test_affine_ramp_closed_form_vs_cv2_matrix(dx, dy, s, theta):
    """On a ramp image (ch0 = x, ch1 = y, ch2 = x*y) bilinear sampling reproduces
    the source coordinate exactly, so interior outputs must equal
    round_half_up of the source coordinates that cv2.getRotationMatrix2D +
    invertAffineTransform give (pins centre, direction, scale/shift composition
    and the bilinear weights)."""
    h, w = 15, 16
    img = _ramp(h, w)
    ops = [{"kind": "ShiftScaleRotate", "lo": [dx, dy, s, theta], "hi": [dx, dy, s, theta],
            "interp": "bilinear", "border": "constant"}]
    out = run(ops, img)["image"].astype(np.int64)
    Mi = _cv2_inverse(h, w, dx, dy, s, theta)
    checked = 0
    for y in range(h):
        for x in range(w):
            xs = Mi[0, 0] * x + Mi[0, 1] * y + Mi[0, 2]
            ys = Mi[1, 0] * x + Mi[1, 1] * y + Mi[1, 2]
            if not (0 <= xs <= w - 1.001 and 0 <= ys <= h - 1.001):
                continue
            vals = [xs, ys, xs * ys]
            for c in range(3):
                if abs((vals[c] % 1.0) - 0.5) < 1e-6:
                    continue
                assert out[y, x, c] == int(np.floor(vals[c] + 0.5)), (x, y, c)
            checked += 1
    assert checked > 50


def test_rotate_identities():
    img = rand_img(9, 11)
    for interp in ["nearest", "bilinear"]:
        for border in ["constant", "reflect_101"]:
            r = run([{"kind": "Rotate", "lo": [0], "hi": [0], "interp": interp,
                      "border": border}], img)
            assert (r["image"] == img).all()
            s = run([{"kind": "ShiftScaleRotate", "lo": [0, 0, 1, 0], "hi": [0, 0, 1, 0],
                      "interp": interp, "border": border}], img)
            assert (s["image"] == img).all()


@pytest.mark.parametrize("interp", ["nearest", "bilinear"])
def test_rotate90_equals_rot90(interp):
    """Rotate(90) nearest on a square = rot90 k=1 (np.rot90 is CCW,
    out[y][x] = in[x][W-1-y])."""
    for n in [1, 4, 7, 16]:
        img = rand_img(n, n)
        m = RNG.integers(0, 9, size=(n, n), dtype=np.uint8)
        r = run([{"kind": "Rotate", "lo": [90], "hi": [90], "interp": interp}], img, mask=m)
        assert (r["image"] == np.rot90(img)).all()
        assert (r["mask"] == np.rot90(m)).all()
        r = run([{"kind": "Rotate", "lo": [180], "hi": [180], "interp": interp}], img)
        assert (r["image"] == img[::-1, ::-1]).all()


def test_rotate_centre_fixed_and_ssr_reduces_to_rotate():
    img = rand_img(9, 13)
    for t in [13.0, 47.0, -66.0]:
        r = run([{"kind": "Rotate", "lo": [t], "hi": [t], "interp": "nearest"}], img)
        assert (r["image"][4, 6] == img[4, 6]).all()
    for t in [0.0, 30.0, 90.0]:
        a = run([{"kind": "Rotate", "lo": [t], "hi": [t]}], img)["image"]
        b = run([{"kind": "ShiftScaleRotate", "lo": [0, 0, 1, t], "hi": [0, 0, 1, t]}], img)["image"]
        assert (a == b).all()


def test_ssr_integer_shift_constant_and_reflect():
    """dx=0.25 on a 4-wide image shifts by one column; col 0 = fill.
    With reflect_101 col 0 reads x=-1 -> 1."""
    img = rand_img(3, 4)
    ops = {"kind": "ShiftScaleRotate", "lo": [0.25, 0, 1, 0], "hi": [0.25, 0, 1, 0],
           "fill": (9, 8, 7)}
    a = run([dict(ops, border="constant")], img)["image"]
    assert (a[:, 1:] == img[:, :3]).all() and (a[:, 0] == [9, 8, 7]).all()
    b = run([dict(ops, border="reflect_101")], img)["image"]
    assert (b[:, 1:] == img[:, :3]).all() and (b[:, 0] == img[:, 1]).all()


def test_mask_equals_channel0_under_nearest():
    """an image whose channel 0 equals its mask stays equal under
    every geometric op with nearest interpolation."""
    for i in range(10):
        img = rand_img(12, 10)
        m = img[:, :, 0].copy()
        for ops in [[{"kind": "ShiftScaleRotate", "lo": [-.1, -.1, .8, -90], "hi": [.1, .1, 1.2, 90],
                      "interp": "nearest", "border": b}] for b in ["constant", "reflect_101"]] + \
                   [[{"kind": "Resize", "size": (7, 15), "interp": "nearest"}],
                    [{"kind": "RandomSizedCrop", "side": (3, 9), "size": (5, 6), "interp": "nearest"}],
                    [{"kind": "RandomCrop", "size": (4, 5)}, {"kind": "HorizontalFlip", "p": 0.5}],
                    [{"kind": "PadToSize", "size": (13, 16)}, {"kind": "VerticalFlip"}]]:
            r = run(ops, img, seed=i, mask=m)
            assert (r["image"][:, :, 0] == r["mask"]).all()


def test_rotate_roundtrip_bound():
    """rotate(t) then rotate(-t) bilinear stays within 2 levels on
    the interior 50% window (smooth content: resampling round trip)."""
    y, x = np.mgrid[0:64, 0:64]
    f = [128 + 100 * np.sin(x / 9.0) * np.cos(y / 11.0), 2.0 * x + y, 255 - 3.0 * y]
    img = np.stack([np.floor(t + 0.5) for t in f], 2).astype(np.uint8)
    for t in [10.0, 33.0, -45.0]:
        a = run([{"kind": "Rotate", "lo": [t], "hi": [t], "border": "reflect_101"}], img)["image"]
        b = run([{"kind": "Rotate", "lo": [-t], "hi": [-t], "border": "reflect_101"}], a)["image"]
        d = np.abs(b.astype(int) - img.astype(int))[16:48, 16:48]
        assert d.max() <= 2


# ----------------------------------------------------------- O3/O4 window

def test_crop_pad_pins():
    img = rand_img(6, 8)
    assert (run([{"kind": "Crop", "origin": (0, 0), "size": (8, 6)}], img)["image"] == img).all()
    ab = np.array([[[1, 2, 3], [4, 5, 6]]], np.uint8)
    assert (run([{"kind": "Crop", "origin": (1, 0), "size": (1, 1)}], ab)["image"] == ab[:, 1:]).all()
    r = run([{"kind": "Crop", "origin": (2, 1), "size": (5, 3)}], img)["image"]
    assert (r == img[1:4, 2:7]).all()
    v = np.array([[[200, 100, 50]]], np.uint8)
    p = run([{"kind": "PadToSize", "size": (3, 3)}], v)["image"]
    assert (p[1, 1] == v[0, 0]).all() and p.sum() == v.sum()
    for (h, w, th, tw) in [(6, 8, 9, 13), (5, 5, 5, 6), (1, 2, 4, 4)]:
        img = rand_img(h, w)
        p = run([{"kind": "PadToSize", "size": (tw, th), "fill": (1, 2, 3)}], img)["image"]
        top, left = (th - h) // 2, (tw - w) // 2
        ref = np.stack([np.pad(img[:, :, c], ((top, th - h - top), (left, tw - w - left)),
                               constant_values=c + 1) for c in range(3)], 2)
        assert (p == ref).all()
        ref2 = cv2.copyMakeBorder(img, top, th - h - top, left, tw - w - left,
                                  cv2.BORDER_CONSTANT, value=(1, 2, 3))
        assert (p == ref2).all()


def test_random_crop_is_window_of_params():
    img = rand_img(20, 30)
    ops = [{"kind": "RandomCrop", "size": (7, 5)}]
    for i in range(20):
        prm, _ = A.sample_params(ops, 1, i, 20, 30)
        x0, y0 = int(prm[0][0]), int(prm[0][1])
        assert (A.apply(ops, 1, i, img)["image"] == img[y0:y0 + 5, x0:x0 + 7]).all()
    assert (run([{"kind": "RandomCrop", "size": (30, 20)}], img)["image"] == img).all()


def test_min_visibility_filter():
    """R19: clipped area / unclipped area >= min_visibility."""
    img = rand_img(100, 100)
    ops = [{"kind": "Crop", "origin": (40, 40), "size": (50, 50)}]
    bx = np.array([[0.0, 0.0, 0.5, 0.5], [0.4, 0.4, 0.6, 0.6], [0.95, 0.95, 1.0, 1.0]], np.float32)
    r0 = run(ops, img, boxes=bx, labels=np.array([1, 2, 3], np.int32))
    assert list(r0["labels"]) == [1, 2]  # third box lies outside the window
    assert np.allclose(r0["boxes"][0], [0, 0, 0.2, 0.2], atol=1e-6)
    r1 = run(ops, img, boxes=bx, labels=np.array([1, 2, 3], np.int32), min_visibility=0.3)
    assert list(r1["labels"]) == [2]  # box 1 visible 100/2500 = 0.04


# ------------------------------------------------------------- O5 resize

def test_resize_pins():
    img = rand_img(9, 12)
    for interp in ["nearest", "bilinear"]:
        r = run([{"kind": "Resize", "size": (12, 9), "interp": interp}], img)["image"]
        assert (r == img).all()  # SPEC.md:262 (x_s = x_d exactly)
    two = np.array([[[1, 1, 1], [2, 2, 2]], [[3, 3, 3], [4, 4, 4]]], np.uint8)
    r = run([{"kind": "Resize", "size": (1, 1), "interp": "nearest"}], two)["image"]
    assert (r[0, 0] == 4).all()  # x_s = 0.5 rounds to index 1


@pytest.mark.parametrize("hw,nhw", [((30, 40), (64, 51)), ((64, 64), (17, 23)),
                                    ((37, 50), (37, 80)), ((5, 3), (512 // 16, 7))])
def test_resize_vs_cv2_float(hw, nhw):
    """cv2.resize(INTER_LINEAR) on float32 input uses the same half-pixel,
    replicate-border bilinear; after round-half-up the oracle must agree except
    where cv2's float value sits within 1e-3 of a .5 tie."""
    h, w = hw
    nh, nw = nhw
    img = rand_img(h, w)
    r = run([{"kind": "Resize", "size": (nw, nh), "interp": "bilinear"}], img)["image"]
    f = cv2.resize(img.astype(np.float32), (nw, nh), interpolation=cv2.INTER_LINEAR)
    ref = np.floor(f.astype(np.float64) + 0.5)
    tie = np.abs((f % 1.0) - 0.5) < 1e-3
    assert ((r == ref) | tie).all()


def test_rsc_reduces_to_resize_and_crop():
    img = rand_img(40, 40)
    a = run([{"kind": "RandomSizedCrop", "side": (40, 40), "size": (23, 23)}], img)["image"]
    b = run([{"kind": "Resize", "size": (23, 23)}], img)["image"]
    assert (a == b).all()
    img = rand_img(30, 50)
    ops = [{"kind": "RandomSizedCrop", "side": (10, 400), "size": (10, 10)}]
    for i in range(30):
        prm, _ = A.sample_params(ops, 2, i, 30, 50)
        side, x0, y0 = [int(v) for v in prm[0][:3]]
        assert 10 <= side <= 30 and 0 <= x0 <= 50 - side and 0 <= y0 <= 30 - side
        out = A.apply(ops, 2, i, img)["image"]
        assert out.shape == (10, 10, 3)
        if side == 10:
            assert (out == img[y0:y0 + 10, x0:x0 + 10]).all()


# --------------------------------------------------------------- O8 LUTs

def test_lut_closed_forms():
    v = np.arange(256)
    assert (A.build_lut("Gamma", [2.0])[0] == (2 * v * v + 255) // 510).all()
    assert (A.build_lut("Brightness", [0.5])[0] == (v + 1) // 2).all()
    assert (A.build_lut("Brightness", [1.5])[0] == np.minimum((3 * v + 1) // 2, 255)).all()
    assert (A.build_lut("Contrast", [2.0])[0] == np.clip(2 * v - 127, 0, 255)).all()
    for k, p in [("Brightness", [1.0]), ("Contrast", [1.0]), ("Gamma", [1.0]),
                 ("ShiftRGB", [0, 0, 0]), ("BrightnessContrast", [1.0, 1.0])]:
        assert (A.build_lut(k, p) == v).all()
    s = A.build_lut("ShiftRGB", [5.0, -3.0, 0.5])  # per-channel deltas
    assert (s[0] == np.minimum(v + 5, 255)).all() and (s[1] == np.maximum(v - 3, 0)).all()
    assert (s[2] == np.minimum(v + 1, 255)).all()  # 0.5 rounds half up


def test_lut_monotone_and_bc_composition():
    rng = np.random.default_rng(3)
    for _ in range(200):
        b, c, g = rng.uniform(0.5, 1.5), rng.uniform(0.5, 1.5), rng.uniform(0.5, 2.0)
        for k, p in [("Brightness", [b]), ("Contrast", [c]), ("Gamma", [g])]:
            assert (np.diff(A.build_lut(k, p)[0].astype(int)) >= 0).all()
        bc = A.build_lut("BrightnessContrast", [b, c])[0]
        comp = A.build_lut("Contrast", [c])[0][A.build_lut("Brightness", [b])[0]]
        assert (bc == comp).all()  # R12


def test_gamma_lut_vs_fraction_free_direct():
    """Gamma LUT equals direct per-pixel evaluation, checked in
    numpy float64 on all 256 inputs away from .5 ties."""
    for g in [0.8, 0.93, 1.17, 1.2]:
        lut = A.build_lut("Gamma", [g])[0]
        x = 255.0 * (np.arange(256) / 255.0) ** g
        tie = np.abs(x % 1.0 - 0.5) < 1e-9
        assert ((lut == np.floor(x + 0.5)) | tie).all()


# ---------------------------------------------------------------- O9 HSV

def test_hsv_vs_colorsys():
    rng = np.random.default_rng(9)
    for r, g, b in rng.integers(0, 256, size=(5000, 3)):
        h, s, v = A.rgb_to_hsv(r, g, b)
        ch, cs, cv = colorsys.rgb_to_hsv(r / 255.0, g / 255.0, b / 255.0)
        assert abs(h / 360.0 - ch) < 1e-12 or abs(abs(h / 360.0 - ch) - 1) < 1e-12
        assert abs(s - cs) < 1e-12 and abs(v - cv) < 1e-12
        rr, gg, bb = A.hsv_to_rgb(h, s, v)
        cr, cg, cb = colorsys.hsv_to_rgb(ch, cs, cv)
        assert max(abs(rr / 255 - cr), abs(gg / 255 - cg), abs(bb / 255 - cb)) < 1e-12


def test_shift_hsv_pins():
    rng = np.random.default_rng(10)
    img = rng.integers(0, 256, size=(200, 500, 3), dtype=np.uint8)
    zero = [{"kind": "ShiftHSV", "lo": [0, 0, 0], "hi": [0, 0, 0]}]
    assert (run(zero, img)["image"] == img).all()  # round trip exact
    red = np.array([[[255, 0, 0]]], np.uint8)
    g = run([{"kind": "ShiftHSV", "lo": [120, 0, 0], "hi": [120, 0, 0]}], red)["image"]
    assert (g == [0, 255, 0]).all()
    gray = np.repeat(rng.integers(0, 256, size=(50, 1, 1), dtype=np.uint8), 3, 2)
    for dh, ds in [(77, -0.2), (-150, 0.0)]:
        o = run([{"kind": "ShiftHSV", "lo": [dh, ds, 0], "hi": [dh, ds, 0]}], gray)["image"]
        assert (o == gray).all()
    # hue shift by 360 is the identity
    o = run([{"kind": "ShiftHSV", "lo": [360, 0, 0], "hi": [360, 0, 0]}], img)["image"]
    assert (o == img).all()


def test_shift_hsv_vs_colorsys_pipeline():
    """Independent route: colorsys + round-half-up on random pixels and shifts."""
    rng = np.random.default_rng(11)
    img = rng.integers(0, 256, size=(1, 400, 3), dtype=np.uint8)
    for dh, ds, dv in [(17.3, 0.05, -0.07), (-19.9, -0.1, 0.1)]:
        o = run([{"kind": "ShiftHSV", "lo": [dh, ds, dv], "hi": [dh, ds, dv]}], img)["image"]
        bad = 0
        for x in range(400):
            r, g, b = img[0, x] / 255.0
            h, s, v = colorsys.rgb_to_hsv(r, g, b)
            h = (h + dh / 360.0) % 1.0
            s = min(1.0, max(0.0, s + ds))
            v = min(1.0, max(0.0, v + dv))
            raw = [255 * t for t in colorsys.hsv_to_rgb(h, s, v)]
            for c in range(3):
                ref = int(np.floor(raw[c] + 0.5))
                if o[0, x, c] != ref:
                    # only where the value is a .5 tie up to rounding noise
                    assert abs(raw[c] % 1.0 - 0.5) < 1e-9
                    assert abs(int(o[0, x, c]) - ref) == 1
                    bad += 1
        assert bad <= 10


# ------------------------------------------------------------ O10 gray

def test_grayscale_exact_rational():
    rng = np.random.default_rng(12)
    px = rng.integers(0, 256, size=(1, 20000, 3), dtype=np.uint8)
    o = run([{"kind": "Grayscale"}], px)["image"]
    assert (o[:, :, 0] == o[:, :, 1]).all() and (o[:, :, 1] == o[:, :, 2]).all()
    for x in range(0, 20000, 7):
        r, g, b = [int(t) for t in px[0, x]]
        y = Fraction(299, 1000) * r + Fraction(587, 1000) * g + Fraction(114, 1000) * b
        want = int(y + Fraction(1, 2))  # floor(y + 1/2), y >= 0
        assert o[0, x, 0] == want
    gray = np.repeat(np.arange(256, dtype=np.uint8).reshape(1, 256, 1), 3, 2)
    assert (run([{"kind": "Grayscale"}], gray)["image"] == gray).all()
    assert (run([{"kind": "Grayscale"}] * 2, px)["image"] == o).all()
    cv = cv2.cvtColor(px, cv2.COLOR_RGB2GRAY)
    assert np.abs(cv.astype(int) - o[:, :, 0]).max() <= 1
    assert (cv == o[:, :, 0]).mean() > 0.995


# ---------------------------------------------------------- O11 equalize

def test_equalize_tiny_golden():
    n = 0
    for line in open(os.path.join(GOLD, "equalize_tiny.txt")):
        if line.startswith("#") or not line.strip():
            continue
        a, b = line.split(":")
        x = np.array([int(t) for t in a.split()], np.uint8)
        want = np.array([int(t) for t in b.split()], np.uint8)
        img = np.repeat(x.reshape(1, -1, 1), 3, 2)
        o = run([{"kind": "Equalize"}], img)["image"]
        assert (o[0, :, 0] == want).all(), line
        n += 1
    assert n == 6


def test_equalize_properties_and_cv2():
    from synth.gen import gen_images
    img = gen_images([(375, 500)], seed=0).image(0)
    o = run([{"kind": "Equalize"}], img)["image"]
    for c in range(3):
        hist = np.bincount(img[:, :, c].ravel(), minlength=256)
        lut = A.equalize_lut(hist)
        assert (np.diff(lut.astype(int)) >= 0).all()
        nz = np.nonzero(hist)[0]
        assert lut[nz[0]] == 0 and lut[nz[-1]] == 255
        assert (o[:, :, c] == lut[img[:, :, c]]).all()
        # near-uniform output CDF (BASELINE.json:5 invariant)
        cdf = np.cumsum(np.bincount(o[:, :, c].ravel(), minlength=256)) / o[:, :, c].size
        vals = np.unique(o[:, :, c])
        f0 = hist[nz[0]] / img[:, :, c].size  # mass of the lowest bin maps to 0
        dev = np.abs(cdf[vals] - (f0 + (1 - f0) * vals.astype(np.float64) / 255.0)).max()
        assert dev <= 0.5 / 255 + 1e-12
        # cv2.equalizeHist agrees except at exact .5 ties (Fraction-checked)
        cvl = cv2.equalizeHist(np.ascontiguousarray(img[:, :, c]))
        diff = np.nonzero(cvl.ravel() != o[:, :, c].ravel())[0]
        cdfc = np.cumsum(hist)
        D = img[:, :, c].size - hist[nz[0]]
        for v in np.unique(img[:, :, c].ravel()[diff]):
            fr = Fraction(255 * int(cdfc[v] - hist[nz[0]]), int(D))
            assert fr - int(fr) == Fraction(1, 2)
    k = np.repeat(np.arange(256, dtype=np.uint8), 3)  # every value k=3 times -> identity
    hist = np.bincount(k, minlength=256)
    assert (A.equalize_lut(hist) == np.arange(256)).all()
    two = np.array([[[3, 3, 3], [200, 200, 200], [3, 3, 3]]], np.uint8)
    assert set(np.unique(run([{"kind": "Equalize"}], two)["image"])) == {0, 255}


# --------------------------------------------------------- O12 normalize

def test_normalize_exact_rational_and_layout():
    mean, std = (0.485, 0.456, 0.406), (0.229, 0.224, 0.225)
    img = np.zeros((2, 3, 3), np.uint8)
    img[..., 0], img[..., 1], img[..., 2] = 10, 128, 255
    o = run([{"kind": "Normalize", "mean": mean, "std": std}], img)["nchw"]
    assert o.shape == (3, 2, 3) and o.dtype == np.float32
    for c, v in enumerate([10, 128, 255]):
        exact = (Fraction(v, 255) - Fraction(mean[c])) / Fraction(std[c])
        f = np.float32(float(exact))
        assert (o[c] == f).all() or np.abs(o[c] - f).max() <= np.spacing(f)


# ---------------------------------------------------------- O13 boxes

def test_boxes_affine_vs_cv2_transform():
    """affine boxes = envelope of the 4 corners mapped by an
    independent route (cv2 matrix on pixel-centre coordinates), 200 cases."""
    rng = np.random.default_rng(13)
    h, w = 40, 60
    img = rand_img(h, w)
    for _ in range(200):
        dx, dy = rng.uniform(-0.1, 0.1, 2)
        s, t = rng.uniform(0.8, 1.2), rng.uniform(-90, 90)
        x0, y0 = rng.uniform(0.3, 0.5, 2)
        bx = np.array([[x0, y0, x0 + 0.1, y0 + 0.15]], np.float32)
        ops = [{"kind": "ShiftScaleRotate", "lo": [dx, dy, s, t], "hi": [dx, dy, s, t]}]
        r = run(ops, img, boxes=bx)
        M = cv2.getRotationMatrix2D(((w - 1) / 2.0, (h - 1) / 2.0), t, s)
        M[0, 2] += dx * w
        M[1, 2] += dy * h
        X = np.array([bx[0, 0], bx[0, 2]], np.float64) * w
        Y = np.array([bx[0, 1], bx[0, 3]], np.float64) * h
        pts = np.array([[x - 0.5, y - 0.5] for x in X for y in Y]).reshape(-1, 1, 2)
        q = cv2.transform(pts, M).reshape(-1, 2) + 0.5
        env = [max(q[:, 0].min(), 0) / w, max(q[:, 1].min(), 0) / h,
               min(q[:, 0].max(), w) / w, min(q[:, 1].max(), h) / h]
        assert np.allclose(r["boxes"][0], env, atol=1e-6)
        b = r["boxes"][0]
        assert 0 <= b[0] < b[2] <= 1 and 0 <= b[1] < b[3] <= 1


def test_boxes_rotate180_equals_double_flip():
    img = rand_img(20, 30)
    rng = np.random.default_rng(14)
    xs = np.sort(rng.uniform(0, 1, size=(30, 2)), axis=1)
    ys = np.sort(rng.uniform(0, 1, size=(30, 2)), axis=1)
    bx = np.stack([xs[:, 0], ys[:, 0], xs[:, 1], ys[:, 1]], 1).astype(np.float32)
    a = run([{"kind": "Rotate", "lo": [180], "hi": [180]}], img, boxes=bx)["boxes"]
    b = run([{"kind": "HorizontalFlip"}, {"kind": "VerticalFlip"}], img, boxes=bx)["boxes"]
    assert np.allclose(a, b, atol=1e-6)


# ----------------------------------------------------------- O14 compose

def test_pipeline_identities():
    img = rand_img(10, 12)
    assert (run([], img)["image"] == img).all()
    allp0 = [{"kind": k, "p": 0.0, "lo": [1.5], "hi": [1.5]}
             for k in ["HorizontalFlip", "Brightness", "Rotate", "Gamma"]]
    for s in range(20):
        assert (run(allp0, img, seed=s)["image"] == img).all()


def test_pipeline_equals_chain_of_fixed_single_ops():
    """cfg4 composite = the same ops applied one by one with the drawn params
    fixed (lo == hi): pins O14 sequencing with per-op u8 rounding."""
    from synth.configs import CFG4_OPS
    from synth.gen import gen_images
    img = gen_images([(75, 100)], seed=3).image(0)
    ops = [dict(o) for o in CFG4_OPS]
    ops[0]["side"] = (20, 75)
    ops[0]["size"] = (32, 32)
    ops[1]["size"] = (32, 32)
    for idx in range(8):
        prm, fired = A.sample_params(ops, 9, idx, 75, 100)
        full = A.apply(ops, 9, idx, img)["nchw"]
        side, x0, y0 = [int(v) for v in prm[0][:3]]
        x = A.apply([{"kind": "Crop", "origin": (x0, y0), "size": (side, side)}], 0, 0, img)["image"]
        x = A.apply([{"kind": "Resize", "size": (32, 32)}], 0, 0, x)["image"]
        if fired[2]:
            x = A.apply([{"kind": "HorizontalFlip"}], 0, 0, x)["image"]
        x = A.apply([{"kind": "ShiftHSV", "lo": list(prm[3][:3]), "hi": list(prm[3][:3])}], 0, 0, x)["image"]
        x = A.apply([{"kind": "BrightnessContrast", "lo": list(prm[4][:2]), "hi": list(prm[4][:2])}], 0, 0, x)["image"]
        n = A.apply([ops[5]], 0, 0, x)["nchw"]
        assert (n == full).all()


def test_validation_errors():
    img = rand_img(10, 10)
    bad = [([{"kind": "Gamma", "lo": [0.0], "hi": [1.0]}], A.OracleError),
           ([{"kind": "Brightness", "p": 1.5, "lo": [1], "hi": [1]}], A.OracleError),
           ([{"kind": "RandomCrop", "size": (11, 5)}], A.OracleError),
           ([{"kind": "PadToSize", "size": (5, 5)}], A.OracleError),
           ([{"kind": "Resize", "p": 0.5, "size": (5, 5)}], A.OracleError),
           ([{"kind": "Normalize"}, {"kind": "HorizontalFlip"}], A.OracleError)]
    for ops, exc in bad:
        with pytest.raises(exc):
            run(ops, img)
    with pytest.raises(A.OracleError):
        A.apply([{"kind": "Grayscale"}], 0, 0, img[:, :, :1])


# --------------------------------------------------- D4 / rot90

def _r90(k):
    return [{"kind": "Rotate90", "lo": [k], "hi": [k]}]


def _d4(e):
    return [{"kind": "D4", "lo": [e], "hi": [e]}]


def test_rot90_spec_examples_and_numpy():
    """1x2 [a, b], k=1 -> 2x1 [b; a]; k=0 identity; the pixel
    map out[y][x] = in[x][W-1-y] is numpy's counter-clockwise np.rot90."""
    ab = np.array([[[1, 1, 1], [2, 2, 2]]], np.uint8)
    r = run(_r90(1), ab)["image"]
    assert r.shape == (2, 1, 3) and (r[:, 0, 0] == [2, 1]).all()
    img = rand_img(5, 8)
    m = RNG.integers(0, 7, size=(5, 8), dtype=np.uint8)
    for k in range(4):
        out = run(_r90(k), img, mask=m)
        assert (out["image"] == np.rot90(img, k)).all(), k
        assert (out["mask"] == np.rot90(m, k)).all(), k
    four = run(_r90(1) * 4, img)["image"]  # group law r^4 = e
    assert (four == img).all()


def test_rot90_boxes_spec_example_and_half_turn():
    """box (0.0, 0.0, 0.5, 0.25), k=1 -> envelope (0.0, 0.5, 0.25, 1.0);
    k=2 on boxes equals hflip o vflip."""
    img = rand_img(12, 12)
    r = run(_r90(1), img, boxes=np.array([[0.0, 0.0, 0.5, 0.25]], np.float32))
    assert np.allclose(r["boxes"][0], [0.0, 0.5, 0.25, 1.0], atol=1e-7)
    rng = np.random.default_rng(21)
    xs = np.sort(rng.uniform(0, 1, size=(20, 2)), axis=1)
    ys = np.sort(rng.uniform(0, 1, size=(20, 2)), axis=1)
    bx = np.stack([xs[:, 0], ys[:, 0], xs[:, 1], ys[:, 1]], 1).astype(np.float32)
    img2 = rand_img(9, 14)
    a = run(_r90(2), img2, boxes=bx)["boxes"]
    b = run([{"kind": "HorizontalFlip"}, {"kind": "VerticalFlip"}], img2, boxes=bx)["boxes"]
    assert np.allclose(a, b, atol=1e-6)
    # k=1 boxes by the corner map (x, y) -> (y, 1 - x), non-square
    c = run(_r90(1), img2, boxes=bx)["boxes"]
    want = np.stack([bx[:, 1], 1 - bx[:, 2], bx[:, 3], 1 - bx[:, 0]], 1)
    assert np.allclose(c, want, atol=1e-6)


def test_d4_elements_and_cayley_closure():
    """element 0 identity, element 4 = hflip, element e =
    h^(e>=4) o r^(e&3) (= np.fliplr(np.rot90(x, e&3))), and the 8 x 8 Cayley
    table is closed on a random 8x8 image (brute force)."""
    ab = np.array([[[1, 1, 1], [2, 2, 2]]], np.uint8)
    assert (run(_d4(4), ab)["image"] == ab[:, ::-1]).all()
    img = rand_img(8, 8)
    outs = []
    for e in range(8):
        o = run(_d4(e), img)["image"]
        ref = np.rot90(img, e & 3)
        if e >= 4:
            ref = ref[:, ::-1]
        assert (o == ref).all(), e
        outs.append(o)
    assert (outs[0] == img).all()
    for i in range(8):
        for j in range(8):
            comp = run(_d4(i) + _d4(j), img)["image"]
            assert any((comp == outs[k]).all() for k in range(8)), (i, j)
    assert len({o.tobytes() for o in outs}) == 8  # the 8 elements are distinct


def test_rot90_shape_rule_and_draws():
    """Reading R30: a random element range whose parity can change on a
    non-square image is rejected; odd-only ranges transpose the shape; on a
    square image any range is fine; draws are uniform over the range."""
    assert A.output_shape([{"kind": "Rotate90", "lo": [3], "hi": [3]}], 5, 8) == (8, 5)
    assert A.output_shape([{"kind": "D4", "lo": [5], "hi": [5]}], 5, 8) == (8, 5)
    assert A.output_shape([{"kind": "Rotate90", "lo": [2], "hi": [2]}], 5, 8) == (5, 8)
    with pytest.raises(A.OracleError):  # {1, 2, 3} mixes parities on a non-square image
        A.output_shape([{"kind": "Rotate90", "lo": [1], "hi": [3]}], 5, 8)
    assert A.output_shape([{"kind": "Rotate90", "lo": [0], "hi": [3]}], 6, 6) == (6, 6)
    with pytest.raises(A.OracleError):
        A.output_shape([{"kind": "Rotate90", "lo": [0], "hi": [3]}], 5, 8)
    with pytest.raises(A.OracleError):  # p < 1 on a non-square image with an odd element
        A.output_shape([{"kind": "D4", "p": 0.5, "lo": [1], "hi": [1]}], 5, 8)
    with pytest.raises(A.OracleError):
        A.output_shape([{"kind": "D4", "lo": [0], "hi": [8]}], 6, 6)
    counts = np.zeros(8, int)
    for idx in range(4000):
        prm, fired = A.sample_params([{"kind": "D4", "lo": [0], "hi": [7]}], 3, idx, 6, 6)
        counts[int(prm[0][0])] += 1
    assert counts.min() > 400 and counts.max() < 600


# ------------------------------------------------------------ GridDistortion

def _grid(lo, hi, n, interp="bilinear", p=1.0):
    return [{"kind": "GridDistortion", "p": p, "lo": [lo], "hi": [hi], "num_steps": n, "interp": interp}]


def test_grid_axis_hand_example():
    """Reading R31 traced by hand: L = 11, n = 2, f = (1.5, 0.5): knots d = (0, 5, 10),
    S = 2, s = (0, 7.5, 10), so slope 1.5 on [0, 5] and 0.5 on [5, 10].  f[n] is unused."""
    want = [0, 1.5, 3, 4.5, 6, 7.5, 8, 8.5, 9, 9.5, 10]
    for last in (1.0, 0.3, 1.9):
        assert A.grid_axis(11, 2, [1.5, 0.5, last]).tolist() == want
    assert A.grid_axis(1, 3, [1.2, 0.7, 1.1, 1.0]).tolist() == [0.0]
    with pytest.raises(A.OracleError):
        A.grid_axis(10, 0, [1.0])
    with pytest.raises(A.OracleError):
        A.grid_axis(10, 2, [1.0, 0.0, 1.0])


def test_grid_axis_monotone_span_and_knots():
    """over 1000 random draws the axis map is strictly
    monotone, keeps the span (src[0] = 0, src[L-1] = L-1 exactly), passes
    through the rescaled knots s_i = (L-1) c_i / S (exact rational arithmetic)
    and is linear inside each cell with slope n f_i / S."""
    rng = np.random.default_rng(31)
    for _ in range(1000):
        L = int(rng.integers(1, 400))
        n = int(rng.integers(1, 33))
        d = float(rng.uniform(0.0, 0.95))
        f = 1.0 + rng.uniform(-d, d, n + 1)
        src = A.grid_axis(L, n, f)
        assert src[0] == 0.0 and src[-1] == L - 1
        if L == 1:
            continue
        assert (np.diff(src) > 0).all()
        S = sum(Fraction(float(v)) for v in f[:n])
        c = Fraction(0)
        for i in range(n + 1):
            if (i * (L - 1)) % n == 0:  # knot on an integer destination index
                x = i * (L - 1) // n
                assert abs(src[x] - float((L - 1) * c / S)) < 1e-9, (L, n, i)
            if i < n:
                c += Fraction(float(f[i]))
        cell = np.minimum((np.arange(L) * n) // (L - 1), n - 1)
        for x in range(L - 1):
            if (x + 1) * n <= (cell[x] + 1) * (L - 1):  # x + 1 still inside (or closing) x's cell
                assert abs((src[x + 1] - src[x]) - n * f[cell[x]] / float(S)) < 1e-9


def test_grid_identity_at_zero_limit():
    """distort_limit = 0 is the identity, bit-exact, for both
    interpolations, image and mask, any n (also n > L - 1) and degenerate sizes."""
    rng = np.random.default_rng(7)
    for (h, w) in [(1, 1), (1, 17), (23, 1), (19, 31), (64, 48)]:
        img = rand_img(h, w, rng=rng)
        m = rng.integers(0, 5, (h, w), dtype=np.uint8)
        for n in (1, 5, 32):
            for interp in ("bilinear", "nearest"):
                r = run(_grid(0.0, 0.0, n, interp), img, mask=m, seed=3, idx=9)
                assert (r["image"] == img).all() and (r["mask"] == m).all()


def _grid_maps(lo, hi, n, h, w, seed, idx, slot=0):
    """factor draws as SPEC.md:332 orders them: x steps j = 1..n+1, then y steps"""
    fx = [1.0 + lo + (hi - lo) * A.draw(seed, idx, slot, 1 + i) for i in range(n + 1)]
    fy = [1.0 + lo + (hi - lo) * A.draw(seed, idx, slot, n + 2 + i) for i in range(n + 1)]
    return A.grid_axis(w, n, fx), A.grid_axis(h, n, fy)


def test_grid_remap_of_linear_ramp():
    """Bilinear interpolation reproduces an affine image g(x, y) exactly, so the
    bilinear output is round_half_up(g(mx[x], my[y])) and the nearest output is
    g(round(mx), round(my)): pins the draw order (x factors before y), the axis
    orientation and the taps.  Masks follow the nearest taps."""
    h, w = 90, 100
    yy, xx = np.mgrid[0:h, 0:w]
    img = np.stack([xx + yy, 2 * xx, 255 - yy], -1).astype(np.uint8)
    mask = ((3 * xx + 7 * yy) % 11).astype(np.uint8)
    for (lo, hi, n, seed) in [(-0.3, 0.3, 5, 11), (-0.6, 0.2, 3, 12), (-0.1, 0.5, 8, 13)]:
        mx, my = _grid_maps(lo, hi, n, h, w, seed, 4)
        assert np.abs(mx - np.arange(w)).max() > 0.5  # a visible distortion
        X, Y = np.meshgrid(mx, my)
        g = np.stack([X + Y, 2 * X, 255 - Y], -1)
        r = run(_grid(lo, hi, n), img, mask=mask, seed=seed, idx=4)
        frac = g - np.floor(g)
        ok = np.abs(frac - 0.5) > 1e-9
        assert (r["image"][ok] == np.floor(g + 0.5)[ok]).all()
        xn, yn = np.floor(mx + 0.5).astype(int), np.floor(my + 0.5).astype(int)
        rn = run(_grid(lo, hi, n, "nearest"), img, mask=mask, seed=seed, idx=4)
        assert (rn["image"] == img[yn][:, xn]).all()
        assert (r["mask"] == mask[yn][:, xn]).all() and (rn["mask"] == mask[yn][:, xn]).all()


def test_grid_validation_and_boxes_rejected():
    """SPEC.md:313 factors stay > 0 (|d| < 1), num_steps >= 1 (cap 32, R31);
    SPEC.md:318/346: boxes under a free-form warp are an unsupported target."""
    img = rand_img(10, 12)
    for bad in (_grid(-1.0, 0.2, 4), _grid(0.0, 1.0, 4), _grid(0.0, 0.1, 0), _grid(0.0, 0.1, 33)):
        with pytest.raises(A.OracleError) as e:
            run(bad, img)
        assert e.value.code == -3
    with pytest.raises(A.OracleError) as e:
        run(_grid(-0.2, 0.2, 4), img, boxes=np.array([[0.1, 0.1, 0.5, 0.5]], np.float32))
    assert e.value.code == -5
    r = run(_grid(-0.2, 0.2, 4, p=0.0), img)  # gate off: identity
    assert (r["image"] == img).all()


# ---------------------------------------------------------- ElasticTransform

def _elastic(alpha, sigma, interp="bilinear", border="reflect_101", p=1.0):
    return [{"kind": "ElasticTransform", "p": p, "lo": [alpha, sigma], "hi": [alpha, sigma],
             "interp": interp, "border": border}]


def test_elastic_gauss_kernel():
    """SPEC.md:341 / invariant SPEC.md:350: symmetric, nonnegative, sums to 1
    (1e-12), radius ceil(3 sigma), weights proportional to math.exp(-k^2/2s^2)."""
    import math
    for sigma in (0.1, 0.5, 1.0, 1.7, 3.0, 4.0, 7.3, 16.0):
        w = A.gauss_kernel(sigma)
        r = math.ceil(3 * sigma)
        assert len(w) == 2 * r + 1
        assert (w >= 0).all() and abs(w.sum() - 1.0) < 1e-12
        assert np.array_equal(w, w[::-1])
        for k in range(-r, r + 1):
            assert abs(w[k + r] / w[r] - math.exp(-k * k / (2 * sigma * sigma))) < 1e-14
    for bad in (0.0, -1.0, 16.5):
        with pytest.raises(A.OracleError):
            A.gauss_kernel(bad)


def _reflect_idx(i, n):
    """reflect-101 by literal mirror steps (independent of the oracle's modular form)"""
    if n == 1:
        return 0
    while i < 0 or i >= n:
        i = -i if i < 0 else 2 * (n - 1) - i
    return i


def test_elastic_field_direct_2d_convolution():
    """separable blur == direct 2-D convolution (1e-9) on small
    fields, incl. kernels wider than the image (repeated reflection); the raw
    planes come from the draws in SPEC.md:341's order (u plane, then v plane,
    row-major) -- a transposed or swapped plane fails."""
    import math
    for (h, w, sigma, alpha) in [(9, 9, 1.0, 3.0), (9, 9, 2.5, 1.0), (5, 12, 1.3, 7.0), (1, 6, 0.7, 2.0),
                                 (4, 1, 2.0, 5.0)]:
        seed, idx, slot = 5, 17, 2
        raw = [np.array([[-1.0 + 2.0 * A.draw(seed, idx, slot, 1 + pl * h * w + y * w + x)
                          for x in range(w)] for y in range(h)]) for pl in (0, 1)]
        r = math.ceil(3 * sigma)
        g = np.array([math.exp(-k * k / (2 * sigma * sigma)) for k in range(-r, r + 1)])
        g /= g.sum()
        dx, dy = A.elastic_field(h, w, alpha, sigma, seed, idx, slot)
        for plane, d in zip(raw, (dx, dy)):
            ref = np.zeros((h, w))
            for y in range(h):
                for x in range(w):
                    ref[y, x] = alpha * sum(g[a + r] * g[b + r] * plane[_reflect_idx(y + a, h), _reflect_idx(x + b, w)]
                                            for a in range(-r, r + 1) for b in range(-r, r + 1))
            assert np.abs(d - ref).max() < 1e-9, (h, w, sigma)


def test_elastic_bound_and_identity():
    """|displacement| <= alpha (convexity); alpha = 0
    is the identity bit-exact (nearest and bilinear, image and mask)."""
    rng = np.random.default_rng(32)
    for _ in range(40):
        h, w = int(rng.integers(1, 40)), int(rng.integers(1, 40))
        alpha, sigma = float(rng.uniform(0, 50)), float(rng.uniform(0.05, 6))
        dx, dy = A.elastic_field(h, w, alpha, sigma, int(rng.integers(0, 1 << 40)), int(rng.integers(0, 1000)))
        assert np.abs(dx).max() <= alpha and np.abs(dy).max() <= alpha
    img = rand_img(23, 37, rng=rng)
    m = rng.integers(0, 4, (23, 37), dtype=np.uint8)
    for interp in ("bilinear", "nearest"):
        for border in ("constant", "reflect_101"):
            r = run(_elastic(0.0, 4.0, interp, border), img, mask=m, seed=9)
            assert (r["image"] == img).all() and (r["mask"] == m).all()


def test_elastic_remap_of_linear_ramp():
    """source = (x + dx, y + dy): on an affine ramp the bilinear
    output equals round(g(x + dx, y + dy)) wherever the sample is inside the
    image, the nearest output and the mask equal the ramp at the rounded
    source; outside, constant border gives the fill (all four taps out)."""
    h, w = 60, 80
    yy, xx = np.mgrid[0:h, 0:w]
    img = np.stack([xx + yy, 3 * xx, 200 - yy], -1).astype(np.uint8)
    mask = ((5 * xx + 3 * yy) % 7).astype(np.uint8)
    alpha, sigma = 40.0, 2.0
    dx, dy = A.elastic_field(h, w, alpha, sigma, 3, 6)
    xs, ys = xx + dx, yy + dy
    g = np.stack([xs + ys, 3 * xs, 200 - ys], -1)
    inside = (xs >= 0) & (xs <= w - 1) & (ys >= 0) & (ys <= h - 1)
    r = run(_elastic(alpha, sigma, border="constant"), img, mask=mask, seed=3, idx=6)
    ok = inside[..., None] & (np.abs(g - np.floor(g) - 0.5) > 1e-9)
    assert inside.mean() > 0.8 and (~inside).sum() > 0
    assert (r["image"][ok] == np.floor(g + 0.5)[ok]).all()
    out = (xs < -1) | (xs > w) | (ys < -1) | (ys > h)
    assert (r["image"][out] == 0).all()
    xn, yn = np.floor(xs + 0.5).astype(int), np.floor(ys + 0.5).astype(int)
    inn = (xn >= 0) & (xn < w) & (yn >= 0) & (yn < h)
    rn = run(_elastic(alpha, sigma, "nearest", "constant"), img, mask=mask, seed=3, idx=6)
    assert (rn["image"][inn] == img[yn[inn], xn[inn]]).all()
    assert (r["mask"][inn] == mask[yn[inn], xn[inn]]).all() and (r["mask"][~inn] == 0).all()


def test_elastic_validation_and_boxes_rejected():
    img = rand_img(10, 12)
    bad = [_elastic(-1.0, 2.0), _elastic(1.0, 0.0), _elastic(1.0, 17.0),
           [{"kind": "ElasticTransform", "lo": [1.0, 2.0], "hi": [2.0, 2.0]}]]
    for b in bad:
        with pytest.raises(A.OracleError) as e:
            run(b, img)
        assert e.value.code == -3
    with pytest.raises(A.OracleError) as e:
        run(_elastic(5.0, 2.0), img, boxes=np.array([[0.1, 0.1, 0.5, 0.5]], np.float32))
    assert e.value.code == -5


# ------------------------------------------ nearest-tie candidate sets (R20)

def test_cand_outputs_equal_apply_and_contain_result():
    """albref_apply_cand returns albref_apply's outputs unchanged, and every
    pixel's own value is a member of its candidate set."""
    rng = np.random.default_rng(77)
    cases = [([{"kind": "Rotate", "lo": [-90.0], "hi": [90.0], "interp": "nearest",
                "border": "reflect_101"}], (41, 57)),
             ([{"kind": "ShiftScaleRotate", "lo": [-.06, -.06, .9, -45.0], "hi": [.06, .06, 1.1, 45.0],
                "interp": "bilinear", "border": "constant", "fill": (3, 4, 5), "mask_fill": 9},
               {"kind": "RandomCrop", "size": (30, 20)}, {"kind": "HorizontalFlip", "p": 0.5}], (50, 60)),
             ([{"kind": "Resize", "size": (37, 23), "interp": "nearest"}, {"kind": "ShiftHSV",
               "lo": [-20, -.1, -.1], "hi": [20, .1, .1]}, {"kind": "Equalize"}], (61, 44)),
             ([{"kind": "ElasticTransform", "lo": [30.0, 3.0], "hi": [30.0, 3.0], "interp": "nearest"},
               {"kind": "Rotate90", "lo": [1], "hi": [1]}, {"kind": "PadToSize", "size": (70, 50)},
               {"kind": "Grayscale"}], (40, 33))]
    for specs, (h, w) in cases:
        img = rand_img(h, w, rng=rng)
        mask = rng.integers(0, 256, size=(h, w), dtype=np.uint8)
        for seed in range(4):
            a = A.apply(specs, seed, 3, img, mask)
            b = A.apply_cand(specs, seed, 3, img, mask)
            assert np.array_equal(a["image"], b["image"]) and np.array_equal(a["mask"], b["mask"])
            for which, val in (("image", b["image"]), ("mask", b["mask"])):
                cv, cn = b[which + "_cand"], b[which + "_cand_n"]
                v3 = val.reshape(val.shape[0], val.shape[1], -1)
                cv = cv.reshape(cv.shape[0], cv.shape[1], cv.shape[2], -1)
                for y in range(v3.shape[0]):
                    for x in range(v3.shape[1]):
                        n = cn[y, x]
                        assert n == 0 or any(np.array_equal(cv[y, x, k], v3[y, x]) for k in range(n))


def test_cand_exact_ties_brute_force():
    """Resize 4 -> 2 (nearest) samples x_s = (x + 0.5) 2 - 0.5 = 2x + 0.5:
    every output is an exact .5 tie.  round_half_up picks
    column 2x + 1; the candidate set is exactly {in[2x], in[2x+1]}, and an
    HFlip afterwards moves the sets with the pixels (O2)."""
    img = np.array([[[10, 11, 12], [20, 21, 22], [30, 31, 32], [40, 41, 42]]], np.uint8)
    mask = np.array([[1, 2, 3, 4]], np.uint8)
    rz = {"kind": "Resize", "size": (2, 1), "interp": "nearest"}
    for specs, order in (([rz], [0, 1]), ([rz, {"kind": "HorizontalFlip"}], [1, 0])):
        o = A.apply_cand(specs, 0, 0, img, mask)
        for x, src in enumerate(order):
            assert o["image"][0, x].tolist() == img[0, 2 * src + 1].tolist()
            assert o["mask"][0, x] == mask[0, 2 * src + 1]
            assert o["image_cand_n"][0, x] == 2 and o["mask_cand_n"][0, x] == 2
            assert sorted(o["mask_cand"][0, x, :2].tolist()) == [mask[0, 2 * src], mask[0, 2 * src + 1]]
            got = sorted(map(tuple, o["image_cand"][0, x, :2].tolist()))
            assert got == sorted([tuple(img[0, 2 * src]), tuple(img[0, 2 * src + 1])])


def test_cand_no_ties_on_integer_coordinates():
    """Rotate 90 on a square image maps pixel centres onto pixel centres
    (SPEC.md:196, 218): no source coordinate is near a tie, every set is the
    singleton of the result."""
    img = rand_img(31, 31)
    mask = RNG.integers(0, 256, size=(31, 31), dtype=np.uint8)
    o = A.apply_cand([{"kind": "Rotate", "lo": [90.0], "hi": [90.0], "interp": "nearest"}], 0, 0,
                     img, mask)
    assert (o["image_cand_n"] == 1).all() and (o["mask_cand_n"] == 1).all()
    assert np.array_equal(o["mask"], np.rot90(mask, 1))


def test_cand_band_rate_matches_survey():
    """SSR on 512^2 (cfg3): the 1e-4 px band holds about 0.04% of the mask
    pixels (SURVEY.md §8(c) tolerance table: 2 axes x 2e-4 of each unit)."""
    img = rand_img(512, 512)
    mask = RNG.integers(0, 256, size=(512, 512), dtype=np.uint8)
    specs = [{"kind": "ShiftScaleRotate", "lo": [-.0625, -.0625, .9, -45.0],
              "hi": [.0625, .0625, 1.1, 45.0], "interp": "bilinear", "border": "reflect_101"}]
    rates = []
    for seed in range(3):
        o = A.apply_cand(specs, seed, 0, img, mask)
        rates.append(float((o["mask_cand_n"] != 1).mean()))
    assert 1e-4 < np.mean(rates) < 1e-3, rates
