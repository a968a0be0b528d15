"""ctypes wrapper around the CPU oracle ``oracle/libalbref.so``.

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and the
``cpu_baseline`` / ``--impl reference`` legs of bench.py.  The product package
(paper_1809_06839_b200) never imports this module.

Op specs are plain dicts (see synth/configs.py); this module converts them to
its own ``albref_op`` struct.  Conversion is argument marshalling only; all
arithmetic is in albref.c.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from concurrent.futures import ThreadPoolExecutor

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "albref.c")
HDR = os.path.join(HERE, "albref.h")
LIB = os.path.join(HERE, "libalbref.so")

KINDS = {
    "HorizontalFlip": 0, "VerticalFlip": 1, "Rotate": 2, "ShiftScaleRotate": 3,
    "RandomCrop": 4, "PadToSize": 5, "Resize": 6, "RandomSizedCrop": 7,
    "Brightness": 8, "Contrast": 9, "BrightnessContrast": 10, "Gamma": 11,
    "ShiftRGB": 12, "ShiftHSV": 13, "Grayscale": 14, "Equalize": 15,
    "Normalize": 16, "Crop": 17, "Rotate90": 18, "D4": 19, "GridDistortion": 20, "ElasticTransform": 21,
}
INTERP = {"nearest": 0, "bilinear": 1}
BORDER = {"constant": 0, "reflect_101": 1}
MAX_PARAMS = 8
MAX_CAND = 8       # ALBREF_MAX_CAND
TIE_BAND = 1e-4    # ALBREF_TIE_BAND


class AlbrefOp(ctypes.Structure):
    _fields_ = [
        ("kind", ctypes.c_int32),
        ("p", ctypes.c_double),
        ("lo", ctypes.c_double * 4),
        ("hi", ctypes.c_double * 4),
        ("out_w", ctypes.c_int32), ("out_h", ctypes.c_int32),
        ("min_side", ctypes.c_int32), ("max_side", ctypes.c_int32),
        ("crop_x", ctypes.c_int32), ("crop_y", ctypes.c_int32),
        ("interp", ctypes.c_int32), ("border", ctypes.c_int32),
        ("fill", ctypes.c_uint8 * 3), ("mask_fill", ctypes.c_uint8),
        ("mean", ctypes.c_double * 3), ("std", ctypes.c_double * 3),
        ("num_steps", ctypes.c_int32), ("reserved", ctypes.c_int32),
    ]


def build(force: bool = False) -> str:
    """Compile the oracle (plain C, -O2 -ffp-contract=off, no SIMD intrinsics)."""
    stale = (not os.path.exists(LIB)
             or os.path.getmtime(LIB) < max(os.path.getmtime(SRC), os.path.getmtime(HDR)))
    if force or stale:
        tmp = LIB + ".tmp%d" % os.getpid()
        subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-std=c11",
                               "-Wall", "-fPIC", "-shared", "-o", tmp, SRC, "-lm"])
        os.replace(tmp, LIB)
    return LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(LIB)
        P = ctypes.POINTER
        L.albref_philox4x32_10.argtypes = [P(ctypes.c_uint32), P(ctypes.c_uint32), P(ctypes.c_uint32)]
        L.albref_u53.argtypes = [ctypes.c_uint32, ctypes.c_uint32]
        L.albref_u53.restype = ctypes.c_double
        L.albref_draw.argtypes = [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int32, ctypes.c_int32]
        L.albref_draw.restype = ctypes.c_double
        L.albref_clip_round.argtypes = [ctypes.c_double]
        L.albref_clip_round.restype = ctypes.c_uint8
        L.albref_reflect101.argtypes = [ctypes.c_int32, ctypes.c_int32]
        L.albref_reflect101.restype = ctypes.c_int32
        D = P(ctypes.c_double)
        L.albref_rgb_to_hsv.argtypes = [ctypes.c_double] * 3 + [D] * 3
        L.albref_hsv_to_rgb.argtypes = [ctypes.c_double] * 3 + [D] * 3
        L.albref_build_lut.argtypes = [ctypes.c_int32, D, ctypes.c_void_p]
        L.albref_equalize_lut.argtypes = [ctypes.c_void_p, ctypes.c_void_p]
        L.albref_grid_axis.argtypes = [ctypes.c_int32, ctypes.c_int32, ctypes.c_void_p, ctypes.c_void_p]
        L.albref_gauss_kernel.argtypes = [ctypes.c_double, ctypes.c_void_p]
        L.albref_elastic_field.argtypes = [ctypes.c_int32, ctypes.c_int32, ctypes.c_double, ctypes.c_double,
                                           ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int32,
                                           ctypes.c_void_p, ctypes.c_void_p]
        L.albref_output_shape.argtypes = [P(AlbrefOp), ctypes.c_int32, ctypes.c_int32,
                                          ctypes.c_int32, P(ctypes.c_int32), P(ctypes.c_int32)]
        L.albref_sample_params.argtypes = [P(AlbrefOp), ctypes.c_int32, ctypes.c_uint64,
                                           ctypes.c_uint64, ctypes.c_int32, ctypes.c_int32,
                                           ctypes.c_void_p, ctypes.c_void_p]
        L.albref_apply.argtypes = [P(AlbrefOp), ctypes.c_int32, ctypes.c_uint64, ctypes.c_uint64,
                                   ctypes.c_void_p, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                                   ctypes.c_void_p,
                                   ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int32, ctypes.c_float,
                                   ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                   ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
        L.albref_apply_cand.argtypes = [P(AlbrefOp), ctypes.c_int32, ctypes.c_uint64, ctypes.c_uint64,
                                        ctypes.c_void_p, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                                        ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                        ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
        _lib = L
    return _lib


class OracleError(RuntimeError):
    def __init__(self, code):
        super().__init__("albref error %d" % code)
        self.code = code


def _check(rc):
    if rc != 0:
        raise OracleError(rc)


def make_ops(specs):
    """list of op-spec dicts -> ctypes array of AlbrefOp"""
    arr = (AlbrefOp * max(1, len(specs)))()
    for k, s in enumerate(specs):
        o = arr[k]
        o.kind = KINDS[s["kind"]] if isinstance(s["kind"], str) else int(s["kind"])
        o.p = float(s.get("p", 1.0))
        lo = list(s.get("lo", [])) + [0.0] * 4
        hi = list(s.get("hi", s.get("lo", []))) + [0.0] * 4
        for j in range(4):
            o.lo[j] = float(lo[j])
            o.hi[j] = float(hi[j])
        o.out_w, o.out_h = [int(v) for v in s.get("size", (0, 0))]
        o.min_side, o.max_side = [int(v) for v in s.get("side", (0, 0))]
        o.crop_x, o.crop_y = [int(v) for v in s.get("origin", (0, 0))]
        o.interp = INTERP[s.get("interp", "bilinear")]
        o.border = BORDER[s.get("border", "constant")]
        f = list(s.get("fill", (0, 0, 0)))
        for c in range(3):
            o.fill[c] = int(f[c])
        o.mask_fill = int(s.get("mask_fill", 0))
        o.num_steps = int(s.get("num_steps", 0))
        m = s.get("mean", (0.0, 0.0, 0.0))
        d = s.get("std", (1.0, 1.0, 1.0))
        for c in range(3):
            o.mean[c] = float(m[c])
            o.std[c] = float(d[c])
    return arr, len(specs)


# ---------------------------------------------------------------- primitives

def philox(ctr, key):
    c = (ctypes.c_uint32 * 4)(*[int(v) & 0xFFFFFFFF for v in ctr])
    k = (ctypes.c_uint32 * 2)(*[int(v) & 0xFFFFFFFF for v in key])
    o = (ctypes.c_uint32 * 4)()
    lib().albref_philox4x32_10(c, k, o)
    return [int(v) for v in o]


def u53(a, b):
    return lib().albref_u53(a, b)


def draw(seed, image_index, slot, j):
    return lib().albref_draw(seed, image_index, slot, j)


def clip_round(v):
    return int(lib().albref_clip_round(float(v)))


def reflect101(i, n):
    return int(lib().albref_reflect101(int(i), int(n)))


def rgb_to_hsv(r, g, b):
    h, s, v = ctypes.c_double(), ctypes.c_double(), ctypes.c_double()
    lib().albref_rgb_to_hsv(float(r), float(g), float(b), ctypes.byref(h), ctypes.byref(s),
                            ctypes.byref(v))
    return h.value, s.value, v.value


def hsv_to_rgb(h, s, v):
    r, g, b = ctypes.c_double(), ctypes.c_double(), ctypes.c_double()
    lib().albref_hsv_to_rgb(float(h), float(s), float(v), ctypes.byref(r), ctypes.byref(g),
                            ctypes.byref(b))
    return r.value, g.value, b.value


def build_lut(kind, params):
    p = (ctypes.c_double * MAX_PARAMS)(*(list(params) + [0.0] * MAX_PARAMS)[:MAX_PARAMS])
    lut = np.zeros((3, 256), np.uint8)
    k = KINDS[kind] if isinstance(kind, str) else int(kind)
    _check(lib().albref_build_lut(k, p, lut.ctypes.data))
    return lut


def equalize_lut(hist):
    h = np.ascontiguousarray(hist, dtype=np.int64)
    assert h.shape == (256,)
    lut = np.zeros(256, np.uint8)
    _check(lib().albref_equalize_lut(h.ctypes.data, lut.ctypes.data))
    return lut


def grid_axis(L, n, factors):
    """GridDistortion source coordinate of every destination index along an
    axis of length L for step factors f[0..n] (reading R31)."""
    f = np.ascontiguousarray(factors, np.float64)
    out = np.zeros(max(1, L), np.float64)
    _check(lib().albref_grid_axis(L, n, f.ctypes.data, out.ctypes.data))
    return out[:L]


def gauss_kernel(sigma):
    """ElasticTransform smoothing weights w[0..2r] (reading R32)."""
    w = np.zeros(97, np.float64)
    r = lib().albref_gauss_kernel(sigma, w.ctypes.data)
    _check(min(r, 0))
    return w[:2 * r + 1]


def elastic_field(h, w, alpha, sigma, seed, image_index, slot=0):
    """ElasticTransform displacement planes (dx, dy), each (h, w) float64."""
    dx = np.zeros((h, w), np.float64)
    dy = np.zeros((h, w), np.float64)
    _check(lib().albref_elastic_field(h, w, alpha, sigma, seed, image_index, slot,
                                      dx.ctypes.data, dy.ctypes.data))
    return dx, dy


def output_shape(specs, h, w):
    ops, n = make_ops(specs)
    oh, ow = ctypes.c_int32(), ctypes.c_int32()
    _check(lib().albref_output_shape(ops, n, h, w, ctypes.byref(oh), ctypes.byref(ow)))
    return oh.value, ow.value


def sample_params(specs, seed, image_index, h, w):
    ops, n = make_ops(specs)
    prm = np.zeros((max(1, n), MAX_PARAMS), np.float64)
    fired = np.zeros(max(1, n), np.uint8)
    _check(lib().albref_sample_params(ops, n, seed, image_index, h, w, prm.ctypes.data,
                                      fired.ctypes.data))
    return prm[:n], fired[:n]


def apply(specs, seed, image_index, img, mask=None, boxes=None, labels=None,
          min_visibility=0.0, _ops=None):
    """Apply the pipeline to one sample.  img: (h, w, c) uint8.

    Returns dict(image=(oh,ow,c) uint8 or None, nchw=(3,oh,ow) f32 or None,
    mask=(oh,ow) or None, boxes=(k,4) f32 or None, labels=(k,) or None)."""
    img = np.ascontiguousarray(img, dtype=np.uint8)
    if img.ndim == 2:
        img = img[:, :, None]
    h, w, c = img.shape
    ops, n = _ops if _ops is not None else make_ops(specs)
    oh, ow = output_shape(specs, h, w)
    ends_norm = n > 0 and ops[n - 1].kind == KINDS["Normalize"]
    out = None if ends_norm else np.zeros((oh, ow, c), np.uint8)
    nchw = np.zeros((3, oh, ow), np.float32) if ends_norm else None
    mk = None
    if mask is not None:
        mask = np.ascontiguousarray(mask, dtype=np.uint8)
        assert mask.shape == (h, w)
        mk = np.zeros((oh, ow), np.uint8)
    nb = 0
    bx = lb = bo = lo = None
    nbo = ctypes.c_int32(0)
    if boxes is not None:
        bx = np.ascontiguousarray(boxes, dtype=np.float32).reshape(-1, 4)
        nb = bx.shape[0]
        lb = (np.ascontiguousarray(labels, dtype=np.int32) if labels is not None
              else np.zeros(nb, np.int32))
        bo = np.zeros((max(1, nb), 4), np.float32)
        lo = np.zeros(max(1, nb), np.int32)

    def ptr(a):
        return None if a is None else a.ctypes.data

    _check(lib().albref_apply(ops, n, seed, image_index, img.ctypes.data, h, w, c, ptr(mask),
                              ptr(bx), ptr(lb), nb, min_visibility,
                              ptr(out), ptr(nchw), ptr(mk), ptr(bo), ptr(lo),
                              ctypes.byref(nbo) if boxes is not None else None))
    res = {"image": None if out is None else (out if c > 1 else out[:, :, 0]),
           "nchw": nchw, "mask": mk, "boxes": None, "labels": None}
    if boxes is not None:
        k = nbo.value
        res["boxes"] = bo[:k].copy()
        res["labels"] = lo[:k].copy()
    return res


def apply_cand(specs, seed, image_index, img, mask=None, _ops=None):
    """albref_apply_cand: as apply() (no boxes) plus the nearest-tie candidate
    sets of every output pixel: image_cand (oh, ow, MAX_CAND, c) with
    image_cand_n (oh, ow) members (0 = any), likewise mask_cand / mask_cand_n."""
    img = np.ascontiguousarray(img, dtype=np.uint8)
    if img.ndim == 2:
        img = img[:, :, None]
    h, w, c = img.shape
    ops, n = _ops if _ops is not None else make_ops(specs)
    oh, ow = output_shape(specs, h, w)
    ends_norm = n > 0 and ops[n - 1].kind == KINDS["Normalize"]
    out = None if ends_norm else np.zeros((oh, ow, c), np.uint8)
    nchw = np.zeros((3, oh, ow), np.float32) if ends_norm else None
    ci = np.zeros((oh, ow, MAX_CAND, c), np.uint8)
    cin = np.zeros((oh, ow), np.uint8)
    mk = cm = cmn = None
    if mask is not None:
        mask = np.ascontiguousarray(mask, dtype=np.uint8)
        assert mask.shape == (h, w)
        mk = np.zeros((oh, ow), np.uint8)
        cm = np.zeros((oh, ow, MAX_CAND), np.uint8)
        cmn = np.zeros((oh, ow), np.uint8)

    def ptr(a):
        return None if a is None else a.ctypes.data

    _check(lib().albref_apply_cand(ops, n, seed, image_index, img.ctypes.data, h, w, c, ptr(mask),
                                   ptr(out), ptr(nchw), ptr(mk), ci.ctypes.data, cin.ctypes.data,
                                   ptr(cm), ptr(cmn)))
    return {"image": None if out is None else (out if c > 1 else out[:, :, 0]), "nchw": nchw,
            "mask": mk, "image_cand": ci, "image_cand_n": cin, "mask_cand": cm, "mask_cand_n": cmn}


def apply_batch_cand(specs, seed, first_image_index, images, masks=None, threads=1):
    ops = make_ops(specs)

    def one(i):
        return apply_cand(specs, seed, first_image_index + i, images[i],
                          None if masks is None else masks[i], _ops=ops)

    if threads <= 1:
        return [one(i) for i in range(len(images))]
    with ThreadPoolExecutor(threads) as ex:
        return list(ex.map(one, range(len(images))))


def apply_batch(specs, seed, first_image_index, images, masks=None, boxes=None, labels=None,
                min_visibility=0.0, threads=1):
    """Apply to a list of samples; image i gets global index first_image_index + i.
    ``threads`` > 1 runs images concurrently (ctypes releases the GIL)."""
    ops = make_ops(specs)

    def one(i):
        return apply(specs, seed, first_image_index + i, images[i],
                     None if masks is None else masks[i],
                     None if boxes is None else boxes[i],
                     None if labels is None else labels[i], min_visibility, _ops=ops)

    if threads <= 1:
        return [one(i) for i in range(len(images))]
    with ThreadPoolExecutor(threads) as ex:
        return list(ex.map(one, range(len(images))))
