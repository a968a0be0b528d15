"""Thin Python wrappers with the ABI's names (alb_pipeline / alb_layout /
alb_plan / alb_apply).  Argument marshalling only; torch supplies device
memory and the current stream.  Op specs are dicts:

    {"kind": "Rotate", "p": 1.0, "lo": [-90], "hi": [90],
     "interp": "bilinear", "border": "reflect_101"}

with optional size=(w, h), side=(min, max), origin=(x, y), fill, mask_fill, num_steps,
mean, std (see include/alb_b200.h for the meaning of every field).
"""
from __future__ import annotations

import ctypes
import json

import numpy as np
import torch

from . import _lib
from ._lib import AlbImageDesc, AlbOp, check, lib


def make_ops(specs):
    arr = (AlbOp * max(1, len(specs)))()
    for k, s in enumerate(specs):
        o = arr[k]
        kind = s["kind"]
        o.kind = _lib.KINDS[kind] if isinstance(kind, str) else int(kind)
        o.p = float(s.get("p", 1.0))
        lo = list(s.get("lo", [])) + [0.0] * 4
        hi = list(s.get("hi", s.get("lo", []))) + [0.0] * 4
        for j in range(4):
            o.lo[j] = float(lo[j])
            o.hi[j] = float(hi[j])
        o.out_w, o.out_h = [int(v) for v in s.get("size", (0, 0))]
        o.min_side, o.max_side = [int(v) for v in s.get("side", (0, 0))]
        o.crop_x, o.crop_y = [int(v) for v in s.get("origin", (0, 0))]
        o.interp = _lib.INTERP[s.get("interp", "bilinear")]
        o.border = _lib.BORDER[s.get("border", "constant")]
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


class Pipeline:
    """alb_pipeline: a validated, immutable op list."""

    def __init__(self, specs):
        self.specs = [dict(s) for s in specs]
        ops, n = make_ops(self.specs)
        h = ctypes.c_void_p()
        check(lib().alb_pipeline_create(ops, n, ctypes.byref(h)))
        self.handle = h
        self.n_ops = n

    @classmethod
    def from_json(cls, text):
        """alb_pipeline_from_json: (Pipeline, seed or None) from a config document."""
        h = ctypes.c_void_p()
        seed = ctypes.c_uint64()
        has = ctypes.c_int32()
        check(lib().alb_pipeline_from_json(text.encode("utf-8"), ctypes.byref(h), ctypes.byref(seed),
                                           ctypes.byref(has)))
        self = cls.__new__(cls)
        self.specs = None
        self.handle = h
        self.n_ops = len(json.loads(self.to_json())["transforms"])
        return self, (seed.value if has.value else None)

    def to_json(self, seed=None):
        """alb_pipeline_to_json: the config document (str)."""
        s = None if seed is None else ctypes.byref(ctypes.c_uint64(seed))
        size = ctypes.c_size_t()
        check(lib().alb_pipeline_to_json(self.handle, s, None, 0, ctypes.byref(size)))
        buf = ctypes.create_string_buffer(size.value + 1)
        check(lib().alb_pipeline_to_json(self.handle, s, buf, size.value + 1, ctypes.byref(size)))
        return buf.value.decode("utf-8")

    def __del__(self):
        if getattr(self, "handle", None) and _lib._lib is not None:
            _lib._lib.alb_pipeline_destroy(self.handle)
            self.handle = None

    def output_shape(self, h, w):
        oh, ow = ctypes.c_int32(), ctypes.c_int32()
        check(lib().alb_output_shape(self.handle, h, w, ctypes.byref(oh), ctypes.byref(ow)))
        return oh.value, ow.value

    def sample_params(self, seed, first_image_index, hw):
        """Device-drawn params [n][n_ops][8] and gates [n][n_ops] (synchronous)."""
        hw = np.ascontiguousarray(np.asarray(hw, dtype=np.int32).reshape(-1, 2))
        n = hw.shape[0]
        prm = np.zeros((max(1, n), max(1, self.n_ops), _lib.MAX_PARAMS), np.float64)
        fired = np.zeros((max(1, n), max(1, self.n_ops)), np.uint8)
        check(lib().alb_sample_params(self.handle, seed, first_image_index, hw.ctypes.data, n,
                                      prm.ctypes.data, fired.ctypes.data))
        return prm[:n, :self.n_ops], fired[:n, :self.n_ops]


class Layout:
    """alb_layout: geometry of a ragged batch (desc rows: offset, h, w, pitch)."""

    def __init__(self, desc, channels):
        desc = np.asarray(desc, dtype=np.int64).reshape(-1, 4)
        self.desc = desc.copy()
        self.n = desc.shape[0]
        self.channels = channels
        arr = (AlbImageDesc * max(1, self.n))()
        for i, (off, h, w, pitch) in enumerate(desc.tolist()):
            arr[i].offset, arr[i].height, arr[i].width, arr[i].pitch = off, h, w, pitch
        hd = ctypes.c_void_p()
        check(lib().alb_layout_create(arr, self.n, channels, ctypes.byref(hd)))
        self.handle = hd

    def __del__(self):
        if getattr(self, "handle", None) and _lib._lib is not None:
            _lib._lib.alb_layout_destroy(self.handle)
            self.handle = None


def _ptr(t):
    if t is None:
        return None
    if isinstance(t, torch.Tensor):
        return t.data_ptr()
    return int(t)


class Plan:
    """alb_plan: a pipeline bound to batch layouts (kernel selection, fusion,
    work tables).  Keeps references to its layouts (they must outlive it)."""

    def __init__(self, pipeline, in_layout, out_layout=None, mask_in=None, mask_out=None,
                 max_boxes=0, min_visibility=0.0):
        self.pipeline, self.in_layout, self.out_layout = pipeline, in_layout, out_layout
        self.mask_in, self.mask_out = mask_in, mask_out
        self.max_boxes = max_boxes
        h = ctypes.c_void_p()
        g = lambda L: None if L is None else L.handle
        check(lib().alb_plan_create(pipeline.handle, in_layout.handle, g(out_layout), g(mask_in),
                                    g(mask_out), int(max_boxes), float(min_visibility),
                                    ctypes.byref(h)))
        self.handle = h
        sz = ctypes.c_size_t()
        check(lib().alb_plan_workspace_size(self.handle, ctypes.byref(sz)))
        self.workspace_bytes = sz.value
        self.num_launches = int(lib().alb_plan_num_launches(self.handle))

    def __del__(self):
        if getattr(self, "handle", None) and _lib._lib is not None:
            _lib._lib.alb_plan_destroy(self.handle)
            self.handle = None

    def workspace(self, device="cuda"):
        return torch.empty(self.workspace_bytes + 256, dtype=torch.uint8, device=device)

    @staticmethod
    def _ws(ws):
        p = ws.data_ptr()
        return (p + 255) // 256 * 256, ws.numel() - ((p + 255) // 256 * 256 - p)

    def apply(self, seed, first_image_index, img_in, img_out=None, out_nchw=None,
              mask_in=None, mask_out=None, boxes_in=None, labels_in=None, count_in=None,
              boxes_out=None, labels_out=None, count_out=None, workspace=None, stream=None):
        if workspace is None:
            workspace = self.workspace(img_in.device)
        wp, wn = self._ws(workspace)
        if stream is None:
            stream = torch.cuda.current_stream(img_in.device)
        check(lib().alb_apply(self.handle, int(seed), int(first_image_index), _ptr(img_in),
                              _ptr(img_out), _ptr(out_nchw), _ptr(mask_in), _ptr(mask_out),
                              _ptr(boxes_in), _ptr(labels_in), _ptr(count_in), _ptr(boxes_out),
                              _ptr(labels_out), _ptr(count_out), wp, wn, stream.cuda_stream))

    def apply_host(self, seed, first_image_index, host_in, dev_in, host_out, dev_out,
                   workspace, stream=None):
        """End-to-end: pinned host in -> device -> kernels -> pinned host out."""
        wp, wn = self._ws(workspace)
        if stream is None:
            stream = torch.cuda.current_stream(dev_in.device)
        check(lib().alb_apply_host(self.handle, int(seed), int(first_image_index),
                                   host_in.data_ptr(), host_in.numel() * host_in.element_size(),
                                   dev_in.data_ptr(), host_out.data_ptr(),
                                   host_out.numel() * host_out.element_size(), dev_out.data_ptr(),
                                   wp, wn, stream.cuda_stream))


class Decoder:
    """alb_decoder: nvJPEG batch decode of host JPEG bitstreams into a ragged
    RGB u8 device layout (the input of Plan.apply)."""

    def __init__(self, prefer_hardware=True):
        h = ctypes.c_void_p()
        check(lib().alb_decoder_create(1 if prefer_hardware else 0, ctypes.byref(h)))
        self.handle = h

    def __del__(self):
        if getattr(self, "handle", None) and _lib._lib is not None:
            _lib._lib.alb_decoder_destroy(self.handle)
            self.handle = None

    @property
    def backend(self):
        """1 = hardware JPEG engines, 2 = GPU-assisted Huffman, 0 = default backend"""
        return lib().alb_decoder_backend(self.handle)

    @property
    def hardware(self):
        return self.backend == 1

    def info(self, data):
        """(height, width) of one bitstream (bytes)."""
        h, w = ctypes.c_int32(), ctypes.c_int32()
        check(lib().alb_jpeg_info(self.handle, data, len(data), ctypes.byref(h), ctypes.byref(w)))
        return h.value, w.value

    def decode(self, streams, layout, dev_out):
        """Decode the list of bitstreams into dev_out (uint8 CUDA tensor) laid out
        by `layout` (a 3-channel Layout), on the current stream."""
        n = len(streams)
        arr = (ctypes.c_char_p * max(1, n))(*streams)
        lens = (ctypes.c_size_t * max(1, n))(*[len(s) for s in streams])
        stream = torch.cuda.current_stream(dev_out.device)
        check(lib().alb_decode_jpeg(self.handle, arr, lens, n, layout.handle, _ptr(dev_out), stream.cuda_stream))
