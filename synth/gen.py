"""Seeded synthetic inputs.

This module is shared by the CUDA path's tests/bench and by the oracle's
tests.  It holds NONE of the method's arithmetic: it only manufactures input
bytes, boxes and masks.  It carries its own Philox4x32-10 (a third,
independent implementation, KAT-pinned in tests/test_synth.py) keyed with
generator tags >= 0x47454E00 so its streams never collide with the method's
parameter draws (tag 0).

BASELINE.json names no dataset; these images stand in for a natural-photo
corpus of the stated sizes: a per-channel smooth gradient (random direction
mix alpha) plus uniform integer noise in [-20, 20].
"""
from __future__ import annotations

import numpy as np
import torch

TAG_GEN_ALPHA = 0x47454E00
TAG_GEN_NOISE = 0x47454E01
TAG_GEN_SIZE = 0x47454E02
TAG_GEN_BOX = 0x47454E03
_M32 = 0xFFFFFFFF


def philox_t(c0, c1, c2, c3, k0, k1):
    """Philox4x32-10 on int64 tensors holding uint32 values (broadcasting).

    Products wrap modulo 2^64 in int64; masking recovers the exact hi/lo words.
    """
    c0, c1, c2, c3 = [torch.as_tensor(v, dtype=torch.int64) for v in (c0, c1, c2, c3)]
    k0 = int(k0) & _M32
    k1 = int(k1) & _M32
    for r in range(10):
        if r:
            k0 = (k0 + 0x9E3779B9) & _M32
            k1 = (k1 + 0xBB67AE85) & _M32
        p0 = c0 * 0xD2511F53
        p1 = c2 * 0xCD9E8D57
        hi0 = (p0 >> 32) & _M32
        lo0 = p0 & _M32
        hi1 = (p1 >> 32) & _M32
        lo1 = p1 & _M32
        c0, c1, c2, c3 = (hi1 ^ c1) ^ k0, lo1, (hi0 ^ c3) ^ k1, lo0
    return c0, c1, c2, c3


def _u53(a, b):
    return ((a >> 5).double() * 67108864.0 + (b >> 6).double()) * (1.0 / 9007199254740992.0)


def _uniform_int(u, n):
    k = torch.floor(u * n).long()
    return torch.minimum(k, torch.as_tensor(n, dtype=torch.int64) - 1)


def gen_draw(seed, i, a, b, tag, j, device="cpu"):
    """u53 draw j of generator stream (i, a, tag)."""
    w = philox_t(torch.as_tensor(i, device=device), torch.as_tensor(a, device=device),
                 torch.as_tensor(j >> 1, device=device), torch.as_tensor(tag, device=device),
                 seed, seed >> 32)
    return _u53(w[2 * (j & 1)], w[2 * (j & 1) + 1])


def cfg2_sizes(n, seed=0, first_image_index=0):
    """cfg2 sizes (reading R24): W = 400 + uniform_int(101), H = round_half_up(0.75 W)."""
    i = torch.arange(first_image_index, first_image_index + n, dtype=torch.int64)
    u = gen_draw(seed, i, 0, 0, TAG_GEN_SIZE, 0)
    W = 400 + _uniform_int(u, 101)
    H = torch.floor(0.75 * W.double() + 0.5).long()
    return [(int(h), int(w)) for h, w in zip(H.tolist(), W.tolist())]


class Batch:
    """A ragged batch of packed HWC uint8 images in one flat buffer.

    desc[i] = (offset, height, width, pitch) in bytes; images 256-byte aligned."""

    def __init__(self, buf, desc, channels):
        self.buf = buf
        self.desc = desc
        self.channels = channels

    @property
    def n(self):
        return len(self.desc)

    def image(self, i):
        """image i as a contiguous numpy (h, w, c) array (host copy)."""
        off, h, w, pitch = [int(v) for v in self.desc[i]]
        a = self.buf[off:off + h * pitch].view(h, pitch)[:, :w * self.channels]
        a = a.cpu().numpy().reshape(h, w, self.channels)
        return a if self.channels > 1 else a[:, :, 0]

    def to(self, device):
        return Batch(self.buf.to(device), self.desc.copy(), self.channels)


def layout(sizes, channels=3, align=256, pitch_pad=0):
    """Offsets for packed images (pitch = w*c + pitch_pad), each aligned."""
    desc = np.zeros((len(sizes), 4), np.int64)
    off = 0
    for k, (h, w) in enumerate(sizes):
        pitch = w * channels + pitch_pad
        desc[k] = (off, h, w, pitch)
        off += h * pitch
        off = (off + align - 1) // align * align
    return desc, off + align  # trailing slack: aligned-down/up vector loads stay inside


def empty_batch(sizes, channels=3, device="cpu", align=256, pitch_pad=0, fill=0):
    desc, total = layout(sizes, channels, align, pitch_pad)
    buf = torch.full((total,), fill, dtype=torch.uint8, device=device)
    return Batch(buf, desc, channels)


def gen_images(sizes, seed=0, first_image_index=0, device="cpu", align=256, pitch_pad=0,
               chunk_pixels=1 << 23):
    """Gradient + noise images (DESIGN.md input recipe), global index first+k."""
    b = empty_batch(sizes, 3, device, align, pitch_pad)
    n = len(sizes)
    ii = torch.arange(first_image_index, first_image_index + n, dtype=torch.int64, device=device)
    alpha = torch.stack([gen_draw(seed, ii, c, 0, TAG_GEN_ALPHA, 0, device) for c in range(3)],
                        1)  # [n,3]
    k = 0
    while k < n:
        # gather a chunk of whole images
        k1, px = k, 0
        while k1 < n and (px == 0 or px + sizes[k1][0] * sizes[k1][1] <= chunk_pixels):
            px += sizes[k1][0] * sizes[k1][1]
            k1 += 1
        for j in range(k, k1):
            h, w = sizes[j]
            off, _, _, pitch = [int(v) for v in b.desc[j]]
            y = torch.arange(h, dtype=torch.int64, device=device).view(h, 1).expand(h, w)
            x = torch.arange(w, dtype=torch.int64, device=device).view(1, w).expand(h, w)
            gi = first_image_index + j
            words = philox_t(torch.full_like(y, gi), y, x, torch.full_like(y, TAG_GEN_NOISE),
                             seed, seed >> 32)
            a = alpha[j]
            fx = x.double() / (w - 1) if w > 1 else torch.zeros_like(x, dtype=torch.float64)
            fy = y.double() / (h - 1) if h > 1 else torch.zeros_like(y, dtype=torch.float64)
            chans = []
            for c in range(3):
                base = 255.0 * (a[c] * fx + (1.0 - a[c]) * fy)
                noise = torch.floor(words[c].double() * (1.0 / 4294967296.0) * 41.0).long() - 20
                v = torch.floor(base + 0.5).long() + noise
                chans.append(v.clamp(0, 255).to(torch.uint8))
            img = torch.stack(chans, 2).reshape(h, w * 3)
            view = b.buf[off:off + h * pitch].view(h, pitch)
            view[:, :w * 3] = img
        k = k1
    return b


def gen_boxes(sizes, seed=0, first_image_index=0, max_boxes=50, with_mask=True, device="cpu"):
    """cfg5 targets: count = uniform_int(max_boxes+1); box w,h = 16+uniform_int(241)
    (capped at the image size); x_min = uniform_int(W-w+1), y_min likewise;
    label 1+(k mod 20); mask = boxes painted in order over background 0.

    Returns (boxes [n,max_boxes,4] f32 normalized, labels [n,max_boxes] i32,
    count [n] i32, masks Batch or None)."""
    n = len(sizes)
    boxes = np.zeros((n, max_boxes, 4), np.float32)
    labels = np.zeros((n, max_boxes), np.int32)
    count = np.zeros(n, np.int32)
    masks = empty_batch(sizes, 1, "cpu") if with_mask else None
    ii = torch.arange(first_image_index, first_image_index + n, dtype=torch.int64)
    cnt = _uniform_int(gen_draw(seed, ii, 0, 0, TAG_GEN_BOX, 0), max_boxes + 1)
    kk = torch.arange(max_boxes, dtype=torch.int64)
    # draws [n, max_boxes, 4]
    d = torch.stack([gen_draw(seed, ii.view(n, 1), kk.view(1, -1) + 1, 0, TAG_GEN_BOX, j)
                     for j in range(4)], 2)
    Hs = torch.tensor([s[0] for s in sizes], dtype=torch.int64).view(n, 1)
    Ws = torch.tensor([s[1] for s in sizes], dtype=torch.int64).view(n, 1)
    bw = torch.minimum(16 + _uniform_int(d[:, :, 0], 241), Ws)
    bh = torch.minimum(16 + _uniform_int(d[:, :, 1], 241), Hs)
    x0 = torch.floor(d[:, :, 2] * (Ws - bw + 1).double()).long()
    x0 = torch.minimum(x0, Ws - bw)
    y0 = torch.floor(d[:, :, 3] * (Hs - bh + 1).double()).long()
    y0 = torch.minimum(y0, Hs - bh)
    for i in range(n):
        c = int(cnt[i])
        count[i] = c
        H, W = sizes[i]
        if masks is not None:
            off, _, _, pitch = [int(v) for v in masks.desc[i]]
            mv = masks.buf[off:off + H * pitch].view(H, pitch)
        for k in range(c):
            X0, Y0, BW, BH = int(x0[i, k]), int(y0[i, k]), int(bw[i, k]), int(bh[i, k])
            boxes[i, k] = (X0 / W, Y0 / H, (X0 + BW) / W, (Y0 + BH) / H)
            labels[i, k] = 1 + (k % 20)
            if masks is not None:
                mv[Y0:Y0 + BH, X0:X0 + BW] = 1 + (k % 20)
    if masks is not None and device != "cpu":
        masks = masks.to(device)
    return boxes, labels, count, masks
