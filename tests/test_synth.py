"""The synthetic-input generator (synth/): its own Philox is KAT-pinned and the
recipe's shapes/ranges hold (CPU only)."""
import os

import numpy as np
import torch

from synth import gen

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def test_generator_philox_kat():
    for line in open(os.path.join(GOLD, "philox_kat.txt")):
        if line.startswith("#") or not line.strip():
            continue
        lhs, rhs = line.split(":")
        v = [int(t, 16) for t in lhs.split()]
        want = [int(t, 16) for t in rhs.split()]
        got = gen.philox_t(v[0], v[1], v[2], v[3], v[4], v[5])
        assert [int(t) for t in got] == want


def test_cfg2_sizes():
    s = gen.cfg2_sizes(2000)
    W = np.array([w for _, w in s])
    H = np.array([h for h, _ in s])
    assert W.min() >= 400 and W.max() <= 500 and H.min() >= 300 and H.max() <= 375
    assert (H == np.floor(0.75 * W + 0.5)).all()
    assert len(set(W.tolist())) > 90


def test_images_deterministic_and_ranged():
    a = gen.gen_images([(20, 30), (7, 5)], seed=3)
    b = gen.gen_images([(20, 30), (7, 5)], seed=3)
    c = gen.gen_images([(20, 30), (7, 5)], seed=4)
    assert torch.equal(a.buf, b.buf) and not torch.equal(a.buf, c.buf)
    for k in range(2):
        assert int(a.desc[k][0]) % 256 == 0
    img = gen.gen_images([(300, 400)], seed=0).image(0).astype(int)
    assert img.min() == 0 and img.max() == 255
    # smooth gradient + bounded noise: neighbour differences stay small
    assert np.abs(np.diff(img, axis=1)).max() <= 42


def test_boxes_and_masks():
    sizes = [(64, 80)] * 5
    bx, lb, cnt, masks = gen.gen_boxes(sizes, seed=1, max_boxes=50)
    for i in range(5):
        for k in range(cnt[i]):
            b = bx[i, k]
            assert 0 <= b[0] < b[2] <= 1 and 0 <= b[1] < b[3] <= 1
            assert lb[i, k] == 1 + k % 20
        m = masks.image(i)
        assert m.shape == (64, 80) and m.max() <= 20
