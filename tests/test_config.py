"""Pipeline config documents:
alb_pipeline_from_json / alb_pipeline_to_json through the C ABI.  Parsing and
validation are host code, so everything but the apply-equivalence test runs
without a GPU."""
import json
import random

import numpy as np
import pytest

from paper_1809_06839_b200 import Pipeline
from paper_1809_06839_b200._lib import AlbError

# one op of every kind, as dict specs (the API's native form) and as the config
# document's {"name", "p", "params"} the schema in include/alb_b200.h defines
ALL = [
    ({"kind": "HorizontalFlip", "p": 0.5}, {}),
    ({"kind": "VerticalFlip", "p": 0.25}, {}),
    ({"kind": "Rotate", "lo": [-30.5], "hi": [45.0], "interp": "nearest", "border": "reflect_101",
      "fill": (1, 2, 3), "mask_fill": 7},
     {"angle": [-30.5, 45.0], "interpolation": "nearest", "border": "reflect_101", "fill": [1, 2, 3],
      "mask_fill": 7}),
    ({"kind": "ShiftScaleRotate", "lo": [-0.0625, -0.1, 0.9, -45], "hi": [0.0625, 0.1, 1.1, 45]},
     {"shift_x": [-0.0625, 0.0625], "shift_y": [-0.1, 0.1], "scale": [0.9, 1.1], "angle": [-45, 45]}),
    ({"kind": "RandomCrop", "size": (64, 48)}, {"width": 64, "height": 48}),
    ({"kind": "PadToSize", "size": (512, 500), "fill": (9, 8, 7), "mask_fill": 255},
     {"width": 512, "height": 500, "fill": [9, 8, 7], "mask_fill": 255}),
    ({"kind": "Resize", "size": (224, 200), "interp": "nearest"},
     {"width": 224, "height": 200, "interpolation": "nearest"}),
    ({"kind": "RandomSizedCrop", "side": (64, 375), "size": (224, 224)},
     {"min_side": 64, "max_side": 375, "width": 224, "height": 224}),
    ({"kind": "Brightness", "lo": [0.8], "hi": [1.2]}, {"beta": [0.8, 1.2]}),
    ({"kind": "Contrast", "lo": [0.7], "hi": [0.7]}, {"c": 0.7}),
    ({"kind": "BrightnessContrast", "lo": [0.8, 0.9], "hi": [1.2, 1.1]}, {"beta": [0.8, 1.2], "c": [0.9, 1.1]}),
    ({"kind": "Gamma", "lo": [2.0], "hi": [2.0]}, {"g": 2.0}),
    ({"kind": "ShiftRGB", "lo": [-20, -10, 0], "hi": [20, 10, 5]}, {"dr": [-20, 20], "dg": [-10, 10], "db": [0, 5]}),
    ({"kind": "ShiftHSV", "lo": [-20, -0.2, -0.1], "hi": [20, 0.2, 0.1]},
     {"dh": [-20, 20], "ds": [-0.2, 0.2], "dv": [-0.1, 0.1]}),
    ({"kind": "Grayscale", "p": 0.1}, {}),
    ({"kind": "Equalize"}, {}),
    ({"kind": "Crop", "origin": (3, 4), "size": (10, 12)}, {"x": 3, "y": 4, "width": 10, "height": 12}),
    ({"kind": "Rotate90", "lo": [1], "hi": [3]}, {"k": [1, 3]}),
    ({"kind": "D4", "lo": [0], "hi": [7]}, {"element": [0, 7]}),
    ({"kind": "GridDistortion", "lo": [-0.3], "hi": [0.3], "num_steps": 5}, {"num_steps": 5, "distort_limit": 0.3}),
    ({"kind": "ElasticTransform", "lo": [34.0, 4.0], "hi": [34.0, 4.0], "border": "reflect_101"},
     {"alpha": 34.0, "sigma": 4.0, "border": "reflect_101"}),
    ({"kind": "Normalize", "mean": (0.485, 0.456, 0.406), "std": (0.229, 0.224, 0.225)},
     {"mean": [0.485, 0.456, 0.406], "std": [0.229, 0.224, 0.225]}),
]


def doc(entries, seed=None):
    d = {"transforms": [{"name": s["kind"], "p": s.get("p", 1.0), "params": prm} for s, prm in entries]}
    if seed is not None:
        d["seed"] = seed
    return json.dumps(d)


def err(text):
    with pytest.raises(AlbError) as e:
        Pipeline.from_json(text)
    return e.value


def test_spec_examples():
    """the empty pipeline round-trips; Gamma g=2 round-trips and
    is gamma(2); an unknown name is rejected with the list of valid names."""
    p, seed = Pipeline.from_json('{"transforms": []}')
    assert seed is None and json.loads(p.to_json()) == {"transforms": []}
    p, _ = Pipeline.from_json('{"name_free": 1}' if False else
                              '{"transforms": [{"name": "Gamma", "p": 1, "params": {"g": 2.0}}]}')
    assert json.loads(p.to_json()) == {"transforms": [{"name": "Gamma", "p": 1.0, "params": {"g": [2.0, 2.0]}}]}
    assert p.to_json() == Pipeline([{"kind": "Gamma", "lo": [2.0], "hi": [2.0]}]).to_json()
    e = err('{"transforms": [{"name": "Sepia", "p": 1, "params": {}}]}')
    assert e.code == -2 and "Sepia" in str(e) and "ElasticTransform" in str(e) and "HorizontalFlip" in str(e)


def test_every_kind_matches_dict_specs_and_round_trips():
    """A document with one op of every kind builds the same pipeline as the
    dict specs (identical serialisation), and serialise -> parse -> serialise is
    a fixpoint with the seed preserved."""
    specs = [s for s, _ in ALL]
    for chunk in (specs[:16], specs[16:]):  # <= 16 ops per pipeline
        ents = [e for e in ALL if e[0] in chunk]
        text = doc(ents, seed=12345)
        p, seed = Pipeline.from_json(text)
        assert seed == 12345
        ref = Pipeline(chunk)
        assert p.to_json(seed) == ref.to_json(12345)
        again, s2 = Pipeline.from_json(p.to_json(seed))
        assert s2 == 12345 and again.to_json(s2) == p.to_json(seed)


def test_numbers_round_trip_exactly():
    rng = random.Random(5)
    for _ in range(200):
        lo = rng.uniform(-1e3, 1e3) * 10 ** rng.randint(-12, 3)
        hi = lo + abs(rng.gauss(0, 1)) * 10 ** rng.randint(-15, 2)
        p = Pipeline([{"kind": "Rotate", "lo": [lo], "hi": [hi]}])
        q, _ = Pipeline.from_json(p.to_json())
        got = json.loads(q.to_json())["transforms"][0]["params"]["angle"]
        assert got == [lo, hi]
    for seed in (0, 1, 2 ** 53 + 1, 2 ** 64 - 1):
        assert Pipeline.from_json(Pipeline([]).to_json(seed))[1] == seed


def test_errors_name_the_culprit():
    e = err('{"transforms": [{"name": "Gamma", "p": 1, "params": {}}]}')
    assert e.code == -1 and "'g'" in str(e)                               # missing required param
    e = err('{"transforms": [{"name": "Resize", "p": 1, "params": {"width": 5}}]}')
    assert e.code == -1 and "'height'" in str(e)
    e = err('{"transforms": [{"name": "Gamma", "params": {"g": 1}}]}')
    assert e.code == -1 and "'p'" in str(e)                               # p is mandatory
    assert err('{"transforms": [{"name": "Gamma", "p": 1.5, "params": {"g": 1}}]}').code == -3
    assert err('{"transforms": [{"name": "Gamma", "p": 1, "params": {"g": -1}}]}').code == -3
    e = err('{"transforms": [{"name": "Gamma", "p": 1, "params": {"g": 1, "gain": 2}}]}')
    assert e.code == -1 and "'gain'" in str(e)                            # unknown param
    e = err('{"transforms": [{"name": "Resize", "p": 1, "params": {"width": 5.5, "height": 4}}]}')
    assert e.code == -1 and "'width'" in str(e)                           # wrong type
    e = err('{"transforms": [{"name": "Rotate", "p": 1, "params": {"angle": 5, "border": "wrap"}}]}')
    assert e.code == -1 and "'border'" in str(e)
    assert err('{"transforms": [], "extra": 1}').code == -1
    assert err('{"seed": -3, "transforms": []}').code == -1
    assert err('{"seed": 18446744073709551616, "transforms": []}').code == -1
    for bad in ('', '{', '{"transforms": [}', '{"transforms": []} x', '[1, 2]', '{"transforms": [], "transforms": []}',
                '{"transforms": [{"name": "Ga\\qmma"}]}', '{"transforms": [1e999]}'):
        assert err(bad).code in (-1, -2), bad
    too_many = doc([ALL[0]] * 17)
    assert err(too_many).code == -5


def test_unicode_and_whitespace():
    text = '\n {\t"transforms" :\r\n [ { "name" : "Gamma" , "p" : 1e0 , "params" : { "g" : [ 5E-1 , 2 ] } } ] }\n'
    p, _ = Pipeline.from_json(text)
    assert json.loads(p.to_json())["transforms"][0]["params"]["g"] == [0.5, 2.0]
    assert err('{"transforms": [{"name": "Gamm\\u00e9", "p": 1}]}').code == -2
    p, _ = Pipeline.from_json('{"transforms": [{"name": "\\u0047amma", "p": 1, "params": {"g": 1}}]}')


def test_fuzzed_documents_never_crash():
    """Random byte edits of valid documents: every call returns OK or an error
    status (no crash, no hang)."""
    rng = random.Random(11)
    base = doc(ALL[:16], seed=7)
    alphabet = '{}[]",:0123456789.-eE abcdefghijklmnopqrstuvwxyz\\\n'
    ok = 0
    for _ in range(3000):
        t = list(base)
        for _ in range(rng.randint(1, 4)):
            i = rng.randrange(len(t))
            op = rng.random()
            if op < 0.4:
                t[i] = rng.choice(alphabet)
            elif op < 0.7:
                del t[i]
            else:
                t.insert(i, rng.choice(alphabet))
        try:
            Pipeline.from_json("".join(t))
            ok += 1
        except AlbError:
            pass
    assert ok < 3000


@pytest.mark.gpu
def test_json_pipeline_applies_like_dict_pipeline():
    """The same pipeline from a config document and from dict specs produces
    identical outputs (images and sampled parameters) on the GPU."""
    import torch
    from synth import gen
    from tests.harness import out_batch
    from paper_1809_06839_b200 import Layout, Plan
    chosen = [ALL[i] for i in (0, 2, 8, 13, 19)]
    sizes = [(45, 130), (70, 17), (129, 300), (1, 1)]
    b = gen.gen_images(sizes, seed=3, first_image_index=0, device="cuda")
    outs = []
    for pipe in (Pipeline.from_json(doc(chosen))[0], Pipeline([s for s, _ in chosen])):
        out = out_batch([pipe.output_shape(h, w) for h, w in sizes])
        plan = Plan(pipe, Layout(b.desc, 3), Layout(out.desc, 3))
        plan.apply(5, 10, b.buf, out.buf)
        torch.cuda.synchronize()
        outs.append([out.image(i) for i in range(len(sizes))])
        pj = pipe.sample_params(5, 10, sizes)
        outs.append(pj)
    for a, c in zip(outs[0], outs[2]):
        assert np.array_equal(a, c)
    assert np.array_equal(outs[1][0], outs[3][0]) and np.array_equal(outs[1][1], outs[3][1])
