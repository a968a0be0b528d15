"""The C-ABI library builds for sm_100a, loads, exports every symbol the
header declares, validates pipelines on the host, and fails loudly (no CPU
fallback) when there is no GPU.  CPU only."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def L():
    from paper_1809_06839_b200 import build
    build.build()
    from paper_1809_06839_b200 import _lib
    return _lib.lib()


def header_symbols():
    src = open(os.path.join(ROOT, "include", "alb_b200.h")).read()
    return sorted(set(re.findall(r"^\s*(?:[A-Za-z_][\w\s\*]*?)\b(alb_\w+)\s*\(", src, re.M)))


def test_exports_every_header_symbol(L):
    syms = header_symbols()
    assert len(syms) >= 14, syms
    for s in syms:
        assert hasattr(L, s), s
    from paper_1809_06839_b200 import _lib
    assert sorted(_lib.EXPORTS) == syms
    assert L.alb_version() == 1


def test_sass_is_sm100a_and_kernels_present():
    lib = os.path.join(ROOT, "paper_1809_06839_b200", "libalb_b200.so")
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-lelf", lib], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", lib], capture_output=True,
                          text=True).stdout
    for k in ["k_prep", "k_point", "k_rowgather", "k_resample", "k_affine", "k_eq_hist",
              "k_eq_lut", "k_boxes"]:
        assert k in sass, k
    assert "HMMA" not in sass and "UTCHMMA" not in sass  # no tensor-core work on this path


def _status(L, specs):
    from paper_1809_06839_b200.api import make_ops
    ops, n = make_ops(specs)
    h = ctypes.c_void_p()
    rc = L.alb_pipeline_create(ops, n, ctypes.byref(h))
    if rc == 0:
        L.alb_pipeline_destroy(h)
    return rc


def test_pipeline_validation_on_host(L):
    assert _status(L, [{"kind": "HorizontalFlip"}]) == 0
    assert _status(L, [{"kind": 99}]) == -2                      # unknown op
    assert _status(L, [{"kind": "Gamma", "lo": [0.0], "hi": [1.0]}]) == -3  # g <= 0
    assert _status(L, [{"kind": "Brightness", "lo": [-1], "hi": [1]}]) == -3
    assert _status(L, [{"kind": "ShiftScaleRotate", "lo": [0, 0, 0, 0], "hi": [0, 0, 1, 0]}]) == -3
    assert _status(L, [{"kind": "Brightness", "p": 1.5, "lo": [1], "hi": [1]}]) == -3
    assert _status(L, [{"kind": "Brightness", "lo": [1.2], "hi": [0.8]}]) == -3   # lo > hi
    assert _status(L, [{"kind": "Resize", "p": 0.5, "size": (4, 4)}]) == -3      # R17
    assert _status(L, [{"kind": "Normalize"}, {"kind": "HorizontalFlip"}]) == -3
    assert _status(L, [{"kind": "HorizontalFlip"}] * 17) == -5
    assert L.alb_last_error()


def test_output_shape_and_window_errors(L):
    from paper_1809_06839_b200 import Pipeline, AlbError
    p = Pipeline([{"kind": "RandomSizedCrop", "side": (64, 375), "size": (224, 224)},
                  {"kind": "HorizontalFlip", "p": 0.5}])
    assert p.output_shape(375, 500) == (224, 224)
    with pytest.raises(AlbError) as e:
        Pipeline([{"kind": "RandomCrop", "size": (64, 64)}]).output_shape(30, 100)
    assert e.value.code == -1
    with pytest.raises(AlbError):
        Pipeline([{"kind": "PadToSize", "size": (10, 10)}]).output_shape(11, 5)
    assert Pipeline([{"kind": "PadToSize", "size": (512, 512)}]).output_shape(300, 400) == (512, 512)


def test_no_gpu_fails_loudly(L):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_1809_06839_b200 import Layout, AlbError
    import numpy as np
    with pytest.raises(AlbError) as e:
        Layout(np.array([[0, 4, 4, 12]]), 3)
    assert e.value.code == -7  # ALB_E_CUDA: no device, no fallback


def test_missing_library_raises(monkeypatch):
    from paper_1809_06839_b200 import _lib
    monkeypatch.setattr(_lib, "_lib", None)
    monkeypatch.setattr(_lib, "LIB_PATH", "/nonexistent/libalb_b200.so")
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        _lib.lib()


def test_product_never_imports_oracle():
    """The product package shares no code with oracle/ and never loads it."""
    pkg = os.path.join(ROOT, "paper_1809_06839_b200")
    for dp, _, fs in os.walk(pkg):
        for f in fs:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                src = open(os.path.join(dp, f)).read()
                assert "albref" not in src, f
                assert not re.search(r"^\s*(import|from)\s+oracle|#\s*include\s*[<\"].*oracle",
                                     src, re.M), f
