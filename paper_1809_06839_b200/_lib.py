"""ctypes binding of libalb_b200.so (include/alb_b200.h): argument marshalling
only.  Every step of the hot path runs in the sm_100a kernels of the library;
there is no CPU fallback -- a missing library raises immediately."""
from __future__ import annotations

import ctypes
import os

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(PKG, "libalb_b200.so")

ALB_OK = 0
STATUS = {0: "ALB_OK", -1: "ALB_E_INVALID_ARG", -2: "ALB_E_UNKNOWN_OP", -3: "ALB_E_RANGE",
          -4: "ALB_E_SHAPE", -5: "ALB_E_UNSUPPORTED", -6: "ALB_E_ALIGN", -7: "ALB_E_CUDA",
          -8: "ALB_E_WORKSPACE"}
KINDS = {
    "HorizontalFlip": 0, "VerticalFlip": 1, "Rotate": 2, "ShiftScaleRotate": 3,
    "RandomCrop": 4, "PadToSize": 5, "Resize": 6, "RandomSizedCrop": 7,
    "Brightness": 8, "Contrast": 9, "BrightnessContrast": 10, "Gamma": 11,
    "ShiftRGB": 12, "ShiftHSV": 13, "Grayscale": 14, "Equalize": 15,
    "Normalize": 16, "Crop": 17, "Rotate90": 18, "D4": 19, "GridDistortion": 20, "ElasticTransform": 21,
}
INTERP = {"nearest": 0, "bilinear": 1}
BORDER = {"constant": 0, "reflect_101": 1}
MAX_OPS = 16
MAX_PARAMS = 8


class AlbOp(ctypes.Structure):
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


class AlbImageDesc(ctypes.Structure):
    _fields_ = [("offset", ctypes.c_int64), ("height", ctypes.c_int32),
                ("width", ctypes.c_int32), ("pitch", ctypes.c_int32),
                ("reserved", ctypes.c_int32)]


class AlbError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__("%s (%d): %s" % (STATUS.get(code, "?"), code, msg))
        self.code = code
        self.name = STATUS.get(code, "?")


EXPORTS = ["alb_pipeline_create", "alb_pipeline_destroy", "alb_output_shape",
           "alb_layout_create", "alb_layout_destroy", "alb_plan_create", "alb_plan_destroy",
           "alb_plan_workspace_size", "alb_plan_num_launches", "alb_apply", "alb_apply_host",
           "alb_sample_params", "alb_last_error", "alb_version", "alb_pipeline_from_json",
           "alb_pipeline_to_json", "alb_decoder_create", "alb_decoder_destroy", "alb_decoder_backend",
           "alb_jpeg_info", "alb_decode_jpeg"]

_lib = None


def lib():
    """Load the in-tree library; raise loudly if it has not been built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError("libalb_b200.so is not built (run __graft_entry__.build() or "
                           "python -m paper_1809_06839_b200.build); there is no CPU fallback")
    L = ctypes.CDLL(LIB_PATH)
    P = ctypes.POINTER
    vp = ctypes.c_void_p
    L.alb_pipeline_create.argtypes = [P(AlbOp), ctypes.c_int32, P(vp)]
    L.alb_pipeline_destroy.argtypes = [vp]
    L.alb_pipeline_destroy.restype = None
    L.alb_output_shape.argtypes = [vp, ctypes.c_int32, ctypes.c_int32, P(ctypes.c_int32),
                                   P(ctypes.c_int32)]
    L.alb_layout_create.argtypes = [P(AlbImageDesc), ctypes.c_int32, ctypes.c_int32, P(vp)]
    L.alb_layout_destroy.argtypes = [vp]
    L.alb_layout_destroy.restype = None
    L.alb_plan_create.argtypes = [vp, vp, vp, vp, vp, ctypes.c_int32, ctypes.c_float, P(vp)]
    L.alb_plan_destroy.argtypes = [vp]
    L.alb_plan_destroy.restype = None
    L.alb_plan_workspace_size.argtypes = [vp, P(ctypes.c_size_t)]
    L.alb_plan_num_launches.argtypes = [vp]
    L.alb_apply.argtypes = [vp, ctypes.c_uint64, ctypes.c_uint64, vp, vp, vp, vp, vp,
                            vp, vp, vp, vp, vp, vp, vp, ctypes.c_size_t, vp]
    L.alb_apply_host.argtypes = [vp, ctypes.c_uint64, ctypes.c_uint64, vp, ctypes.c_size_t, vp,
                                 vp, ctypes.c_size_t, vp, vp, ctypes.c_size_t, vp]
    L.alb_sample_params.argtypes = [vp, ctypes.c_uint64, ctypes.c_uint64, vp, ctypes.c_int32,
                                    vp, vp]
    L.alb_last_error.restype = ctypes.c_char_p
    L.alb_last_error.argtypes = []
    L.alb_version.restype = ctypes.c_int32
    L.alb_pipeline_from_json.argtypes = [ctypes.c_char_p, P(vp), P(ctypes.c_uint64), P(ctypes.c_int32)]
    L.alb_pipeline_to_json.argtypes = [vp, P(ctypes.c_uint64), ctypes.c_char_p, ctypes.c_size_t,
                                       P(ctypes.c_size_t)]
    L.alb_decoder_create.argtypes = [ctypes.c_int32, P(vp)]
    L.alb_decoder_destroy.argtypes = [vp]
    L.alb_decoder_backend.argtypes = [vp]
    L.alb_decoder_backend.restype = ctypes.c_int32
    L.alb_jpeg_info.argtypes = [vp, ctypes.c_char_p, ctypes.c_size_t, P(ctypes.c_int32), P(ctypes.c_int32)]
    L.alb_decode_jpeg.argtypes = [vp, P(ctypes.c_char_p), P(ctypes.c_size_t), ctypes.c_int32, vp, vp, vp]
    for name in ["alb_decoder_create", "alb_jpeg_info", "alb_decode_jpeg",
                 "alb_pipeline_create", "alb_output_shape", "alb_layout_create",
                 "alb_plan_create", "alb_plan_workspace_size", "alb_apply", "alb_apply_host",
                 "alb_sample_params", "alb_pipeline_from_json", "alb_pipeline_to_json"]:
        getattr(L, name).restype = ctypes.c_int32
    _lib = L
    return L


def check(rc):
    if rc != ALB_OK:
        raise AlbError(rc, lib().alb_last_error().decode(errors="replace"))
