"""B200-native (sm_100a) augmentation hot path of arXiv 1809.06839.

The C ABI (include/alb_b200.h) lives in libalb_b200.so, built in-tree by
paper_1809_06839_b200.build; this package is the thin ctypes binding."""
from ._lib import AlbError, KINDS, lib  # noqa: F401
from .api import Decoder, Layout, Pipeline, Plan, make_ops  # noqa: F401
