"""B200-native GLCM engine with the capabilities of arXiv 1710.06189.

The hot path (fused quantise + pixel-pair voting into privatised shared-memory
sub-GLCMs, merge, symmetrise/normalise/Haralick, the stream pipeline) is
hand-written CUDA for sm_100a in ``csrc/``, exported through the C ABI in
``include/texforge_cuda.h``. ``texforge`` mirrors the reference's C++ API.
"""
from . import _lib  # noqa: F401
from .texforge import *  # noqa: F401,F403
from .texforge import Engine, default_engine  # noqa: F401

__all__ = [n for n in dir() if not n.startswith("_")]
